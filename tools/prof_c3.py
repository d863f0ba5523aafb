"""A short C3 s-Omin run (256^3, s=4, k=2) for kernel profiling: python tools/prof_c3.py [iterations] [s]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    it = int(sys.argv[1]) if len(sys.argv) > 1 else 10
    s = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    import torch
    from paper_2001_04886_b200 import Context, SStepConfig, convection_diffusion, splitmix64_uniform
    from paper_2001_04886_b200.sstep import somin_solve_device
    st = convection_diffusion(3, 256, 20.0)
    f = splitmix64_uniform(20010486, st.n)
    ctx = Context(0)
    op = ctx.stencil(st)
    fd = torch.from_numpy(f).cuda()
    xd = torch.zeros(st.n, dtype=torch.float64, device="cuda")
    rep = somin_solve_device(op, fd.data_ptr(), xd.data_ptr(), SStepConfig(s=s, k=2, tol=0.0, max_iterations=it))
    torch.cuda.synchronize()
    print("iterations", rep.iterations, "breakdown", rep.breakdown)


if __name__ == "__main__":
    main()
