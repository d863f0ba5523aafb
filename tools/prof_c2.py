"""A short C2 s-GMRES run for kernel profiling (ncu -k regex:... -s N -c M python tools/prof_c2.py).

    python tools/prof_c2.py [iterations] [nx] [s] [m]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    it = int(sys.argv[1]) if len(sys.argv) > 1 else 80
    nx = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    s = int(sys.argv[3]) if len(sys.argv) > 3 else 4
    m = int(sys.argv[4]) if len(sys.argv) > 4 else 10
    import torch
    from paper_2001_04886_b200 import Context, SStepConfig, convection_diffusion, splitmix64_uniform
    from paper_2001_04886_b200.sstep import sgmres_solve_device
    st = convection_diffusion(2, nx, 50.0)
    f = splitmix64_uniform(20010486, st.n)
    ctx = Context(0)
    op = ctx.stencil(st)
    fd = torch.from_numpy(f).cuda()
    xd = torch.zeros(st.n, dtype=torch.float64, device="cuda")
    cfg = SStepConfig(s=s, m=m, tol=0.0, max_iterations=it)
    rep = sgmres_solve_device(op, fd.data_ptr(), xd.data_ptr(), cfg)
    torch.cuda.synchronize()
    print("iterations", rep.iterations, "breakdown", rep.breakdown)


if __name__ == "__main__":
    main()
