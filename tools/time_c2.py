"""Quick A/B timing of the C2 s-GMRES solve (device-resident f, x): s-steps/s over R repeats.

    python tools/time_c2.py [repeats] [nx] [s] [m]

Environment switches of the library (SKC_PF, SKC_ZFUSE, SKC_ORTH, ...) apply, so the same
command under different settings compares kernel variants.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
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
    cfg = SStepConfig(s=s, m=m, tol=1e-8 * float(np.linalg.norm(f)), max_iterations=100000)
    best = None
    for r in range(reps + 1):
        xd.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = sgmres_solve_device(op, fd.data_ptr(), xd.data_ptr(), cfg)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        ss = rep.iterations / s
        if r > 0:
            best = dt if best is None else min(best, dt)
        print(f"rep {r}: {rep.iterations} inner steps ({ss:.0f} s-steps), cycles {rep.cycles}, "
              f"{dt * 1e3:.1f} ms, {ss / dt:.0f} s-steps/s, converged {rep.converged}")
    print(f"BEST {ss / best:.1f} s-steps/s  env SPOW={os.environ.get('SKC_SPOW', '-')} "
          f"ZFUSE={os.environ.get('SKC_ZFUSE', '-')} ORTH={os.environ.get('SKC_ORTH', '-')}")


if __name__ == "__main__":
    main()
