"""ILU(0)-preconditioned solves on the GPU (the paper's Table 6.1 setting, h^2-scaled operator).

    python tools/bench_ilu0.py [nx ...]

For each grid: the host factorization time, the device time of one preconditioned apply
A (LU)^{-1} (two level-scheduled triangular solves + the stencil kernel) and of the two solves
alone, and solve_linear (driver flow) with 2-Omin(2) and 2-GMRES(5) to a relative 1e-8.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def csr_2d(st):
    """CSR of the 5-point stencil (natural order, ascending columns, Dirichlet truncation)."""
    nx, ny = st.nx, st.ny
    offs, cols, vals = [0], [], []
    for j in range(ny):
        for i in range(nx):
            p = j * nx + i
            for q, c, ok in ((p - nx, st.coef[1], j > 0), (p - 1, st.coef[2], i > 0), (p, st.coef[3], True),
                             (p + 1, st.coef[4], i + 1 < nx), (p + nx, st.coef[5], j + 1 < ny)):
                if ok:
                    cols.append(q)
                    vals.append(c)
            offs.append(len(cols))
    return np.array(offs, np.uint64), np.array(cols, np.uint64), np.array(vals)


def main():
    import torch
    from paper_2001_04886_b200 import Context, SStepConfig, convection_diffusion, solve_linear, splitmix64_uniform
    ctx = Context(0)
    for nx in [int(a) for a in sys.argv[1:]] or [64, 256, 1024]:
        st = convection_diffusion(2, nx, 50.0)
        offs, cols, vals = csr_2d(st)
        f = splitmix64_uniform(20010486, st.n)
        t0 = time.perf_counter()
        op = ctx.ilu0(offs, cols, vals)
        t_fac = time.perf_counter() - t0
        x = splitmix64_uniform(3, st.n)
        op.apply(x)  # warm-up
        reps = 20
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            op.apply(x)
        t_apply = (time.perf_counter() - t0) / reps
        t0 = time.perf_counter()
        for _ in range(reps):
            op.ilu0_solve(x)
        t_solve = (time.perf_counter() - t0) / reps
        ctx.reset_stats()
        ctx.set_profiling(True)
        for _ in range(reps):
            op.ilu0_solve(x)
        torch.cuda.synchronize()
        ks = ctx.kernel_stats()
        ctx.set_profiling(False)
        dev = sum(v["ms"] for k, v in ks.items() if k.startswith("ilu_")) / reps
        line = (f"nx={nx}: factor(host) {t_fac * 1e3:.1f} ms, A(LU)^-1 apply {t_apply * 1e3:.3f} ms, (LU)^-1 "
                f"{t_solve * 1e3:.3f} ms (host round trip incl.), device {dev * 1e3:.1f} us per (LU)^-1")
        for method, cfg in (("somin", dict(s=2, k=2)), ("sgmres", dict(s=2, m=5))):
            c = SStepConfig(tol=1e-8 * float(np.linalg.norm(f)), max_iterations=20000, **cfg)
            t0 = time.perf_counter()
            xs, rep = solve_linear(ctx, offs, cols, vals, f, np.zeros(st.n), method, c, precondition=True)
            dt = time.perf_counter() - t0
            line += f" | {method} {rep.iterations} it, {dt * 1e3:.1f} ms, converged {rep.converged}"
        print(line, flush=True)


if __name__ == "__main__":
    main()
