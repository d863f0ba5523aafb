"""Throughput of every BASELINE configuration on one GPU (beside bench.py's C2 headline).

    python tools/bench_configs.py [C1 C3s1 C3s2 C3s4 C3s8 C4 C5] [--steps K]

Each line: s-steps/s, ms per s-step, the SURVEY 8(d) effective HBM GB/s and fraction of the
measured peak, plus the per-kernel-class breakdown of one profiled run.  Fixed-step configs
run with tol = 0 (the reference's "fixed N s-steps"); s = 8 runs continue past the
reference's basis collapse only if the GPU's Gram solves do not collapse -- the breakdown (if
any) is reported.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def somin_vecs(s, k, extra=0):
    return 3 * k * s + 7 * s + 6 + extra


def sgmres_vecs_per_sstep(s, m):
    return (2 * s * m * (m - 1) + (m - 1) * (4 * s + 5) + 3 * m * s + 3 * s + 13) / m


CASES = {
    "C1": dict(method="somin", dim=2, nx=128, conv=10.0, s=4, k=2, rel_tol=1e-8, steps=200, vecs=somin_vecs(4, 2, 5)),
    "C3s1": dict(method="somin", dim=3, nx=256, conv=20.0, s=1, k=2, steps=100, vecs=somin_vecs(1, 2)),
    "C3s2": dict(method="somin", dim=3, nx=256, conv=20.0, s=2, k=2, steps=100, vecs=somin_vecs(2, 2)),
    "C3s4": dict(method="somin", dim=3, nx=256, conv=20.0, s=4, k=2, steps=100, vecs=somin_vecs(4, 2)),
    "C3s8": dict(method="somin", dim=3, nx=256, conv=20.0, s=8, k=2, steps=100, vecs=somin_vecs(8, 2)),
    "C4": dict(method="sgmres", dim=2, nx=16384, conv=50.0, s=8, m=8, steps=48, vecs=sgmres_vecs_per_sstep(8, 8)),
    "C5": dict(method="somin", dim=3, nx=512, conv=20.0, s=8, k=2, steps=50, vecs=somin_vecs(8, 2, 1), vark=True),
}


def run(name, steps_override=None):
    from paper_2001_04886_b200 import Context, SStepConfig, convection_diffusion, splitmix64_uniform
    from paper_2001_04886_b200.sstep import sgmres_solve_device, somin_solve_device
    import torch
    c = CASES[name]
    st = convection_diffusion(c["dim"], c["nx"], c["conv"], variable_k=c.get("vark", False))
    kcell = None
    if c.get("vark"):
        from paper_2001_04886_b200.problems import lognormal_k
        kcell = lognormal_k(4886, st.n)
    f = splitmix64_uniform(20010486, st.n)
    steps = steps_override or c["steps"]
    tol = c["rel_tol"] * float(np.linalg.norm(f)) if "rel_tol" in c else 0.0
    s = c["s"]
    if c["method"] == "somin":
        cfg = SStepConfig(s=s, k=c["k"], tol=tol, max_iterations=steps)
        fn = somin_solve_device
    else:
        cfg = SStepConfig(s=s, m=c["m"], tol=tol, max_iterations=steps * s)
        fn = sgmres_solve_device
    ctx = Context(0)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    op = ctx.stencil(st, kcell=kcell)
    fd = torch.from_numpy(f).cuda()
    xd = torch.zeros(st.n, dtype=torch.float64, device="cuda")
    del f
    xd.zero_()
    rep = fn(op, fd.data_ptr(), xd.data_ptr(), cfg)  # warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xd.zero_()
    e0.record(stream)
    rep = fn(op, fd.data_ptr(), xd.data_ptr(), cfg)
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    sst = rep.iterations / (s if c["method"] == "sgmres" else 1)
    ctx.reset_stats()
    ctx.set_profiling(True)
    xd.zero_()
    fn(op, fd.data_ptr(), xd.data_ptr(), cfg)
    torch.cuda.synchronize()
    kst = ctx.kernel_stats()
    ctx.set_profiling(False)
    rate = sst / (ms / 1e3)
    eff = c["vecs"] * 8.0 * st.n * rate / 1e9
    out = dict(config=name, n=st.n, s=s, s_steps=sst, ms=round(ms, 2), s_steps_per_s=round(rate, 2),
               ms_per_s_step=round(ms / max(sst, 1), 4), effective_hbm_gbs=round(eff, 1),
               effective_hbm_frac=round(eff / PEAK, 4), breakdown=rep.breakdown, converged=rep.converged,
               kernels={k: dict(launches=v["launches"], ms=round(v["ms"], 3),
                                gbs=round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)) for k, v in kst.items()})
    print(json.dumps(out), flush=True)
    del ctx, op, fd, xd
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    steps = None
    if "--steps" in sys.argv:
        steps = int(sys.argv[sys.argv.index("--steps") + 1])
        args = [a for a in args if a != str(steps)]
    for name in args or list(CASES):
        try:
            run(name, steps)
        except Exception as e:  # keep going: report the failure line
            print(json.dumps(dict(config=name, error=f"{type(e).__name__}: {e}")), flush=True)
