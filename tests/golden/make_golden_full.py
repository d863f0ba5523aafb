"""Full-size golden fixtures for the BASELINE configurations, generated from the UNMODIFIED
reference (oracle/_ref/libskref.so) and, for the per-block LSQ residuals the reference's
SolveReport does not expose, from the oracle restatement (pinned bit-for-bit to the reference
by tests/test_oracle_pin.py; this script re-checks that pin on the full-size histories).

Run in the build container (needs /root/reference to have built oracle/_ref; ~10 min on 8
cores, up to ~20 GB of RAM):

    make -C oracle && python tests/golden/make_golden_full.py [case ...]

Cases (VERDICT r01 "Next round" item 1):
  C2_full_2cyc   configs[1] at 1024^2, two restart cycles (max_iterations = 2 s m): per-cycle
                 residuals, op_history, per-block LSQ residuals rho of both cycles, and the
                 same quantities under three perturbed dot-product summation orders (the
                 reference's own envelope, sstep.hpp:493-654)
  C2_full_conv   configs[1] at 1024^2 solved to rel 1e-8 (the same-input reference run:
                 cycle count, history, iterate sample)
  C3_full_s{1,2,4}  configs[2] at 256^3, 50 fixed s-steps (sstep.hpp:142-249): history, ||x||,
                 a strided sample of x, sha256 of the iterate's bits; envelope in the blocked
                 tree order
  C4_class_4096  configs[3] operator at 4096^2 (the largest 2D grid the 62 GB host holds in
                 reasonable time), 50 fixed s-steps: the breakdown class
  C5_class_256   configs[4] operator (variable k) at 256^3, 50 fixed s-steps: the breakdown
                 class
Only x samples (every XSTRIDE-th entry) are stored, so the fixtures stay small.
"""
from __future__ import annotations

import hashlib
import json
import multiprocessing as mp
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "full")
XSAMPLES = 16384


def _problem(dim, nx, conv, variable_k=False):
    from oracle import Oracle
    from paper_2001_04886_b200.problems import K_SEED, RHS_SEED, convection_diffusion, splitmix64_uniform
    port = Oracle("port")
    st = convection_diffusion(dim, nx, conv, variable_k=variable_k)
    kcell = port.lognormal(K_SEED, st.n) if variable_k else None
    a = port.stencil_csr(dim, st.nx, st.ny, st.nz, st.coef, kcell=kcell, ch2=st.ch2)
    f = splitmix64_uniform(RHS_SEED, st.n)
    sdesc = dict(dim=dim, nx=st.nx, ny=st.ny, nz=st.nz, coef=list(st.coef), ch2=st.ch2, variable_k=variable_k,
                 rhs_seed=RHS_SEED, k_seed=K_SEED, conv=conv)
    return a, f, sdesc


def _xsample(x):
    stride = max(1, x.size // XSAMPLES)
    return stride, x[::stride].copy()


def _result_arrays(res, prefix=""):
    stride, xs = _xsample(res.x)
    return {prefix + "history": np.array(res.residual_history),
            prefix + "op_history": np.array(res.op_history, dtype=np.uint64).reshape(-1, 5),
            prefix + "op_counts": np.array(res.op_counts, dtype=np.uint64),
            prefix + "block_rho": np.array(res.block_rho, dtype=np.float64),
            prefix + "xsample": xs}, stride


def _result_meta(res, x):
    return dict(converged=res.converged, iterations=res.iterations, cycles=res.cycles,
                final_residual=res.final_residual, breakdown=res.breakdown, notes=res.notes,
                fallback_cycles=res.fallback_cycles, steady_iteration=res.steady_iteration,
                xnorm=float(np.linalg.norm(x)), x_sha256=hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest())


def job_c2_2cyc():
    from oracle import Oracle
    a, f, sd = _problem(2, 1024, 50.0)
    cfg = dict(s=4, m=10, tol=1e-8 * float(np.linalg.norm(f)), max_iterations=2 * 4 * 10)
    ref = Oracle("reference").sstep("sgmres", a, f, None, **cfg)
    port = Oracle("port")
    base = port.sstep("sgmres", a, f, None, **cfg)
    assert base.residual_history == ref.residual_history, "port not pinned to the reference at C2 size"
    assert np.array_equal(base.x.view(np.uint64), ref.x.view(np.uint64))
    arrays, stride = _result_arrays(ref)
    arrays["block_rho"] = np.array(base.block_rho)
    meta = dict(_result_meta(ref, ref.x), cfg=cfg, stencil=sd, xstride=stride, method="sgmres",
                ref="BASELINE configs[1] at full size, 2 restart cycles; block_rho from the pinned port")
    env = {}
    for mode, nm in {1: "blocked tree", 2: "reversed", 3: "compensated"}.items():
        port.set_dot_mode(mode)
        r = port.sstep("sgmres", a, f, None, **cfg)
        port.set_dot_mode(0)
        arrays[f"env{mode}_block_rho"] = np.array(r.block_rho)
        arrays[f"env{mode}_history"] = np.array(r.residual_history)
        env[nm] = dict(iterations=r.iterations, breakdown=r.breakdown)
    meta["envelope_modes"] = env
    return "C2_full_2cyc", arrays, meta


def job_c2_conv():
    from oracle import Oracle
    a, f, sd = _problem(2, 1024, 50.0)
    cfg = dict(s=4, m=10, tol=1e-8 * float(np.linalg.norm(f)))
    ref = Oracle("reference").sstep("sgmres", a, f, None, **cfg)
    arrays, stride = _result_arrays(ref)
    meta = dict(_result_meta(ref, ref.x), cfg=cfg, stencil=sd, xstride=stride, method="sgmres",
                ref="BASELINE configs[1] at full size, solved to rel 1e-8 (same-input reference run)")
    return "C2_full_conv", arrays, meta


def job_c3(s, envelope=False):
    from oracle import Oracle
    a, f, sd = _problem(3, 256, 20.0)
    cfg = dict(s=s, k=2, tol=0.0, max_iterations=50)
    if envelope:  # the reference's sensitivity to a GPU-like summation order
        port = Oracle("port")
        port.set_dot_mode(1)
        r = port.sstep("somin", a, f, None, **cfg)
        stride, xs = _xsample(r.x)
        return f"C3_full_s{s}_env", {"history": np.array(r.residual_history), "xsample": xs}, \
            dict(iterations=r.iterations, xnorm=float(np.linalg.norm(r.x)), mode="blocked tree")
    ref = Oracle("reference").sstep("somin", a, f, None, **cfg)
    arrays, stride = _result_arrays(ref)
    meta = dict(_result_meta(ref, ref.x), cfg=cfg, stencil=sd, xstride=stride, method="somin",
                ref=f"BASELINE configs[2] at full size 256^3, s={s}, 50 fixed s-steps")
    return f"C3_full_s{s}", arrays, meta


def job_c4():
    from oracle import Oracle
    a, f, sd = _problem(2, 4096, 50.0)
    cfg = dict(s=8, m=8, tol=0.0, max_iterations=50 * 8)
    ref = Oracle("reference").sstep("sgmres", a, f, None, **cfg)
    arrays, stride = _result_arrays(ref)
    meta = dict(_result_meta(ref, ref.x), cfg=cfg, stencil=sd, xstride=stride, method="sgmres",
                ref="BASELINE configs[3] operator at 4096^2, 50 fixed s-steps (breakdown class)")
    return "C4_class_4096", arrays, meta


def job_c5():
    from oracle import Oracle
    a, f, sd = _problem(3, 256, 20.0, variable_k=True)
    cfg = dict(s=8, k=2, tol=0.0, max_iterations=50)
    ref = Oracle("reference").sstep("somin", a, f, None, **cfg)
    arrays, stride = _result_arrays(ref)
    meta = dict(_result_meta(ref, ref.x), cfg=cfg, stencil=sd, xstride=stride, method="somin",
                ref="BASELINE configs[4] operator (variable k) at 256^3, 50 fixed s-steps (breakdown class)")
    return "C5_class_256", arrays, meta


JOBS = {
    "C2_full_2cyc": (job_c2_2cyc, ()),
    "C2_full_conv": (job_c2_conv, ()),
    "C3_full_s1": (job_c3, (1,)), "C3_full_s2": (job_c3, (2,)), "C3_full_s4": (job_c3, (4,)),
    "C3_full_s1_env": (job_c3, (1, True)), "C3_full_s2_env": (job_c3, (2, True)), "C3_full_s4_env": (job_c3, (4, True)),
    "C4_class_4096": (job_c4, ()),
    "C5_class_256": (job_c5, ()),
}


def _run(name):
    t0 = time.time()
    fn, args = JOBS[name]
    nm, arrays, meta = fn(*args)
    np.savez_compressed(os.path.join(OUT, nm + ".npz"), **arrays)
    meta["generated_s"] = round(time.time() - t0, 1)
    with open(os.path.join(OUT, nm + ".json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(f"{nm}: {time.time() - t0:.1f} s", flush=True)
    return nm


def main():
    os.makedirs(OUT, exist_ok=True)
    todo = sys.argv[1:] or list(JOBS)
    # longest first; every job in its own process (single-threaded reference)
    with mp.get_context("spawn").Pool(min(len(todo), os.cpu_count() or 1)) as pool:
        for nm in pool.imap_unordered(_run, todo):
            pass


if __name__ == "__main__":
    main()
