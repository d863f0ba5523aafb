#!/usr/bin/env python
"""bench.py -- headline benchmark (BASELINE.json metric) for the B200 s-step solvers.

Headline workload (BASELINE configs[1], the metric's single-GPU configuration; default):
    C2: s-step GMRES, s=4, m=10, 2D 5-point convection-diffusion (c=50, h^2-scaled),
        1024x1024, f ~ U[-1,1] (splitmix64, seed 20010486), x0 = 0, tol = 1e-8 ||f||.
    One step = one full solve to tolerance (about 90 restart cycles / 900 s-steps).
metric: s-step iterations per second (one s-step = one block iteration of s inner steps),
with the effective HBM GB/s of the SURVEY 8(d) algorithmic byte model beside it.

The default N=1 run also measures, in the same JSON line under "secondary", the other
BASELINE configurations that carry the north star's scaling targets, each with its own
roofline, e2e and cpu_baseline:
    C3s4: s-step Orthomin s=4 k=2, 3D 7-point c=20, 256^3, 100 fixed s-steps (configs[2])
    C4:   s-step GMRES s=8 m=8, 2D 5-point c=50, 16384^2 (268M unknowns, the largest
          single-GPU grid), 50 fixed s-steps (configs[3])
    C5:   s-step Orthomin s=8 k=2, 3D 7-point variable k, 512^3, 50 fixed s-steps (configs[4])
The s = 8 configurations run in the fixed-step benchmark mode (skc_sstep_config.fixed_steps:
only the Gram pivot-ratio and LSQ rank aborts are bypassed); the reference stops
at those aborts, so their results past that point are flagged numerically meaningless.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config C2|C1|C3s1|C3s2|C3s4|C3s8|C4|C5] [--no-secondary]

Multi-GPU (torchrun, N>1): C2 is weak scaling by row slabs (every GPU owns a 1024 x 1024
slab of a 1024 x (1024 N) grid); C3/C4/C5 (--config) are strong scaling of the global grid
split into row slabs (y in 2D, z in 3D).  Halo rows and dot sums go over NCCL; the time is the
max over ranks of the device time.
--impl reference times the reference's own CPU implementation (oracle/_ref, the unmodified
reference headers; the C restatement oracle/liboracle.so if _ref is absent) on the C2
workload, one restart cycle per step per host thread, all host threads in parallel.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 20010486
K_SEED = 4886
METRIC = "s-step iterations/sec and effective HBM GB/s (fraction of peak) at 1/2/4/8 B200"
UNIT = "s-steps/s"

CONFIGS = {
    "C1": dict(method="somin", dim=2, nx=128, conv=10.0, s=4, k=2, rel_tol=1e-8, max_steps=200,
               workload="C1: s-step Orthomin s=4 k=2, 2D 5-point conv-diff c=10 (h^2-scaled), 128x128, tol 1e-8 rel or 200 s-steps"),
    "C2": dict(method="sgmres", dim=2, nx=1024, conv=50.0, s=4, m=10, rel_tol=1e-8,
               workload="C2: s-step GMRES s=4 m=10, 2D 5-point conv-diff c=50 (h^2-scaled), 1024x1024, tol 1e-8 rel, x0=0"),
    "C4": dict(method="sgmres", dim=2, nx=16384, conv=50.0, s=8, m=8, fixed=50, cpu_nx=1024,
               workload="C4: s-step GMRES s=8 m=8, 2D 5-point conv-diff c=50 (h^2-scaled), 16384x16384, 50 fixed s-steps (7 cycles: max_iterations is checked at cycle start), fixed-step mode"),
    "C5": dict(method="somin", dim=3, nx=512, conv=20.0, s=8, k=2, fixed=50, vark=True, cpu_nx=64,
               workload="C5: s-step Orthomin s=8 k=2, 3D 7-point conv-diff c=20, variable k=exp(N(0,1)), 512^3, 50 fixed s-steps, fixed-step mode"),
}
for _s in (1, 2, 4, 8):
    CONFIGS[f"C3s{_s}"] = dict(method="somin", dim=3, nx=256, conv=20.0, s=_s, k=2, fixed=100,
                               workload=f"C3: s-step Orthomin s={_s} k=2, 3D 7-point conv-diff c=20 (h^2-scaled), 256^3, 100 fixed s-steps"
                               + (", fixed-step mode" if _s == 8 else ""))
SECONDARY = ["C3s4", "C4", "C5"]


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def model_vecs_per_sstep(c):
    """SURVEY 8(d) algorithmic vectors per s-step (block-CGS-equivalent passes)."""
    s = c["s"]
    if c["method"] == "sgmres":
        m = c["m"]
        return (2 * s * m * (m - 1) + (m - 1) * (4 * s + 5) + 3 * m * s + 3 * s + 13) / m
    k = c["k"]
    return 3 * k * s + 7 * s + 6 + (1 if c.get("vark") else 0)  # (+1 vec: k per operator sweep)


def sstep_cfg(c, f):
    from paper_2001_04886_b200 import SStepConfig
    s = c["s"]
    fixed = "fixed" in c
    tol = 0.0 if fixed else c["rel_tol"] * float(np.linalg.norm(f))
    if c["method"] == "sgmres":
        iters = c["fixed"] * s if fixed else 10 ** 7
        return SStepConfig(s=s, m=c["m"], tol=tol, max_iterations=iters, fixed_steps=fixed and s == 8)
    iters = c["fixed"] if fixed else c.get("max_steps", 10 ** 7)
    return SStepConfig(s=s, k=c["k"], tol=tol, max_iterations=iters, fixed_steps=fixed and s == 8)


def config_json(name, c, n_gpus, scaling):
    out = {"workload": c["workload"], "method": c["method"], "s": c["s"], "grid": [c["nx"]] * c["dim"],
           "conv": c["conv"], "rhs_seed": SEED}
    out.update({"m": c["m"]} if c["method"] == "sgmres" else {"k": c["k"]})
    if "fixed" in c:
        out["fixed_s_steps"] = c["fixed"]
        out["fixed_step_mode"] = c["s"] == 8
    else:
        out["rel_tol"] = c["rel_tol"]
    vec_mb = 8.0 * c["nx"] ** c["dim"] / 1e6
    out["l2"] = f"every vector is {vec_mb:.0f} MB; the working set exceeds the 126 MB L2; no flush"
    if n_gpus > 1:
        out["parallelism"] = (f"row-slab x{n_gpus} (NCCL halo + allgather), "
                              + ("weak scaling: 1024 x 1024 per GPU" if scaling == "weak" else "strong scaling of the global grid"))
        if scaling == "weak":
            out["global_grid"] = [c["nx"], c["nx"] * n_gpus]
    else:
        out["parallelism"] = "single"
    return out


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, device):
        self.device = device
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        load = [v for v in sm if mx and v > 0.3 * mx] or sm
        return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def _barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def _allreduce(vals, op, dev, ws):
    if ws == 1:
        return vals
    import torch
    import torch.distributed as dist
    t = torch.tensor(vals, dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=op)
    return [float(v) for v in t]


def measure(name, steps, warmup, cpu=True):
    """One configuration on this process's GPU (or its slab of it under torchrun)."""
    import torch
    from paper_2001_04886_b200 import Context, convection_diffusion, splitmix64_uniform
    from paper_2001_04886_b200.sstep import sgmres_solve, sgmres_solve_device, somin_solve, somin_solve_device

    c = CONFIGS[name]
    ws, rank, local = dist_env()
    dev = torch.device("cuda", local)
    scaling = "weak" if name == "C2" else "strong"
    ny = c["nx"] * ws if (ws > 1 and scaling == "weak") else None
    st = convection_diffusion(c["dim"], c["nx"], c["conv"], ny=ny, variable_k=c.get("vark", False))
    f_glob = splitmix64_uniform(SEED, st.n)
    kcell = None
    if c.get("vark"):
        from paper_2001_04886_b200.problems import lognormal_k
        kcell = lognormal_k(K_SEED, st.n)
    cfg = sstep_cfg(c, f_glob)
    if ws > 1:
        from paper_2001_04886_b200.dist import nccl_context, slab_of, slab_operator
        ctx = nccl_context(local)
        op, lo, hi = slab_operator(ctx, st, kcell=kcell)
        f_host = slab_of(f_glob, st, lo, hi)
    else:
        ctx = Context(local)
        op = ctx.stencil(st, kcell=kcell)
        f_host = f_glob
    del f_glob, kcell
    n = f_host.size
    stream = torch.cuda.Stream(dev)  # the library's kernels and the timing events share it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    f_dev = torch.from_numpy(f_host).to(dev)
    x_dev = torch.zeros(n, dtype=torch.float64, device=dev)
    dev_fn = sgmres_solve_device if c["method"] == "sgmres" else somin_solve_device
    host_fn = sgmres_solve if c["method"] == "sgmres" else somin_solve
    per = c["s"] if c["method"] == "sgmres" else 1  # inner iterations per s-step

    def solve_dev():
        x_dev.zero_()
        return dev_fn(op, f_dev.data_ptr(), x_dev.data_ptr(), cfg)

    for _ in range(warmup):
        rep = solve_dev()
    torch.cuda.synchronize()
    # ---- timed region (device-resident inputs; every vector is larger than L2)
    _barrier(ws)
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    iters, ok = 0, True
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            rep = solve_dev()
            iters += rep.iterations
            ok &= rep.converged if "fixed" not in c else rep.breakdown is None
        e1.record(stream)
        torch.cuda.synchronize()
    _barrier(ws)
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    sst = iters / per  # s-steps of the (global) solve
    ms_max, = _allreduce([ms], _max_op(), dev, ws)
    value = sst * (ws if scaling == "weak" else 1) / (ms_max / 1e3)
    # ---- e2e through the C ABI with pinned host buffers (H2D f, x0; D2H x) in the timed region
    x_host = torch.zeros(n, dtype=torch.float64, pin_memory=True).numpy()
    f_pin = torch.from_numpy(f_host).pin_memory().numpy()
    e_steps = max(1, steps if c["nx"] ** c["dim"] <= 2 ** 24 else 1)
    if warmup > 0:  # one untimed call: the host path's staging buffers exist before the clock starts
        x_host[:] = 0.0
        host_fn(op, f_pin, x_host, cfg)
    torch.cuda.synchronize()
    _barrier(ws)
    t0 = time.perf_counter()
    e_iters = 0
    for _ in range(e_steps):
        x_host[:] = 0.0
        r2 = host_fn(op, f_pin, x_host, cfg)
        e_iters += r2.iterations
    torch.cuda.synchronize()
    e_s, = _allreduce([time.perf_counter() - t0], _max_op(), dev, ws)
    e2e_value = (e_iters / per) * (ws if scaling == "weak" else 1) / e_s
    del x_host, f_pin
    # ---- per-kernel roofline (profiled pass of one solve: CUDA events around every launch, on
    #      the library's stream)
    ctx.reset_stats()
    ctx.set_profiling(True)
    solve_dev()
    torch.cuda.synchronize()
    stats = ctx.kernel_stats()
    ctx.set_profiling(False)
    peak, peak_src = peaks()
    top = max(stats.items(), key=lambda kv: kv[1]["ms"]) if stats else None
    total_ms = sum(v["ms"] for v in stats.values()) or 1.0
    roofline = None
    if top:
        kname, s_ = top
        ach = s_["bytes"] / (s_["ms"] / 1e3) / 1e9
        roofline = {"kernel": kname, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": None, "peak_source": peak_src,
                    "share_of_step": round(s_["ms"] / total_ms, 4), "launches_per_step": s_["launches"],
                    "alg_bytes_per_launch": s_["bytes"] / max(1, s_["launches"]),
                    "bytes_model": ("SURVEY 8(d): 4ks+4s+5 vectors per block step k < m, 2ms+s+6 at k = m"
                                    if kname == "arn_step" else "the kernel's distinct operand vectors read + written")}
        if ach > peak:
            # the measured peak is a 1:1 read+write copy; a read-dominated stream (this kernel reads
            # several vectors per vector written) moves more than that, and operands a launch re-reads
            # can come from the 126 MB L2 (compare "traffic", the DRAM bytes under ncu)
            roofline["note"] = ("above the copy-measured peak: read-dominated stream (HBM reads run faster than a "
                                "1:1 copy) and/or operands served from L2; see traffic")
        tr = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tr):
            try:
                t = json.load(open(tr)).get(name, {})
                roofline["traffic"] = t.get(kname) if isinstance(t, dict) else None
            except Exception:
                pass
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                   "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)} for k, v in stats.items()}
    eff = model_vecs_per_sstep(c) * 8.0 * st.n * value / 1e9
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws, "steps": steps, "warmup": warmup,
        "ms_per_step": round(ms_max / steps, 3), "higher_is_better": True, "scaling": scaling, "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic: seeded splitmix64 U[-1,1] RHS" + (", k=exp(N(0,1)) per cell (seeded Box-Muller)" if c.get("vark") else "")
                + ", h^2-scaled stencil generated on the fly",
        "config": config_json(name, c, ws, scaling),
        "effective_hbm_gbs": round(eff, 1), "effective_hbm_frac": round(eff / peak, 4),
        "roofline": roofline,
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": 16 * n, "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches, "s_steps_per_step": sst / steps, "kernels": kernels,
    }
    if c["method"] == "sgmres":
        out["cycles_per_step"] = rep.cycles
    if not ok:
        out["invalid"] = ("solve did not converge inside the timed region" if "fixed" not in c
                          else f"breakdown: {rep.breakdown}")
    if "fixed" in c and c["s"] == 8:
        out["numerics"] = ("fixed-step benchmark mode: the reference stops at its Gram pivot-ratio / LSQ rank "
                           "abort on this configuration; the iterates past that point are numerically meaningless")
    if rank == 0:
        out["clocks"] = clk.summary()
        if ws == 1 and cpu:
            out["cpu_baseline"] = cpu_baseline_sample(name)
    del op, ctx, f_dev, x_dev
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    return out


def _max_op():
    try:
        import torch.distributed as dist
        return dist.ReduceOp.MAX
    except Exception:
        return None


def _reference_lib(need_fixed=False):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    if not need_fixed and Oracle.available("reference"):
        return Oracle("reference"), "reference"
    return Oracle("port"), "port"


def _port():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    return Oracle("port")


def cpu_baseline_sample(name):
    """The reference CPU path on one host core on a bounded sample of the same workload."""
    from paper_2001_04886_b200 import convection_diffusion, splitmix64_uniform
    c = CONFIGS[name]
    fixed_mode = "fixed" in c and c["s"] == 8
    orc, kind = _reference_lib(need_fixed=fixed_mode)  # (the reference has no fixed-step mode)
    nx = c.get("cpu_nx", c["nx"])
    st = convection_diffusion(c["dim"], nx, c["conv"], variable_k=c.get("vark", False))
    port = _port()  # (input assembly only: the port's CSR builder and k generator)
    kcell = port.lognormal(K_SEED, st.n) if c.get("vark") else None
    a = port.stencil_csr(c["dim"], st.nx, st.ny, st.nz, st.coef, kcell=kcell, ch2=st.ch2)
    f = splitmix64_uniform(SEED, st.n)
    s = c["s"]
    if c["method"] == "sgmres":
        tol = 0.0 if "fixed" in c else c["rel_tol"] * float(np.linalg.norm(f))
        cycles = 1 if "fixed" in c else 2
        kw = dict(s=s, m=c["m"], tol=tol, max_iterations=cycles * s * c["m"])
        per = s
    else:
        kw = dict(s=s, k=c["k"], tol=0.0, max_iterations=2)
        per = 1
    if fixed_mode:
        orc.set_fixed_steps(True)
    try:
        t0 = time.perf_counter()
        r = orc.sstep(c["method"], a, f, None, **kw)
        dt = time.perf_counter() - t0
    finally:
        if fixed_mode:
            orc.set_fixed_steps(False)
    ssteps = r.iterations / per
    rate = ssteps / dt
    scale = st.n / float(c["nx"] ** c["dim"])  # time per s-step is linear in the unknowns
    sample = (f"{ssteps:.0f} s-steps of {c['method']}_solve (s={s}) on the {'x'.join([str(nx)] * c['dim'])} grid from x0=0, "
              f"{dt:.1f} s on 1 core")
    if scale != 1.0:
        sample += (f"; value scaled to the full {'x'.join([str(c['nx'])] * c['dim'])} grid by the unknown count "
                   f"(x{scale:.3g}: an s-step's work is linear in n)")
    if fixed_mode:
        sample += "; oracle port in its fixed-step mode (the reference aborts on this configuration)"
    return {"value": round(rate * scale, 6 if scale != 1.0 else 3), "unit": UNIT, "cores": 1, "kind": kind,
            "sample": sample}


def run_ours(args):
    import torch
    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    out = measure(args.config, args.steps, args.warmup)
    if ws == 1 and args.config == "C2" and not args.no_secondary:
        sec = {}
        for nm in SECONDARY:
            try:
                steps = 2 if nm in ("C4", "C5") else max(2, args.steps // 2)
                sec[nm] = measure(nm, steps, 1)
                for k in ("metric", "unit", "higher_is_better", "dtype", "vs_baseline", "n_gpus"):
                    sec[nm].pop(k, None)
            except Exception as e:  # report, never hide the headline
                sec[nm] = {"error": f"{type(e).__name__}: {e}"}
        out["secondary"] = sec
    if rank == 0:
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    from paper_2001_04886_b200 import convection_diffusion, splitmix64_uniform
    orc, kind = _reference_lib()
    c = CONFIGS["C2"]
    st = convection_diffusion(2, c["nx"], c["conv"])
    a = _port().stencil_csr(2, st.nx, st.ny, 1, st.coef)
    f = splitmix64_uniform(SEED, st.n)
    tol = c["rel_tol"] * float(np.linalg.norm(f))
    S, M = c["s"], c["m"]
    threads = max(1, min(os.cpu_count() or 1, 32))  # ~0.45 GB of vectors per concurrent solve
    try:
        import psutil
        threads = max(1, min(threads, int(psutil.virtual_memory().available / 1.0e9)))
    except Exception:
        pass

    def one_step():
        res = [0] * threads

        def work(i):
            r = orc.sstep("sgmres", a, f, None, s=S, m=M, tol=tol, max_iterations=S * M)
            res[i] = r.iterations

        th = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        t0 = time.perf_counter()
        for t in th:
            t.start()
        for t in th:
            t.join()
        return sum(res), time.perf_counter() - t0

    for _ in range(args.warmup):
        one_step()
    total_it, total_s = 0, 0.0
    for _ in range(args.steps):
        it, dt = one_step()
        total_it += it
        total_s += dt
    value = total_it / S / total_s
    out = {"metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": round(1e3 * total_s / args.steps, 1), "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic: seeded splitmix64 U[-1,1] RHS, h^2-scaled stencil (CSR)",
           "config": config_json("C2", c, 1, "weak"),
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                            "sample": f"per step: one restart cycle (10 s-steps) of sgmres_solve on each of "
                                      f"{threads} host threads in parallel (independent solves)"},
           "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C2", choices=sorted(CONFIGS))
    ap.add_argument("--no-secondary", action="store_true")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
