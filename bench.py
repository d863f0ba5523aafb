#!/usr/bin/env python
"""bench.py -- headline benchmark (BASELINE.json metric) for the B200 s-step solvers.

Workload (BASELINE configs[1], the metric's single-GPU configuration):
    s-step GMRES, s=4, m=10, 2D 5-point convection-diffusion (c=50, h^2-scaled), 1024x1024,
    f ~ U[-1,1] (splitmix64, seed 20010486), x0 = 0, tol = 1e-8 ||f||.
One step = one full solve to tolerance (about 100 restart cycles / 1000 s-steps).
metric: s-step iterations per second (one s-step = one block iteration of s inner steps),
with the effective HBM GB/s of the SURVEY 8(d) algorithmic byte model beside it.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Multi-GPU (torchrun, N>1): weak scaling by row-slab decomposition -- every GPU owns a
1024 x 1024 slab of a 1024 x (1024 N) grid, ghost rows and dot sums exchanged with NCCL
(halo send/recv before each matrix-powers sweep, allgather at every reduction point);
value = N x (global s-steps) / max rank time, i.e. slab s-steps per second summed over GPUs.
--impl reference times the reference's own CPU implementation (oracle/_ref, the unmodified
reference headers; the C restatement oracle/liboracle.so if _ref is absent) on the same
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

S, M, NX, CONV, REL_TOL, SEED = 4, 10, 1024, 50.0, 1e-8, 20010486
METRIC = "s-step iterations/sec and effective HBM GB/s (fraction of peak) at 1/2/4/8 B200"
UNIT = "s-steps/s"
WORKLOAD = "C2: s-step GMRES s=4 m=10, 2D 5-point conv-diff c=50 (h^2-scaled), 1024x1024, tol 1e-8 rel, x0=0"


def peaks():
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def sgmres_bytes_per_cycle(s, m, n):
    """SURVEY 8(d) algorithmic bytes of one s-GMRES(m) cycle (block-CGS-equivalent passes)."""
    return (2 * s * m * (m - 1) + (m - 1) * (4 * s + 5) + 3 * m * s + 3 * s + 13) * 8.0 * n


def config(n_gpus):
    return {"workload": WORKLOAD, "method": "sgmres", "s": S, "m": M, "grid": [NX, NX], "n": NX * NX,
            "conv": CONV, "rel_tol": REL_TOL, "rhs_seed": SEED,
            "l2": "working set (m+2)s+4 = 52 vectors x 8 MiB = 416 MiB > 126 MB L2; no flush",
            "parallelism": f"row-slab x{n_gpus} (NCCL halo + allgather), weak scaling" if n_gpus > 1 else "single",
            "global_grid": [NX, NX * n_gpus]}


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


def run_ours(args):
    import torch
    from paper_2001_04886_b200 import Context, SStepConfig, convection_diffusion, splitmix64_uniform
    from paper_2001_04886_b200.sstep import sgmres_solve, sgmres_solve_device

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # weak scaling: every GPU owns a 1024 x 1024 row slab of a 1024 x (1024 N) grid (same
    # stencil coefficients as C2); N = 1 is exactly BASELINE configs[1]
    st = convection_diffusion(2, NX, CONV, ny=NX * ws)
    f_glob = splitmix64_uniform(SEED, st.n)
    tol = REL_TOL * float(np.linalg.norm(f_glob))
    cfg = SStepConfig(s=S, m=M, tol=tol)
    if ws > 1:
        from paper_2001_04886_b200.dist import nccl_context, slab_of, slab_operator
        ctx = nccl_context(local)
        op, lo, hi = slab_operator(ctx, st)
        f_host = slab_of(f_glob, st, lo, hi)
    else:
        ctx = Context(local)
        op = ctx.stencil(st)
        f_host = f_glob
    n = f_host.size
    stream = torch.cuda.Stream(dev)  # the library's kernels and the timing events share it
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)
    f_dev = torch.from_numpy(f_host).to(dev)
    x_dev = torch.zeros(n, dtype=torch.float64, device=dev)

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    def solve_dev():
        x_dev.zero_()
        return sgmres_solve_device(op, f_dev.data_ptr(), x_dev.data_ptr(), cfg)

    for _ in range(args.warmup):
        rep = solve_dev()
    torch.cuda.synchronize()
    # ---- timed region (device-resident inputs)
    barrier()
    torch.cuda.synchronize()
    l0 = ctx.launch_count()
    iters = 0
    converged = True
    with Clocks(local) as clk:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            rep = solve_dev()
            iters += rep.iterations
            converged &= rep.converged
        e1.record(stream)
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = ctx.launch_count() - l0
    sst = iters / S  # s-steps (block iterations)
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([ms, sst], dtype=torch.float64, device=dev)
        tmax = t.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        tsum = t.clone()
        dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
        ms, sst_total = float(tmax[0]), float(tsum[1])
    else:
        sst_total = sst
    value = sst_total / (ms / 1e3)
    cycles_per_solve = rep.cycles
    # ---- e2e through the C ABI with host buffers (H2D f, x0; D2H x) inside the timed region
    # pinned host buffers (page-locked, so the copies run at the DMA rate, as a serving caller's would)
    x_host = torch.zeros(n, dtype=torch.float64, pin_memory=True).numpy()
    f_pin = torch.from_numpy(f_host).pin_memory().numpy()
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    e_iters = 0
    for _ in range(args.steps):
        x_host[:] = 0.0
        r2 = sgmres_solve(op, f_pin, x_host, cfg)
        e_iters += r2.iterations
    torch.cuda.synchronize()
    e_s = time.perf_counter() - t0
    e2e_value = (e_iters / S) / e_s
    if ws > 1:
        import torch.distributed as dist
        t = torch.tensor([e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_value = (e_iters / S) * ws / float(t[0])
    # ---- per-kernel roofline (profiled pass of one solve: CUDA events around every launch)
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
        name, s_ = top
        ach = s_["bytes"] / (s_["ms"] / 1e3) / 1e9
        roofline = {"kernel": name, "bound": "hbm", "achieved": round(ach, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(ach / peak, 4), "traffic": None, "peak_source": peak_src,
                    "share_of_step": round(s_["ms"] / total_ms, 4), "launches_per_solve": s_["launches"],
                    "alg_bytes_per_launch": s_["bytes"] / max(1, s_["launches"])}
        tr = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tr):
            try:
                roofline["traffic"] = json.load(open(tr)).get(name)
            except Exception:
                pass
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                   "gbs": round(v["bytes"] / max(v["ms"], 1e-9) / 1e6, 1)} for k, v in stats.items()}
    eff = sgmres_bytes_per_cycle(S, M, n) / M * value / 1e9
    out = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: seeded splitmix64 U[-1,1] RHS, h^2-scaled stencil generated on the fly",
        "config": config(ws),
        "effective_hbm_gbs": round(eff, 1), "effective_hbm_frac": round(eff / peak, 4),
        "roofline": roofline,
        "e2e": {"value": round(e2e_value, 2), "unit": UNIT, "h2d_bytes_per_step": 16 * n,
                "d2h_bytes_per_step": 8 * n},
        "gpu_launches": launches, "converged": converged, "cycles_per_solve": cycles_per_solve,
        "s_steps_per_solve": rep.iterations / S, "kernels": kernels,
    }
    if not converged:  # a step is a solve to tolerance: an unconverged solve is not a valid step
        out["invalid"] = "solve did not converge inside the timed region"
    if rank == 0:
        clocks = clk.summary()
        out["clocks"] = clocks
        if ws == 1:
            out["cpu_baseline"] = cpu_baseline_sample()
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


def _reference_lib():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    if Oracle.available("reference"):
        return Oracle("reference"), "reference"
    return Oracle("port"), "port"


def _c2_problem(orc):
    from paper_2001_04886_b200 import convection_diffusion, splitmix64_uniform
    st = convection_diffusion(2, NX, CONV)
    a = orc_port_csr(st)
    f = splitmix64_uniform(SEED, st.n)
    return a, f, REL_TOL * float(np.linalg.norm(f))


def orc_port_csr(st):
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle
    return Oracle("port").stencil_csr(2, st.nx, st.ny, 1, st.coef)


def cpu_baseline_sample(cycles=2):
    """Reference CPU path on one host core: `cycles` restart cycles of the same workload."""
    orc, kind = _reference_lib()
    a, f, tol = _c2_problem(orc)
    t0 = time.perf_counter()
    r = orc.sstep("sgmres", a, f, None, s=S, m=M, tol=tol, max_iterations=cycles * S * M)
    dt = time.perf_counter() - t0
    return {"value": round(r.iterations / S / dt, 3), "unit": UNIT, "cores": 1, "kind": kind,
            "sample": f"{r.iterations // S} s-steps ({r.cycles} restart cycles) of the C2 workload, "
                      f"sgmres_solve from x0=0, {dt:.1f} s on 1 core"}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    orc, kind = _reference_lib()
    a, f, tol = _c2_problem(orc)
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
           "data": "synthetic: seeded splitmix64 U[-1,1] RHS, h^2-scaled stencil (CSR)", "config": config(1),
           "impl": "reference",
           "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": threads, "kind": kind,
                            "sample": f"per step: one restart cycle (10 s-steps) of sgmres_solve on each of "
                                      f"{threads} host threads in parallel"},
           "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
