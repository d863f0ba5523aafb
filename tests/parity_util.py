"""GPU-vs-oracle comparison helpers shared by the GPU parity tests, smoke and the
parity report script (tools/parity_report.py)."""
from __future__ import annotations

import numpy as np

from golden_util import case, matrix


def rel_hist(h1, h2, upto=51, floor=1e-9):
    """max relative difference over the first `upto` entries, skipping entries below
    floor * h[0] in both histories (the reference KATs' convention, test_sstep.cpp:214,362)."""
    k = min(len(h1), len(h2), upto)
    a, b = np.asarray(h1[:k], dtype=float), np.asarray(h2[:k], dtype=float)
    if k and floor:
        keep = np.maximum(np.abs(a), np.abs(b)) >= floor * max(abs(a[0]), abs(b[0]))
        a, b = a[keep], b[keep]
    if a.size == 0:
        return 0.0
    s = np.maximum(np.abs(a), np.abs(b))
    d = np.where(s == 0, 0.0, np.abs(a - b) / np.where(s == 0, 1.0, s))
    return float(d.max())


def rel_vec(x, y):
    ny = np.linalg.norm(y)
    return float(np.linalg.norm(x - y) / ny) if ny > 0 else float(np.linalg.norm(x - y))


def gpu_operator(ctx, meta, arr, prefer_stencil=True):
    """The GPU operator for a golden case: the stencil descriptor when the case is a
    generated stencil (on-the-fly coefficients), else the CSR arrays (pattern-detected)."""
    from paper_2001_04886_b200.problems import Stencil
    st = meta.get("stencil")
    if st is not None and prefer_stencil:
        s = Stencil(st["dim"], st["nx"], st["ny"], st["nz"], tuple(st["coef"]), st["ch2"], st["variable_k"])
        return ctx.stencil(s, kcell=arr.get("kcell"))
    return ctx.csr(arr["offs"], arr["cols"], arr["vals"])


def run_gpu_case(ctx, name, prefer_stencil=True):
    from paper_2001_04886_b200 import SolverConfig, SStepConfig, gmres_solve, sgmres_solve, smr_solve, somin_solve
    meta, arr = case(name)
    op = gpu_operator(ctx, meta, arr, prefer_stencil)
    x = np.array(arr["x0"], dtype=np.float64, copy=True)
    cfg = dict(meta["cfg"])
    if meta["kind"] == "sstep":
        fn = {"somin": somin_solve, "sgmres": sgmres_solve, "smr": smr_solve}[meta["method"]]
        rep = fn(op, arr["f"], x, SStepConfig(**cfg))
    else:
        assert meta["method"] == "gmres"
        rep = gmres_solve(op, arr["f"], x, SolverConfig(**cfg))
    return meta, arr, rep, x, op


def summarize(meta, arr, rep, x):
    ref_hist = arr["history"]
    ref_oh = [tuple(int(v) for v in row) for row in arr["op_history"]]
    return dict(
        iters=(rep.iterations, meta["iterations"]), cycles=(rep.cycles, meta["cycles"]),
        converged=(rep.converged, meta["converged"]), hist50=rel_hist(rep.residual_history, ref_hist),
        hist_all=rel_hist(rep.residual_history, ref_hist, 10 ** 9), x=rel_vec(x, arr["x"]),
        op_history_equal=rep.op_history == ref_oh, op_counts_equal=tuple(rep.op_counts) == tuple(int(v) for v in arr["op_counts"]),
        breakdown=(rep.breakdown, meta["breakdown"]), notes_equal=rep.notes == meta["notes"],
        fallback=(rep.fallback_cycles, meta["fallback_cycles"]),
    )
