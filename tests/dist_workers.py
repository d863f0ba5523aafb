"""Worker functions for the multi-process tests (spawned; must be importable)."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

P = C.POINTER
dbl = C.c_double


def _init(rank, world, port):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def _dp(a):
    return a.ctypes.data_as(P(dbl))


def cpu_exchange_worker(rank, world, port, q):
    """The host-side comm of the slab decomposition, on CPU: allgather in rank order and a
    halo exchange whose ghost rows make a slab-local stencil apply equal the global one."""
    dist = _init(rank, world, port)
    try:
        from oracle import Oracle
        from paper_2001_04886_b200.dist import HostExchange, slab_of, slab_range
        from paper_2001_04886_b200.problems import convection_diffusion, splitmix64_uniform
        ex = HostExchange()
        send = np.arange(5, dtype=np.float64) + 10.0 * rank
        recv = np.zeros(5 * world)
        assert ex._ag(None, _dp(send), _dp(recv), 5) == 0
        ok_ag = all(np.array_equal(recv[r * 5:(r + 1) * 5], np.arange(5) + 10.0 * r) for r in range(world))
        # slab apply with width-1 halos (oracle arithmetic) == rows of the global apply
        st = convection_diffusion(2, 12, 10.0, ny=16)
        lo, hi = slab_range(st.ny, world, rank)
        v = splitmix64_uniform(5, st.n)
        vl = slab_of(v, st, lo, hi)
        nx = st.nx
        lo_recv, hi_recv = np.zeros(nx), np.zeros(nx)
        has_lo, has_hi = rank > 0, rank + 1 < world
        rc = ex._halo(None, _dp(vl[:nx]) if has_lo else None, _dp(lo_recv) if has_lo else None, nx if has_lo else 0,
                      _dp(vl[-nx:]) if has_hi else None, _dp(hi_recv) if has_hi else None, nx if has_hi else 0)
        assert rc == 0
        ext = np.concatenate([lo_recv if has_lo else [], vl, hi_recv if has_hi else []])
        rows = hi - lo + has_lo + has_hi
        orc = Oracle("port")
        # apply the stencil to the extended slab, then keep the owned rows; boundary rows of
        # the extended slab are wrong only where a neighbour row is missing, and those are
        # exactly the ghost rows we drop
        y_ext = orc.stencil_apply(2, nx, rows, 1, st.coef, ext)
        y_loc = y_ext[(nx if has_lo else 0):(nx if has_lo else 0) + (hi - lo) * nx]
        y_glob = slab_of(orc.stencil_apply(2, nx, st.ny, 1, st.coef, v), st, lo, hi)
        q.put((rank, ok_ag, bool(np.array_equal(y_loc, y_glob)), lo, hi))
    finally:
        dist.destroy_process_group()


def gpu_slab_worker(rank, world, port, case, q):
    """One rank of a slab-decomposed solve on the shared GPU (host-staged exchanges)."""
    dist = _init(rank, world, port)
    try:
        from paper_2001_04886_b200 import SStepConfig, sgmres_solve, somin_solve
        from paper_2001_04886_b200.dist import callback_context, slab_of, slab_operator
        st, f, kcell, method, cfg = case
        ctx = callback_context(0)
        op, lo, hi = slab_operator(ctx, st, kcell)
        fl = slab_of(f, st, lo, hi)
        xl = np.zeros_like(fl)
        fn = somin_solve if method == "somin" else sgmres_solve
        rep = fn(op, fl, xl, SStepConfig(**cfg))
        q.put((rank, lo, hi, xl, rep.residual_history, rep.iterations, rep.cycles, rep.op_history, rep.breakdown,
               rep.converged, ctx._exchange.calls))
    finally:
        dist.destroy_process_group()


def nccl_single_worker(rank, world, port, case, q):
    """NCCL backend with one rank (exercises the dlopen'd NCCL path on one GPU)."""
    dist = _init(rank, world, port)
    try:
        from paper_2001_04886_b200 import SStepConfig, somin_solve
        from paper_2001_04886_b200.dist import nccl_context, slab_operator, world_of
        st, f, method, cfg = case
        ctx = nccl_context(0)
        op, lo, hi = slab_operator(ctx, st)
        x = np.zeros(st.n)
        rep = somin_solve(op, f, x, SStepConfig(**cfg))
        q.put((world_of(ctx), rep.residual_history, x))
    finally:
        dist.destroy_process_group()
