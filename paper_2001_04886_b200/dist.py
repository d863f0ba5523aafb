"""Multi-GPU row-slab decomposition front end (one process per GPU, torch.distributed for
the plumbing).

* ``nccl_context(device)`` -- the production path: rank 0 draws an NCCL unique id through the
  library, torch.distributed broadcasts its 128 bytes, every rank builds a context whose
  allgathers and halo exchanges are NCCL operations on the library's stream.
* ``callback_context(device)`` -- the same exchanges staged through host memory and carried
  by torch.distributed (gloo works): several processes may share one GPU, which is how the
  multi-rank data path is tested on a single B200 and how the host side is tested on CPU.

``slab_operator(ctx, stencil, kcell)`` returns the rank's operator and its global row range;
solves take the rank's slab of f and x (rows lo..hi-1 of the slowest dimension).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .problems import Stencil
from .sstep import Context, DeviceOperator

P = C.POINTER
dbl = C.c_double
u64 = C.c_uint64


def slab_range(rows: int, world: int, rank: int):
    """The library's partition rule (skc_slab_range): rows [R*r/P, R*(r+1)/P)."""
    lo, hi = u64(), u64()
    check(lib().skc_slab_range(rows, world, rank, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def slab_rows(st: Stencil) -> int:
    return st.ny if st.dim == 2 else st.nz


def slab_of(vec, st: Stencil, lo: int, hi: int):
    """Rows [lo, hi) of the slowest dimension of a global natural-order vector."""
    rowlen = st.nx if st.dim == 2 else st.nx * st.ny
    return np.ascontiguousarray(np.asarray(vec)[lo * rowlen:hi * rowlen])


class HostExchange:
    """allgather / halo callbacks over torch.distributed (host tensors)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self._ag = _lib.ALLGATHER_FN(self._allgather)
        self._halo = _lib.HALO_FN(self._halo_cb)
        self.calls = 0

    def _allgather(self, user, send, recv, n):
        import torch
        try:
            s = torch.from_numpy(np.ctypeslib.as_array(send, shape=(n,)).copy())
            out = [torch.empty(n, dtype=torch.float64) for _ in range(self.world)]
            self.dist.all_gather(out, s, group=self.group)
            r = np.ctypeslib.as_array(recv, shape=(n * self.world,))
            for i, t in enumerate(out):
                r[i * n:(i + 1) * n] = t.numpy()
            self.calls += 1
            return 0
        except Exception:  # reported to the caller as SKC_ENCCL
            return 1

    def _halo_cb(self, user, lo_send, lo_recv, n_lo, hi_send, hi_recv, n_hi):
        import torch
        try:
            reqs, bufs = [], []
            if n_lo:
                s = torch.from_numpy(np.ctypeslib.as_array(lo_send, shape=(n_lo,)).copy())
                r = torch.empty(n_lo, dtype=torch.float64)
                reqs += [self.dist.isend(s, self.rank - 1, group=self.group),
                         self.dist.irecv(r, self.rank - 1, group=self.group)]
                bufs.append((r, lo_recv, n_lo))
            if n_hi:
                s = torch.from_numpy(np.ctypeslib.as_array(hi_send, shape=(n_hi,)).copy())
                r = torch.empty(n_hi, dtype=torch.float64)
                reqs += [self.dist.isend(s, self.rank + 1, group=self.group),
                         self.dist.irecv(r, self.rank + 1, group=self.group)]
                bufs.append((r, hi_recv, n_hi))
            for q in reqs:
                q.wait()
            for r, ptr, n in bufs:
                np.ctypeslib.as_array(ptr, shape=(n,))[:] = r.numpy()
            self.calls += 1
            return 0
        except Exception:
            return 1


def callback_context(device: int = 0, group=None) -> Context:
    ex = HostExchange(group)
    ctx = Context.__new__(Context)
    ctx.h = C.c_void_p()
    check(lib().skc_ctx_create_callback(device, ex.rank, ex.world, ex._ag, ex._halo, None, C.byref(ctx.h)))
    ctx.device = device
    ctx._exchange = ex  # keeps the ctypes callbacks alive
    return ctx


def nccl_context(device: int, group=None) -> Context:
    """NCCL-backed context; torch.distributed must be initialized (any backend)."""
    import torch
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = (C.c_uint8 * 128)()
    if rank == 0:
        check(lib().skc_nccl_unique_id(uid))
    backend = dist.get_backend(group)
    dev = torch.device("cuda", device) if backend == "nccl" else torch.device("cpu")
    t = torch.tensor(list(bytes(uid)), dtype=torch.uint8, device=dev)
    dist.broadcast(t, 0, group=group)
    raw = bytes(t.cpu().tolist())
    C.memmove(uid, raw, 128)
    ctx = Context.__new__(Context)
    ctx.h = C.c_void_p()
    check(lib().skc_ctx_create_nccl(device, rank, world, uid, C.byref(ctx.h)))
    ctx.device = device
    return ctx


def world_of(ctx: Context):
    r, w = C.c_int(), C.c_int()
    check(lib().skc_ctx_world(ctx.h, C.byref(r), C.byref(w)))
    return r.value, w.value


def slab_operator(ctx: Context, st: Stencil, kcell=None):
    """(operator, lo, hi): the rank's slab of the global stencil."""
    d = _lib.StencilDescC(st.dim, 1 if st.variable_k else 0, st.nx, st.ny, st.nz if st.dim == 3 else 1,
                          (dbl * 7)(*st.coef), st.ch2)
    kp = None
    if st.variable_k:
        if kcell is None:
            raise ValueError("variable-k stencil needs kcell")
        kcell = np.ascontiguousarray(kcell, dtype=np.float64)
        kp = kcell.ctypes.data_as(P(dbl))
    h = C.c_void_p()
    lo, hi = u64(), u64()
    check(lib().skc_op_create_stencil_slab(ctx.h, C.byref(d), kp, C.byref(lo), C.byref(hi), C.byref(h)))
    rowlen = st.nx if st.dim == 2 else st.nx * st.ny
    return DeviceOperator(ctx, h, (hi.value - lo.value) * rowlen), lo.value, hi.value
