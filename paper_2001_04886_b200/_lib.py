"""ctypes binding of libskrylov_b200.so (the C ABI in include/skrylov_b200.h).

The shared library is built in-tree (``make -C paper_2001_04886_b200/csrc`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing or has no
GPU to run on, calls fail loudly.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SKC_LIB") or os.path.join(HERE, "libskrylov_b200.so")  # (SKC_LIB: A/B builds)

u64 = C.c_uint64
i32 = C.c_int32
dbl = C.c_double
P = C.POINTER

SKC_OK, SKC_EINVAL, SKC_EBREAKDOWN, SKC_ELOGIC, SKC_ECUDA, SKC_ENCCL, SKC_ENOMEM = range(7)


class BreakdownError(RuntimeError):
    """skrylov::breakdown_error (kernels.hpp:36-39) escaping a call."""


class LogicError(RuntimeError):
    """std::logic_error raised by debug_checks (sstep.hpp:231)."""


class CudaError(RuntimeError):
    """CUDA / NCCL runtime failure."""


class OpCounter(C.Structure):
    _fields_ = [("dotprods", u64), ("matvecs", u64), ("vec_updates", u64), ("stored_vectors", u64),
                ("termination_dots", u64)]

    def as_tuple(self):
        return (self.dotprods, self.matvecs, self.vec_updates, self.stored_vectors, self.termination_dots)


class SStepConfigC(C.Structure):
    _fields_ = [("s", u64), ("k", u64), ("m", u64), ("tol", dbl), ("max_iterations", u64),
                ("precondition", i32), ("unbounded_window", i32), ("debug_checks", i32),
                ("divergence_factor", dbl), ("fixed_steps", i32)]


class SolverConfigC(C.Structure):
    _fields_ = [("method", i32), ("k", u64), ("m", u64), ("tol", dbl), ("max_iterations", u64),
                ("precondition", i32), ("debug_checks", i32), ("divergence_factor", dbl)]


class StencilDescC(C.Structure):
    _fields_ = [("dim", i32), ("kind", i32), ("nx", u64), ("ny", u64), ("nz", u64), ("coef", dbl * 7),
                ("ch2", dbl)]


class ReportSummaryC(C.Structure):
    _fields_ = [("converged", i32), ("iterations", u64), ("cycles", u64), ("final_residual", dbl),
                ("op_counts", OpCounter), ("steady_iteration", u64), ("has_breakdown", i32),
                ("fallback_cycles", u64), ("n_history", u64), ("n_op_history", u64), ("n_notes", u64),
                ("n_block_rho", u64)]


EXPORTS = [
    "skc_last_error", "skc_version", "skc_device_count", "skc_ctx_create", "skc_ctx_destroy", "skc_ctx_set_stream",
    "skc_ctx_set_profiling", "skc_ctx_kernel_stats", "skc_ctx_kernel_names", "skc_ctx_reset_stats",
    "skc_ctx_launch_count", "skc_op_create_stencil", "skc_op_create_csr", "skc_op_destroy", "skc_op_size",
    "skc_op_kind", "skc_op_apply", "skc_krylov_block", "skc_report_create", "skc_report_destroy",
    "skc_report_get_summary", "skc_report_get_history", "skc_report_get_op_history", "skc_report_get_block_rho",
    "skc_report_get_breakdown", "skc_report_get_note", "skc_somin_solve", "skc_sgmres_solve", "skc_smr_solve",
    "skc_gmres_solve", "skc_smr_step", "skc_somin_solve_device", "skc_sgmres_solve_device", "skc_sarnoldi",
    "skc_gram_solve", "skc_cholesky_upper", "skc_hessenberg_lsq",
    "skc_nccl_unique_id", "skc_ctx_create_nccl", "skc_ctx_create_callback", "skc_ctx_world", "skc_ctx_set_gpu_independent",
    "skc_op_create_stencil_slab", "skc_slab_range",
    "skc_op_create_ilu0", "skc_ilu0_solve", "skc_ilu0_solve_device", "skc_ilu0_factor", "skc_fill_lognormal", "skc_discretize",
]

ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, P(dbl), P(dbl), u64)
HALO_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, P(dbl), P(dbl), u64, P(dbl), P(dbl), u64)

_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is not built; run `make -C paper_2001_04886_b200/csrc` "
                          "(or __graft_entry__.build()). There is no CPU fallback.")
    L = C.CDLL(LIB_PATH)
    vp = C.c_void_p
    L.skc_last_error.restype = C.c_char_p
    L.skc_version.restype = C.c_char_p
    sig = {
        "skc_device_count": [P(C.c_int)],
        "skc_ctx_create": [C.c_int, P(vp)],
        "skc_ctx_destroy": [vp],
        "skc_ctx_set_stream": [vp, C.c_size_t],
        "skc_ctx_set_profiling": [vp, C.c_int],
        "skc_ctx_kernel_stats": [vp, C.c_char_p, P(u64), P(dbl), P(dbl)],
        "skc_ctx_kernel_names": [vp, C.c_char_p, C.c_size_t],
        "skc_ctx_reset_stats": [vp],
        "skc_ctx_launch_count": [vp, P(u64)],
        "skc_op_create_stencil": [vp, P(StencilDescC), P(dbl), P(vp)],
        "skc_op_create_csr": [vp, u64, P(u64), P(u64), P(dbl), P(vp)],
        "skc_op_destroy": [vp],
        "skc_op_size": [vp, P(u64)],
        "skc_op_kind": [vp, P(C.c_int)],
        "skc_op_apply": [vp, vp, P(dbl), P(dbl)],
        "skc_krylov_block": [vp, vp, P(dbl), u64, P(dbl)],
        "skc_report_create": [P(vp)],
        "skc_report_destroy": [vp],
        "skc_report_get_summary": [vp, P(ReportSummaryC)],
        "skc_somin_solve": [vp, vp, P(dbl), P(dbl), P(SStepConfigC), vp],
        "skc_sgmres_solve": [vp, vp, P(dbl), P(dbl), P(SStepConfigC), vp],
        "skc_smr_solve": [vp, vp, P(dbl), P(dbl), P(SStepConfigC), vp],
        "skc_gmres_solve": [vp, vp, P(dbl), P(dbl), P(SolverConfigC), vp],
        "skc_smr_step": [vp, vp, P(dbl), P(dbl), u64, P(dbl), P(OpCounter)],
        "skc_somin_solve_device": [vp, vp, vp, vp, P(SStepConfigC), vp],
        "skc_sgmres_solve_device": [vp, vp, vp, vp, P(SStepConfigC), vp],
        "skc_sarnoldi": [vp, vp, P(dbl), u64, u64, P(dbl), P(dbl), P(dbl), P(dbl), P(dbl), P(OpCounter)],
        "skc_gram_solve": [u64, P(dbl), u64, P(dbl), P(dbl), P(i32), P(dbl)],
        "skc_cholesky_upper": [u64, P(dbl), P(dbl)],
        "skc_hessenberg_lsq": [u64, u64, P(dbl), dbl, P(dbl), P(dbl)],
        "skc_nccl_unique_id": [vp],
        "skc_ctx_create_nccl": [C.c_int, C.c_int, C.c_int, vp, P(vp)],
        "skc_ctx_create_callback": [C.c_int, C.c_int, C.c_int, ALLGATHER_FN, HALO_FN, vp, P(vp)],
        "skc_ctx_world": [vp, P(C.c_int), P(C.c_int)],
        "skc_ctx_set_gpu_independent": [vp, C.c_int],
        "skc_op_create_stencil_slab": [vp, P(StencilDescC), P(dbl), P(u64), P(u64), P(vp)],
        "skc_slab_range": [u64, C.c_int, C.c_int, P(u64), P(u64)],
        "skc_op_create_ilu0": [vp, u64, P(u64), P(u64), P(dbl), P(vp)],
        "skc_ilu0_solve": [vp, vp, P(dbl), P(dbl)],
        "skc_ilu0_solve_device": [vp, vp, vp, vp],
        "skc_ilu0_factor": [C.c_void_p, u64, P(u64), P(u64), P(dbl), P(dbl)],
        "skc_fill_lognormal": [u64, u64, P(dbl)],
        "skc_discretize": [u64, dbl, dbl, P(u64), P(u64), P(dbl), P(dbl), P(dbl), P(dbl)],
    }
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = C.c_int
    for name in ("skc_report_get_history", "skc_report_get_block_rho"):
        getattr(L, name).argtypes = [vp, P(dbl), u64]
        getattr(L, name).restype = u64
    L.skc_report_get_op_history.argtypes = [vp, P(OpCounter), u64]
    L.skc_report_get_op_history.restype = u64
    L.skc_report_get_breakdown.argtypes = [vp, C.c_char_p, u64]
    L.skc_report_get_breakdown.restype = u64
    L.skc_report_get_note.argtypes = [vp, u64, C.c_char_p, u64]
    L.skc_report_get_note.restype = u64
    _lib = L
    return L


def check(status: int):
    if status == SKC_OK:
        return
    msg = lib().skc_last_error().decode()
    if status == SKC_EINVAL:
        raise ValueError(msg)
    if status == SKC_EBREAKDOWN:
        raise BreakdownError(msg)
    if status == SKC_ELOGIC:
        raise LogicError(msg)
    if status == SKC_ENOMEM:
        raise MemoryError(msg)
    raise CudaError(msg)
