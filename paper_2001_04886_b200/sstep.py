"""Reference-shaped Python API over the B200 library.

Mirrors the reference's solver API (proj/include/skrylov/sstep.hpp, solvers.hpp,
report.hpp) name for name so parity tests read like the reference's own tests:

    op = Context().stencil(convection_diffusion(2, 128, 10.0))    # or Context().csr(...)
    x = np.zeros(op.n)
    rep = somin_solve(op, f, x, SStepConfig(s=4, k=2, tol=1e-8))  # x updated in place

Errors follow the reference: ValueError for require() (std::invalid_argument),
BreakdownError for an escaping breakdown_error, LogicError for debug-check failures;
numerical breakdown inside the solvers is reported in ``SolveReport.breakdown``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace

import numpy as np

from . import _lib
from ._lib import BreakdownError, CudaError, LogicError, OpCounter, check, lib  # noqa: F401
from .problems import Stencil

P = C.POINTER
dbl = C.c_double
u64 = C.c_uint64


@dataclass
class SStepConfig:
    """sstep.hpp:48-58 (same defaults)."""
    s: int = 2
    k: int = 2
    m: int = 5
    tol: float = 1e-6
    max_iterations: int = 100000
    precondition: bool = False
    unbounded_window: bool = False
    debug_checks: bool = False
    divergence_factor: float = 10.0
    # not in the reference: fixed-step benchmark mode (bypasses only the Gram pivot-ratio and
    # LSQ rank aborts; results past the reference's stop are meaningless, see skrylov_b200.h)
    fixed_steps: bool = False

    def c(self):
        return _lib.SStepConfigC(self.s, self.k, self.m, self.tol, self.max_iterations, int(self.precondition),
                                 int(self.unbounded_window), int(self.debug_checks), self.divergence_factor,
                                 int(self.fixed_steps))


@dataclass
class SolverConfig:
    """solvers.hpp:45-54; only method="gmres" runs on the GPU (s=1 path and fallback)."""
    method: str = "gmres"
    k: int = 4
    m: int = 10
    tol: float = 1e-6
    max_iterations: int = 100000
    precondition: bool = False
    debug_checks: bool = False
    divergence_factor: float = 10.0

    def c(self):
        meth = {"mr": 0, "omin": 1, "gcr": 2, "gmres": 3}[self.method]
        return _lib.SolverConfigC(meth, self.k, self.m, self.tol, self.max_iterations, int(self.precondition),
                                  int(self.debug_checks), self.divergence_factor)


@dataclass
class SolveReport:
    """report.hpp:53-75, plus block_rho (per-block LSQ residuals of s-GMRES)."""
    converged: bool = False
    iterations: int = 0
    cycles: int = 0
    residual_history: list = field(default_factory=list)
    final_residual: float = 0.0
    op_counts: tuple = (0, 0, 0, 0, 0)
    op_history: list = field(default_factory=list)
    steady_iteration: int = 0
    breakdown: str | None = None
    fallback_cycles: int = 0
    notes: list = field(default_factory=list)
    block_rho: list = field(default_factory=list)
    audit: object = None  # accounting.AuditReport when solve_linear ran the driver's audit


class _Report:
    def __init__(self):
        self.h = C.c_void_p()
        check(lib().skc_report_create(C.byref(self.h)))

    def __del__(self):
        if getattr(self, "h", None) and _lib._lib is not None:
            _lib._lib.skc_report_destroy(self.h)

    def collect(self) -> SolveReport:
        L = lib()
        s = _lib.ReportSummaryC()
        check(L.skc_report_get_summary(self.h, C.byref(s)))
        hist = np.zeros(s.n_history)
        L.skc_report_get_history(self.h, hist.ctypes.data_as(P(dbl)), s.n_history)
        oh = (_lib.OpCounter * max(1, s.n_op_history))()
        L.skc_report_get_op_history(self.h, oh, s.n_op_history)
        br = np.zeros(s.n_block_rho)
        L.skc_report_get_block_rho(self.h, br.ctypes.data_as(P(dbl)), s.n_block_rho)
        breakdown = None
        if s.has_breakdown:
            n = L.skc_report_get_breakdown(self.h, None, 0)
            buf = C.create_string_buffer(n + 1)
            L.skc_report_get_breakdown(self.h, buf, n + 1)
            breakdown = buf.value.decode()
        notes = []
        for i in range(s.n_notes):
            n = L.skc_report_get_note(self.h, i, None, 0)
            buf = C.create_string_buffer(n + 1)
            L.skc_report_get_note(self.h, i, buf, n + 1)
            notes.append(buf.value.decode())
        return SolveReport(bool(s.converged), s.iterations, s.cycles, hist.tolist(), s.final_residual,
                           s.op_counts.as_tuple(), [oh[i].as_tuple() for i in range(s.n_op_history)],
                           s.steady_iteration, breakdown, s.fallback_cycles, notes, br.tolist())


def _dp(a):
    return a.ctypes.data_as(P(dbl))


class Context:
    """One device context (device memory, stream, workspaces); one per calling thread."""

    def __init__(self, device: int = 0):
        self.h = C.c_void_p()
        check(lib().skc_ctx_create(device, C.byref(self.h)))
        self.device = device

    def close(self):
        if self.h:
            check(lib().skc_ctx_destroy(self.h))
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int):
        check(lib().skc_ctx_set_stream(self.h, stream_handle))

    def set_gpu_independent(self, on: bool):
        """GPU-count-independent reductions (bitwise the same results on 1, 2, 4 or 8 GPUs)."""
        check(lib().skc_ctx_set_gpu_independent(self.h, int(on)))

    def set_profiling(self, on: bool):
        check(lib().skc_ctx_set_profiling(self.h, int(on)))

    def reset_stats(self):
        check(lib().skc_ctx_reset_stats(self.h))

    def launch_count(self) -> int:
        v = u64()
        check(lib().skc_ctx_launch_count(self.h, C.byref(v)))
        return v.value

    def kernel_stats(self) -> dict:
        buf = C.create_string_buffer(8192)
        check(lib().skc_ctx_kernel_names(self.h, buf, 8192))
        out = {}
        for name in filter(None, buf.value.decode().split(",")):
            n, ms, b = u64(), dbl(), dbl()
            check(lib().skc_ctx_kernel_stats(self.h, name.encode(), C.byref(n), C.byref(ms), C.byref(b)))
            out[name] = dict(launches=n.value, ms=ms.value, bytes=b.value)
        return out

    def stencil(self, st: Stencil, kcell=None) -> "DeviceOperator":
        d = _lib.StencilDescC(st.dim, 1 if st.variable_k else 0, st.nx, st.ny, st.nz if st.dim == 3 else 1,
                              (dbl * 7)(*st.coef), st.ch2)
        kp = None
        if st.variable_k:
            if kcell is None:
                raise ValueError("variable-k stencil needs kcell")
            kcell = np.ascontiguousarray(kcell, dtype=np.float64)
            kp = _dp(kcell)
        h = C.c_void_p()
        check(lib().skc_op_create_stencil(self.h, C.byref(d), kp, C.byref(h)))
        return DeviceOperator(self, h, st.n)

    def csr(self, row_offsets, col_indices, values) -> "DeviceOperator":
        """as_operator(SparseMatrix) (sparse.hpp:155-160); size_t indices, ascending columns."""
        offs = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        cols = np.ascontiguousarray(col_indices, dtype=np.uint64)
        vals = np.ascontiguousarray(values, dtype=np.float64)
        n = len(offs) - 1
        h = C.c_void_p()
        check(lib().skc_op_create_csr(self.h, n, offs.ctypes.data_as(P(u64)), cols.ctypes.data_as(P(u64)),
                                      _dp(vals), C.byref(h)))
        return DeviceOperator(self, h, n)

    def ilu0(self, row_offsets, col_indices, values) -> "DeviceOperator":
        """right_preconditioned(a, ilu0_factor(a)) (ilu0.hpp:138-146, 45-95): the operator
        A (LU)^{-1}, ILU(0) factored on the host with the reference's algorithm; its
        `ilu0_solve` gives z = (LU)^{-1} r.  breakdown_error ("ilu0: zero pivot at row N") is
        raised as BreakdownError."""
        offs = np.ascontiguousarray(row_offsets, dtype=np.uint64)
        cols = np.ascontiguousarray(col_indices, dtype=np.uint64)
        vals = np.ascontiguousarray(values, dtype=np.float64)
        n = len(offs) - 1
        h = C.c_void_p()
        check(lib().skc_op_create_ilu0(self.h, n, offs.ctypes.data_as(P(u64)), cols.ctypes.data_as(P(u64)),
                                       _dp(vals), C.byref(h)))
        return DeviceOperator(self, h, n)


def ilu0_factor(row_offsets, col_indices, values, ctx: "Context | None" = None) -> np.ndarray:
    """ilu0_factor (ilu0.hpp:45-95), factored on the device (`ctx`, or a context on device 0):
    the factor values in A's pattern (unit-lower L strictly below the diagonal, U on and above
    it)."""
    offs = np.ascontiguousarray(row_offsets, dtype=np.uint64)
    cols = np.ascontiguousarray(col_indices, dtype=np.uint64)
    vals = np.ascontiguousarray(values, dtype=np.float64)
    lu = np.zeros(len(vals))
    ctx = ctx if ctx is not None else Context(0)
    check(lib().skc_ilu0_factor(ctx.h, len(offs) - 1, offs.ctypes.data_as(P(u64)), cols.ctypes.data_as(P(u64)),
                                _dp(vals), _dp(lu)))
    return lu


@dataclass
class DiscretizedProblem:
    """problem.hpp:121-127: the CSR system (columns ascending), rhs, analytic solution, x0."""
    nx: int
    row_offsets: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray
    rhs: np.ndarray
    u_true: np.ndarray
    x0: np.ndarray

    @property
    def n(self) -> int:
        return self.nx * self.nx


def discretize(nx: int, beta: float = 1.0, gamma: float = 50.0) -> DiscretizedProblem:
    """problem.hpp:201-203 discretize(ProblemSpec{nx, beta, gamma}): the paper's five-point
    convection-diffusion problem (1/h^2 scaling) and initial_guess, assembled on the host by the
    library (skc_discretize), bit-identical to the reference's."""
    if nx < 1:
        raise ValueError("assemble: nx must be at least 1")
    n = nx * nx
    nnz = 5 * n - 4 * nx
    out = DiscretizedProblem(nx, np.zeros(n + 1, np.uint64), np.zeros(nnz, np.uint64), np.zeros(nnz),
                             np.zeros(n), np.zeros(n), np.zeros(n))
    check(lib().skc_discretize(nx, beta, gamma, out.row_offsets.ctypes.data_as(P(u64)),
                               out.col_indices.ctypes.data_as(P(u64)), _dp(out.values), _dp(out.rhs),
                               _dp(out.x0), _dp(out.u_true)))
    return out


class DeviceOperator:
    """Device-describable operator (the GPU replacement of LinearOperator, operator.hpp:34-57)."""

    def __init__(self, ctx: Context, handle, n: int):
        self.ctx, self.h, self.n = ctx, handle, n

    def __del__(self):
        if getattr(self, "h", None) and _lib._lib is not None:
            _lib._lib.skc_op_destroy(self.h)

    def size(self) -> int:
        return self.n

    @property
    def kind(self) -> str:
        k = C.c_int()
        check(lib().skc_op_kind(self.h, C.byref(k)))
        return {0: "csr", 2: "stencil2d", 3: "stencil3d", 4: "ilu0"}[k.value]

    def ilu0_solve(self, r) -> np.ndarray:
        """z = (LU)^{-1} r for an ILU(0)-preconditioned operator (ilu0_apply, ilu0.hpp:99-127)."""
        r = np.ascontiguousarray(r, dtype=np.float64)
        if r.shape != (self.n,):
            raise ValueError("ilu0_apply: dimension mismatch")
        z = np.zeros(self.n)
        check(lib().skc_ilu0_solve(self.ctx.h, self.h, _dp(r), _dp(z)))
        return z

    def apply(self, x) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        if x.shape != (self.n,):
            raise ValueError("LinearOperator: dimension mismatch")
        y = np.zeros(self.n)
        check(lib().skc_op_apply(self.ctx.h, self.h, _dp(x), _dp(y)))
        return y

    __call__ = apply


def _check_vec(op, v, what):
    if v.dtype != np.float64 or not v.flags.c_contiguous or v.shape != (op.n,):
        raise ValueError(f"solve: {what} must be a contiguous float64 vector of length n")


def _solve(fn, op: DeviceOperator, f, x: np.ndarray, cfg) -> SolveReport:
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.shape != (op.n,) or x.shape != (op.n,):
        raise ValueError("solve: rhs/guess dimension mismatch")
    _check_vec(op, x, "x")
    rep = _Report()
    cc = cfg.c()
    check(fn(op.ctx.h, op.h, _dp(f), _dp(x), C.byref(cc), rep.h))
    return rep.collect()


def somin_solve(op, f, x, cfg: SStepConfig = SStepConfig()) -> SolveReport:
    """sstep.hpp:142-249 s-step Orthomin(k) / s-GCR; x is updated in place."""
    return _solve(lib().skc_somin_solve, op, f, x, cfg)


def sgmres_solve(op, f, x, cfg: SStepConfig = SStepConfig()) -> SolveReport:
    """sstep.hpp:493-654 restarted s-step GMRES(m); x is updated in place."""
    return _solve(lib().skc_sgmres_solve, op, f, x, cfg)


def smr_solve(op, f, x, cfg: SStepConfig = SStepConfig()) -> SolveReport:
    """sstep.hpp:109-135"""
    return _solve(lib().skc_smr_solve, op, f, x, cfg)


def gmres_solve(op, f, x, cfg: SolverConfig = SolverConfig()) -> SolveReport:
    """solvers.hpp:297-359 (standard MGS-GMRES(m) on the device)."""
    return _solve(lib().skc_gmres_solve, op, f, x, cfg)


def _dispatch(method: str, cfg: SStepConfig):
    """bench.hpp:94-124 dispatch_method for the methods with a device path: smr, somin, sgcr
    (somin with an unbounded window), sgmres, and the standard gmres (its SolverConfig built
    from cfg's m / k / tol / max_iterations as the driver does)."""
    if method == "smr":
        return smr_solve, cfg
    if method in ("somin", "sgcr"):
        return somin_solve, replace(cfg, unbounded_window=method == "sgcr")
    if method == "sgmres":
        return sgmres_solve, cfg
    if method == "gmres":
        return gmres_solve, SolverConfig(method="gmres", k=cfg.k, m=cfg.m, tol=cfg.tol,
                                         max_iterations=cfg.max_iterations, debug_checks=cfg.debug_checks)
    if method in ("mr", "omin", "gcr"):
        raise ValueError(f"solve_linear: method {method} has no device path (the standard "
                         "non-GMRES solvers are outside the s-step hot path)")
    raise ValueError("unknown method: " + method)


def solve_linear(ctx: Context, row_offsets, col_indices, values, f, x0, method: str, cfg: SStepConfig,
                 precondition: bool = True, audit=None):
    """The reference driver around the s-step solvers (solve_linear, bench.hpp:149-191), on the GPU:
    with `precondition`, ILU(0) right preconditioning -- the solver iterates w from zero on
    A (LU)^{-1} with the initial residual as right-hand side, then x = x0 + (LU)^{-1} w -- so the
    residual it minimizes is the true residual; in both cases the true residual is recomputed
    and appended to the history, and a converged solve whose true residual exceeds cfg.tol is
    reported as not converged.  Returns (x, report).  `method`: smr, somin, sgcr, sgmres or
    gmres; cfg.tol is the driver's threshold.  `audit` ("exact" / "bounded" / an AuditMode;
    None = off) runs the driver's op-count audit (bench.hpp:126-143, accounting.hpp) on the
    report and stores the verdict in report.audit."""
    from .accounting import run_audit
    if not (len(row_offsets) - 1 == len(f) == len(x0)):
        raise ValueError("solve_linear: rhs/guess dimension mismatch")
    solve, cfg = _dispatch(method, cfg)
    a = ctx.csr(row_offsets, col_indices, values)
    f = np.ascontiguousarray(f, dtype=np.float64)
    x = np.array(x0, dtype=np.float64, copy=True)
    if precondition:
        op = ctx.ilu0(row_offsets, col_indices, values)
        r0 = f - a.apply(x)
        w = np.zeros(a.n)
        rep = solve(op, r0, w, cfg)
        c = list(rep.op_counts)
        c[1] += 1  # driver-side initial residual
        c[2] += 1
        x += op.ilu0_solve(w)  # axpy(1.0, z, x)
        c[2] += 1
    else:
        rep = solve(a, f, x, cfg)
        c = list(rep.op_counts)
    ax = f - a.apply(x)
    c[1] += 1
    c[2] += 1
    c[4] += 1
    true_norm = float(np.sqrt(np.add.accumulate(ax * ax)[-1]))  # norm2: sequential sum
    rep.op_counts = tuple(c)
    rep.residual_history.append(true_norm)
    rep.final_residual = true_norm
    if rep.converged and true_norm > cfg.tol:
        rep.converged = False
        rep.breakdown = "recomputed true residual exceeds the threshold"
    if audit is not None:
        rep.audit = run_audit(rep, method, cfg.s if method != "gmres" else 1, cfg.k, cfg.m, audit)
    return x, rep


def smr_step(op, x: np.ndarray, r: np.ndarray, s: int, counter: list | None = None) -> np.ndarray:
    """sstep.hpp:89-106: one s-MR step, x and r updated in place; returns a."""
    _check_vec(op, x, "x")
    _check_vec(op, r, "r")
    a = np.zeros(s)
    c = _lib.OpCounter()
    check(lib().skc_smr_step(op.ctx.h, op.h, _dp(x), _dp(r), s, _dp(a), C.byref(c)))
    if counter is not None:
        counter[:] = list(c.as_tuple())
    return a


def krylov_block(op, v, s: int) -> np.ndarray:
    """block.hpp:59-67 -> (s, n) array of columns [v, A v, ..., A^{s-1} v]."""
    v = np.ascontiguousarray(v, dtype=np.float64)
    out = np.zeros((s, op.n))
    check(lib().skc_krylov_block(op.ctx.h, op.h, _dp(v), s, _dp(out)))
    return out


@dataclass
class SStepBasis:
    """sstep.hpp:256-262"""
    blocks: np.ndarray
    grams: np.ndarray
    hess: np.ndarray
    next_seed: np.ndarray
    next_seed_norm: float
    counter: tuple


def sarnoldi(op, v1, s: int, m_blocks: int) -> SStepBasis:
    """sstep.hpp:465-485; raises BreakdownError on collapse or an early invariant subspace."""
    v1 = np.ascontiguousarray(v1, dtype=np.float64)
    n = op.n
    if s < 1:
        raise ValueError("sarnoldi: s must be at least 1")
    if m_blocks < 1:
        raise ValueError("sarnoldi: m_blocks must be at least 1")
    blocks = np.zeros((m_blocks, s, n))
    grams = np.zeros((m_blocks, s, s))
    hess = np.zeros(((m_blocks + 1) * s, m_blocks * s))
    seed = np.zeros(n)
    sn = dbl()
    c = _lib.OpCounter()
    check(lib().skc_sarnoldi(op.ctx.h, op.h, _dp(v1), s, m_blocks, _dp(blocks), _dp(grams), _dp(hess), _dp(seed),
                             C.byref(sn), C.byref(c)))
    return SStepBasis(blocks, grams, hess, seed, sn.value, c.as_tuple())


# ---------------------------------------------------------------- device-resident entry points
def somin_solve_device(op, f_ptr: int, x_ptr: int, cfg: SStepConfig) -> SolveReport:
    rep = _Report()
    cc = cfg.c()
    check(lib().skc_somin_solve_device(op.ctx.h, op.h, C.c_void_p(f_ptr), C.c_void_p(x_ptr), C.byref(cc), rep.h))
    return rep.collect()


def sgmres_solve_device(op, f_ptr: int, x_ptr: int, cfg: SStepConfig) -> SolveReport:
    rep = _Report()
    cc = cfg.c()
    check(lib().skc_sgmres_solve_device(op.ctx.h, op.h, C.c_void_p(f_ptr), C.c_void_p(x_ptr), C.byref(cc), rep.h))
    return rep.collect()


# ---------------------------------------------------------------- host small dense (no GPU)
def gram_solve(w, rhs=None):
    w = np.ascontiguousarray(w, dtype=np.float64)
    n = w.shape[0]
    rhs = np.zeros((n, 0)) if rhs is None else np.ascontiguousarray(rhs, dtype=np.float64).reshape(n, -1)
    x = np.zeros_like(rhs)
    ldlt = C.c_int32()
    piv = np.zeros(n)
    check(lib().skc_gram_solve(n, _dp(w), rhs.shape[1], _dp(rhs), _dp(x), C.byref(ldlt), _dp(piv)))
    return x, bool(ldlt.value), piv


def cholesky_upper(w):
    w = np.ascontiguousarray(w, dtype=np.float64)
    r = np.zeros_like(w)
    check(lib().skc_cholesky_upper(w.shape[0], _dp(w), _dp(r)))
    return r


def hessenberg_lsq(g, beta):
    g = np.ascontiguousarray(g, dtype=np.float64)
    y = np.zeros(g.shape[1])
    res = dbl()
    check(lib().skc_hessenberg_lsq(g.shape[0], g.shape[1], _dp(g), beta, _dp(y), C.byref(res)))
    return y, res.value
