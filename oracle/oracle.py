"""oracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes front end for the CPU checkers:
  * ``liboracle.so``      -- the plain-C restatement (prefix ``orc_``), always built;
  * ``_ref/libskref.so``  -- the unmodified reference headers behind the same ABI
                             (prefix ``ref_``), built only where /root/reference exists.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs import this module.
The product package (paper_2001_04886_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
u64 = C.c_uint64
i32 = C.c_int32
dbl = C.c_double
P = C.POINTER


class Counter(C.Structure):
    _fields_ = [("dotprods", u64), ("matvecs", u64), ("vec_updates", u64),
                ("stored_vectors", u64), ("termination_dots", u64)]

    def as_tuple(self):
        return (self.dotprods, self.matvecs, self.vec_updates, self.stored_vectors,
                self.termination_dots)


class Csr(C.Structure):
    _fields_ = [("n", u64), ("row_offsets", P(u64)), ("col_indices", P(u64)), ("values", P(dbl))]


class SStepCfg(C.Structure):
    _fields_ = [("s", u64), ("k", u64), ("m", u64), ("tol", dbl), ("max_iterations", u64),
                ("precondition", i32), ("unbounded_window", i32), ("debug_checks", i32),
                ("divergence_factor", dbl)]


class SolverCfg(C.Structure):
    _fields_ = [("method", i32), ("k", u64), ("m", u64), ("tol", dbl), ("max_iterations", u64),
                ("precondition", i32), ("debug_checks", i32), ("divergence_factor", dbl)]


class Report(C.Structure):
    _fields_ = [("converged", i32), ("iterations", u64), ("cycles", u64),
                ("history", P(dbl)), ("n_history", u64), ("final_residual", dbl),
                ("op_counts", Counter), ("op_history", P(Counter)), ("n_op_history", u64),
                ("steady_iteration", u64), ("has_breakdown", i32), ("breakdown", C.c_char * 512),
                ("fallback_cycles", u64), ("n_notes", i32), ("notes", (C.c_char * 256) * 4),
                ("block_rho", P(dbl)), ("n_block_rho", u64), ("error", C.c_char * 512)]


METHODS = {"mr": 0, "omin": 1, "gcr": 2, "gmres": 3}
STATUS = {0: None, 1: ValueError, 2: "breakdown", 3: "logic", 4: MemoryError}


class OracleError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(msg)
        self.status = status


@dataclass
class SolveResult:
    converged: bool
    iterations: int
    cycles: int
    residual_history: list
    final_residual: float
    op_counts: tuple
    op_history: list
    steady_iteration: int
    breakdown: str | None
    fallback_cycles: int
    notes: list
    block_rho: list = field(default_factory=list)
    x: np.ndarray | None = None


def _dp(a):
    return a.ctypes.data_as(P(dbl))


def _up(a):
    return a.ctypes.data_as(P(u64))


class CsrMatrix:
    """Keeps the numpy arrays alive for the C struct."""

    def __init__(self, offs, cols, vals):
        self.offs = np.ascontiguousarray(offs, dtype=np.uint64)
        self.cols = np.ascontiguousarray(cols, dtype=np.uint64)
        self.vals = np.ascontiguousarray(vals, dtype=np.float64)
        self.n = len(self.offs) - 1
        self.c = Csr(self.n, _up(self.offs), _up(self.cols), _dp(self.vals))

    @classmethod
    def from_dense(cls, a):
        a = np.asarray(a, dtype=np.float64)
        offs, cols, vals = [0], [], []
        for i in range(a.shape[0]):
            for j in range(a.shape[1]):
                if a[i, j] != 0.0:
                    cols.append(j)
                    vals.append(a[i, j])
            offs.append(len(cols))
        return cls(offs, cols, vals)

    @classmethod
    def from_triplets(cls, n, trip):
        trip = sorted(trip, key=lambda t: (t[0], t[1]))
        offs = np.zeros(n + 1, dtype=np.uint64)
        cols, vals = [], []
        for i, j, v in trip:
            offs[i + 1] += 1
            cols.append(j)
            vals.append(v)
        return cls(np.cumsum(offs, dtype=np.uint64), cols, vals)

    def to_dense(self):
        d = np.zeros((self.n, self.n))
        for i in range(self.n):
            for p in range(int(self.offs[i]), int(self.offs[i + 1])):
                d[i, int(self.cols[p])] = self.vals[p]
        return d


class Oracle:
    """One of the two CPU checkers, selected by ``kind`` ("port" or "reference")."""

    def __init__(self, kind="port"):
        self.kind = kind
        if kind == "port":
            path, self.px = os.path.join(HERE, "liboracle.so"), "orc_"
        elif kind == "reference":
            path, self.px = os.path.join(HERE, "_ref", "libskref.so"), "ref_"
        else:
            raise ValueError(kind)
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} is not built (run `make -C oracle`)")
        self.path = path
        self.lib = C.CDLL(path)
        self._sig()

    @staticmethod
    def available(kind):
        p = os.path.join(HERE, "liboracle.so") if kind == "port" else os.path.join(HERE, "_ref", "libskref.so")
        return os.path.exists(p)

    def f(self, name):
        return getattr(self.lib, self.px + name)

    def _sig(self):
        L = self.f
        solve_args = [P(Csr), P(dbl), P(dbl), P(SStepCfg), P(Report)]
        for nm in ("smr_solve", "somin_solve", "sgmres_solve"):
            L(nm).argtypes = solve_args
            L(nm).restype = C.c_int
        for nm in ("mr_solve", "omin_solve", "gmres_solve"):
            L(nm).argtypes = [P(Csr), P(dbl), P(dbl), P(SolverCfg), P(Report)]
            L(nm).restype = C.c_int
        L("report_free").argtypes = [P(Report)]
        L("spmv").argtypes = [P(Csr), P(dbl), P(dbl)]
        L("krylov_block").argtypes = [P(Csr), P(dbl), u64, P(dbl)]
        L("krylov_block").restype = C.c_int
        L("gram_solve").argtypes = [u64, P(dbl), u64, P(dbl), P(dbl), P(i32), P(dbl), C.c_char_p, u64]
        L("gram_solve").restype = C.c_int
        L("cholesky_upper").argtypes = [u64, P(dbl), P(dbl), C.c_char_p, u64]
        L("cholesky_upper").restype = C.c_int
        L("hessenberg_lsq").argtypes = [u64, u64, P(dbl), dbl, P(dbl), P(dbl), C.c_char_p, u64]
        L("hessenberg_lsq").restype = C.c_int
        L("smr_step").argtypes = [P(Csr), P(dbl), P(dbl), u64, P(dbl), P(Counter)]
        L("smr_step").restype = C.c_int
        L("arnoldi").argtypes = [P(Csr), P(dbl), u64, P(dbl), P(u64), P(i32)]
        L("arnoldi").restype = C.c_int
        L("sarnoldi").argtypes = [P(Csr), P(dbl), u64, u64, P(dbl), P(dbl), P(dbl), P(dbl), P(dbl),
                                  P(Counter), C.c_char_p, u64]
        L("sarnoldi").restype = C.c_int
        L("ilu0_factor").argtypes = [P(Csr), P(dbl), C.c_char_p, u64]
        L("ilu0_factor").restype = C.c_int
        L("ilu0_apply").argtypes = [P(Csr), P(dbl), P(dbl), P(dbl)]
        if self.px == "ref_":
            self.lib.ref_solve_linear.argtypes = [P(Csr), P(dbl), P(dbl), i32, P(SStepCfg), i32, P(dbl), P(Report)]
            self.lib.ref_solve_linear.restype = C.c_int
        if self.px == "orc_":
            self.lib.orc_set_right_preconditioner.argtypes = [P(Csr), P(dbl)]
            self.lib.orc_fill_uniform.argtypes = [u64, u64, u64, P(dbl)]
            self.lib.orc_fill_lognormal.argtypes = [u64, u64, P(dbl)]
            self.lib.orc_build_stencil_csr.argtypes = [i32, u64, u64, u64, P(dbl), P(dbl), dbl,
                                                       P(P(u64)), P(P(u64)), P(P(dbl))]
            self.lib.orc_build_stencil_csr.restype = C.c_int
            self.lib.orc_csr_free.argtypes = [P(u64), P(u64), P(dbl)]
            self.lib.orc_stencil_apply.argtypes = [i32, u64, u64, u64, P(dbl), P(dbl), dbl, P(dbl), P(dbl)]
            self.lib.orc_set_dot_mode.argtypes = [C.c_int]
            self.lib.orc_set_fixed_steps.argtypes = [C.c_int]

    def set_fixed_steps(self, on: bool):
        """Fixed-step benchmark mode (port only): bypass the Gram pivot-ratio and LSQ rank aborts."""
        self.lib.orc_set_fixed_steps(int(bool(on)))

    def set_dot_mode(self, mode: int):
        """0: the reference's sequential summation; 1: blocked/tree (envelope measurement only)."""
        self.lib.orc_set_dot_mode(mode)

    # ------------------------------------------------------------------ solvers
    def _collect(self, rep, x):
        h = [rep.history[i] for i in range(rep.n_history)]
        oh = [rep.op_history[i].as_tuple() for i in range(rep.n_op_history)]
        br = [rep.block_rho[i] for i in range(rep.n_block_rho)]
        res = SolveResult(bool(rep.converged), rep.iterations, rep.cycles, h, rep.final_residual,
                          rep.op_counts.as_tuple(), oh, rep.steady_iteration,
                          rep.breakdown.decode() if rep.has_breakdown else None, rep.fallback_cycles,
                          [rep.notes[i].value.decode() for i in range(rep.n_notes)], br, x)
        return res

    def _run(self, name, a, f, x0, cfg):
        f = np.ascontiguousarray(f, dtype=np.float64)
        x = np.array(x0, dtype=np.float64, copy=True)
        rep = Report()
        st = self.f(name)(C.byref(a.c), _dp(f), _dp(x), C.byref(cfg), C.byref(rep))
        try:
            if st:
                raise OracleError(st, rep.error.decode())
            return self._collect(rep, x)
        finally:
            self.f("report_free")(C.byref(rep))

    def sstep(self, method, a, f, x0=None, *, s=2, k=2, m=5, tol=1e-6, max_iterations=100000,
              precondition=False, unbounded_window=False, debug_checks=False, divergence_factor=10.0):
        x0 = np.zeros(a.n) if x0 is None else x0
        cfg = SStepCfg(s, k, m, tol, max_iterations, int(precondition), int(unbounded_window),
                       int(debug_checks), divergence_factor)
        return self._run(method + "_solve", a, f, x0, cfg)

    def standard(self, method, a, f, x0=None, *, k=4, m=10, tol=1e-6, max_iterations=100000,
                 debug_checks=False, divergence_factor=10.0):
        x0 = np.zeros(a.n) if x0 is None else x0
        cfg = SolverCfg(METHODS[method], k, m, tol, max_iterations, 0, int(debug_checks), divergence_factor)
        name = {"mr": "mr_solve", "omin": "omin_solve", "gcr": "omin_solve", "gmres": "gmres_solve"}[method]
        return self._run(name, a, f, x0, cfg)

    # ------------------------------------------------------------------ kernels
    # ------------------------------------------------------------------ ILU(0) (ilu0.hpp)
    def ilu0_factor(self, a):
        """Factor values in A's pattern (unit-lower L below the diagonal, U on and above)."""
        lu = np.zeros(len(a.vals))
        err = C.create_string_buffer(512)
        st = self.f("ilu0_factor")(C.byref(a.c), _dp(lu), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return lu

    def ilu0_apply(self, a, lu, r):
        """z = (LU)^{-1} r."""
        lu = np.ascontiguousarray(lu, dtype=np.float64)
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(a.n)
        self.f("ilu0_apply")(C.byref(a.c), _dp(lu), _dp(r), _dp(z))
        return z

    def solve_linear(self, method, a, f, x0=None, *, precondition=True, s=2, k=2, m=5, tol=1e-6,
                     max_iterations=100000, divergence_factor=10.0):
        """The reference driver flow (bench.hpp:149-191) around s-Omin / s-GMRES: with
        `precondition`, ILU(0) right preconditioning from w = 0, x = x0 + K^{-1} w; the true
        residual recomputed and appended.  Reference build only."""
        x0 = np.zeros(a.n) if x0 is None else np.ascontiguousarray(x0, dtype=np.float64)
        f = np.ascontiguousarray(f, dtype=np.float64)
        if self.px == "orc_":
            return self._solve_linear_port(method, a, f, x0, precondition, dict(
                s=s, k=k, m=m, tol=tol, max_iterations=max_iterations, divergence_factor=divergence_factor))
        cfg = SStepCfg(s, k, m, tol, max_iterations, 0, 0, 0, divergence_factor)
        x = np.zeros(a.n)
        rep = Report()
        st = self.lib.ref_solve_linear(C.byref(a.c), _dp(f), _dp(x0), {"somin": 0, "sgmres": 1, "gmres": 2}[method],
                                       C.byref(cfg), int(precondition), _dp(x), C.byref(rep))
        try:
            if st:
                raise OracleError(st, rep.error.decode())
            return self._collect(rep, x)
        finally:
            self.f("report_free")(C.byref(rep))

    def _solve_linear_port(self, method, a, f, x0, precondition, cfg):
        """bench.hpp:149-191 with the restatement's solvers (the operator switched to A (LU)^{-1}
        through orc_set_right_preconditioner while the solver runs)."""
        x = np.array(x0, dtype=np.float64, copy=True)
        if precondition:
            lu = self.ilu0_factor(a)
            r0 = f - self.spmv(a, x)
            self.lib.orc_set_right_preconditioner(C.byref(a.c), _dp(lu))
            try:
                res = self.sstep(method, a, r0, np.zeros(a.n), **cfg)
            finally:
                self.lib.orc_set_right_preconditioner(C.byref(a.c), None)
            c = list(res.op_counts)
            c[1] += 1
            c[2] += 1
            z = self.ilu0_apply(a, lu, res.x)
            x += z
            c[2] += 1
        else:
            res = self.sstep(method, a, f, x, **cfg)
            x = res.x
            c = list(res.op_counts)
        ax = f - self.spmv(a, x)
        c[1] += 1
        c[2] += 1
        c[4] += 1
        true_norm = float(np.sqrt(np.add.accumulate(ax * ax)[-1]))
        res.op_counts = tuple(c)
        res.residual_history.append(true_norm)
        res.final_residual = true_norm
        if res.converged and true_norm > cfg["tol"]:
            res.converged = False
            res.breakdown = "recomputed true residual exceeds the threshold"
        res.x = x
        return res

    def spmv(self, a, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(a.n)
        self.f("spmv")(C.byref(a.c), _dp(x), _dp(y))
        return y

    def krylov_block(self, a, v, s):
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.zeros((s, a.n))
        self.f("krylov_block")(C.byref(a.c), _dp(v), s, _dp(out))
        return out

    def gram_solve(self, w, rhs=None):
        w = np.ascontiguousarray(w, dtype=np.float64)
        n = w.shape[0]
        rhs = np.zeros((n, 0)) if rhs is None else np.ascontiguousarray(rhs, dtype=np.float64).reshape(n, -1)
        x = np.zeros_like(rhs)
        ldlt = i32(0)
        piv = np.zeros(n)
        err = C.create_string_buffer(512)
        st = self.f("gram_solve")(n, _dp(w), rhs.shape[1], _dp(rhs), _dp(x), C.byref(ldlt), _dp(piv), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return x, bool(ldlt.value), piv

    def cholesky_upper(self, w):
        w = np.ascontiguousarray(w, dtype=np.float64)
        r = np.zeros_like(w)
        err = C.create_string_buffer(512)
        st = self.f("cholesky_upper")(w.shape[0], _dp(w), _dp(r), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return r

    def hessenberg_lsq(self, g, beta):
        g = np.ascontiguousarray(g, dtype=np.float64)
        y = np.zeros(g.shape[1])
        res = dbl(0)
        err = C.create_string_buffer(512)
        st = self.f("hessenberg_lsq")(g.shape[0], g.shape[1], _dp(g), beta, _dp(y), C.byref(res), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return y, res.value

    def smr_step(self, a, x, r, s):
        x = np.array(x, dtype=np.float64)
        r = np.array(r, dtype=np.float64)
        co = np.zeros(s)
        c = Counter()
        st = self.f("smr_step")(C.byref(a.c), _dp(x), _dp(r), s, _dp(co), C.byref(c))
        if st:
            raise OracleError(st, "smr_step failed")
        return x, r, co, c.as_tuple()

    def arnoldi(self, a, v1, m):
        v1 = np.ascontiguousarray(v1, dtype=np.float64)
        h = np.zeros((m + 1, m))
        steps, happy = u64(0), i32(0)
        self.f("arnoldi")(C.byref(a.c), _dp(v1), m, _dp(h), C.byref(steps), C.byref(happy))
        return h, steps.value, bool(happy.value)

    def sarnoldi(self, a, v1, s, m_blocks):
        v1 = np.ascontiguousarray(v1, dtype=np.float64)
        n = a.n
        blocks = np.zeros((m_blocks, s, n))
        grams = np.zeros((m_blocks, s, s))
        hess = np.zeros(((m_blocks + 1) * s, m_blocks * s))
        seed = np.zeros(n)
        sn = dbl(0)
        c = Counter()
        err = C.create_string_buffer(512)
        st = self.f("sarnoldi")(C.byref(a.c), _dp(v1), s, m_blocks, _dp(blocks), _dp(grams), _dp(hess),
                                _dp(seed), C.byref(sn), C.byref(c), err, 512)
        if st:
            raise OracleError(st, err.value.decode())
        return dict(blocks=blocks, grams=grams, hess=hess, next_seed=seed, next_seed_norm=sn.value,
                    counter=c.as_tuple())

    # ------------------------------------------------------------------ problem generators (port only)
    def uniform(self, seed, n, offset=0):
        out = np.zeros(n)
        self.lib.orc_fill_uniform(seed, offset, n, _dp(out))
        return out

    def lognormal(self, seed, n):
        out = np.zeros(n)
        self.lib.orc_fill_lognormal(seed, n, _dp(out))
        return out

    def stencil_csr(self, dim, nx, ny, nz, coef, kcell=None, ch2=0.0):
        coef = np.ascontiguousarray(coef if coef is not None else np.zeros(7), dtype=np.float64)
        kp = _dp(np.ascontiguousarray(kcell, dtype=np.float64)) if kcell is not None else None
        po, pc, pv = P(u64)(), P(u64)(), P(dbl)()
        st = self.lib.orc_build_stencil_csr(dim, nx, ny, nz, _dp(coef), kp, ch2, C.byref(po), C.byref(pc), C.byref(pv))
        if st:
            raise MemoryError("stencil csr")
        n = nx * ny * (nz if dim == 3 else 1)
        nnz = po[n]
        offs = np.ctypeslib.as_array(po, shape=(n + 1,)).copy()
        cols = np.ctypeslib.as_array(pc, shape=(nnz,)).copy()
        vals = np.ctypeslib.as_array(pv, shape=(nnz,)).copy()
        self.lib.orc_csr_free(po, pc, pv)
        return CsrMatrix(offs, cols, vals)

    def stencil_apply(self, dim, nx, ny, nz, coef, x, kcell=None, ch2=0.0):
        coef = np.ascontiguousarray(coef if coef is not None else np.zeros(7), dtype=np.float64)
        kp = _dp(np.ascontiguousarray(kcell, dtype=np.float64)) if kcell is not None else None
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros_like(x)
        self.lib.orc_stencil_apply(dim, nx, ny, nz, _dp(coef), kp, ch2, _dp(x), _dp(y))
        return y
