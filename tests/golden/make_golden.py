"""Generate tests/golden/ from the UNMODIFIED reference (oracle/_ref/libskref.so).

Run in the build container (needs /root/reference to have built oracle/_ref):

    make -C oracle && python tests/golden/make_golden.py

Each case mirrors a reference known-answer test (tests/test_sstep.cpp, test_block.cpp,
test_small_dense.cpp, test_accounting.cpp) or a reduced-size BASELINE configuration.
Inputs (operator, f, x0, config) and the reference's outputs (residual history, final
iterate, op counters, breakdown/notes strings) are stored together so the GPU parity
tests and the oracle pin tests need no /root/reference at run time.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import CsrMatrix, Oracle, OracleError  # noqa: E402
from paper_2001_04886_b200.problems import RHS_SEED, K_SEED, convection_diffusion, splitmix64_uniform  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
REF = Oracle("reference")
PORT = Oracle("port")
P = C.POINTER
REF.lib.ref_discretize.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_int32, P(P(C.c_uint64)),
                                   P(P(C.c_uint64)), P(P(C.c_double)), P(P(C.c_double)), P(P(C.c_double))]
REF.lib.ref_mt_uniform.argtypes = [C.c_uint32, C.c_uint64, C.c_double, C.c_double, P(C.c_double)]
REF.lib.ref_free.argtypes = [C.c_void_p]


def discretize(nx, beta=1.0, gamma=50.0, symmetric=False):
    """problem.hpp:201-203 discretize(ProblemSpec{nx, beta, gamma}) (1/h^2 scaling)."""
    po, pc, pv, pr, px = P(C.c_uint64)(), P(C.c_uint64)(), P(C.c_double)(), P(C.c_double)(), P(C.c_double)()
    REF.lib.ref_discretize(nx, beta, gamma, int(symmetric), C.byref(po), C.byref(pc), C.byref(pv),
                           C.byref(pr), C.byref(px))
    n = nx * nx
    nnz = po[n]
    offs = np.ctypeslib.as_array(po, (n + 1,)).copy()
    cols = np.ctypeslib.as_array(pc, (nnz,)).copy()
    vals = np.ctypeslib.as_array(pv, (nnz,)).copy()
    rhs = np.ctypeslib.as_array(pr, (n,)).copy()
    x0 = np.ctypeslib.as_array(px, (n,)).copy()
    for p in (po, pc, pv, pr, px):
        REF.lib.ref_free(C.cast(p, C.c_void_p))
    return CsrMatrix(offs, cols, vals), rhs, x0


class MT:
    """Sequential std::mt19937 + uniform_real_distribution(-1,1) draws (oracles.hpp:117-133)."""

    def __init__(self, seed):
        self.seed = seed
        self.pos = 0

    def draw(self, count):
        buf = np.zeros(self.pos + count)
        REF.lib.ref_mt_uniform(self.seed, self.pos + count, -1.0, 1.0, buf.ctypes.data_as(P(C.c_double)))
        out = buf[self.pos:]
        self.pos += count
        return out.copy()

    def dense(self, n, shift):
        a = self.draw(n * n).reshape(n, n)
        a[np.diag_indices(n)] += shift
        return a


def nilpotent_plus_identity(n=24):
    trip = []
    for i in range(n):
        trip.append((i, i, 1.0))
        if i % 3 != 2:
            trip.append((i, i + 1, 0.5))
    return CsrMatrix.from_triplets(n, trip)


manifest = {}


def save(name, arrays, meta):
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **arrays)
    manifest[name] = meta


def solve_case(name, kind, method, a, f, x0, cfg, ref_source):
    """kind: 'sstep' (SStepConfig) or 'standard' (SolverConfig)."""
    if kind == "sstep":
        res = REF.sstep(method, a, f, x0, **cfg)
    else:
        res = REF.standard(method, a, f, x0, **cfg)
    arrays = dict(offs=a.offs, cols=a.cols, vals=a.vals, f=np.asarray(f, float), x0=np.asarray(x0, float),
                  x=res.x, history=np.array(res.residual_history),
                  op_history=np.array(res.op_history, dtype=np.uint64).reshape(-1, 5),
                  op_counts=np.array(res.op_counts, dtype=np.uint64))
    meta = dict(type="solve", kind=kind, method=method, cfg=cfg, ref=ref_source,
                converged=res.converged, iterations=res.iterations, cycles=res.cycles,
                final_residual=res.final_residual, steady_iteration=res.steady_iteration,
                breakdown=res.breakdown, fallback_cycles=res.fallback_cycles, notes=res.notes)
    save(name, arrays, meta)
    return res


def stencil_case(name, method, dim, nx, conv, cfg, rel_tol=None, ref_source="", variable_k=False):
    st = convection_diffusion(dim, nx, conv, variable_k=variable_k)
    kcell = PORT.lognormal(K_SEED, st.n) if variable_k else None
    a = PORT.stencil_csr(dim, st.nx, st.ny, st.nz, st.coef, kcell=kcell, ch2=st.ch2)
    f = splitmix64_uniform(RHS_SEED, a.n)
    cfg = dict(cfg)
    if rel_tol is not None:
        cfg["tol"] = rel_tol * float(np.linalg.norm(f))
    res = solve_case(name, "sstep", method, a, f, np.zeros(a.n), cfg, ref_source)
    manifest[name]["stencil"] = dict(dim=dim, nx=st.nx, ny=st.ny, nz=st.nz, coef=list(st.coef), ch2=st.ch2,
                                     variable_k=variable_k, rhs_seed=RHS_SEED, k_seed=K_SEED, conv=conv)
    if kcell is not None:
        d = dict(np.load(os.path.join(OUT, name + ".npz")))
        d["kcell"] = kcell
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **d)
    return res


def main():
    # ---------------- tests/test_sstep.cpp KATs
    a5, rhs5, x05 = discretize(5)
    a7, rhs7, x07 = discretize(7)
    a3, rhs3, x03 = discretize(3)
    # :45-69 smr_step(s=1) == one MR step; :82-102 smr_step(3) == gmres(3) one cycle
    for nm, (a, rhs, x0, s) in {"smr_step_s1_nx5": (a5, rhs5, x05, 1), "smr_step_s3_nx3": (a3, rhs3, x03, 3),
                                "smr_step_s3_nx5": (a5, rhs5, x05, 3)}.items():
        r0 = rhs - REF.spmv(a, x0)
        x, r, co, cnt = REF.smr_step(a, x0, r0, s)
        save(nm, dict(offs=a.offs, cols=a.cols, vals=a.vals, x0=x0, r0=r0, x=x, r=r, coeffs=co),
             dict(type="smr_step", s=s, counter=list(cnt), ref="test_sstep.cpp:45-127"))
    solve_case("mr_nx5_max1", "standard", "mr", a5, rhs5, x05, dict(tol=1e-30, max_iterations=1), "test_sstep.cpp:56-62")
    solve_case("gmres_m3_nx3", "standard", "gmres", a3, rhs3, x03, dict(m=3, tol=1e-30, max_iterations=3), "test_sstep.cpp:91-100")
    # :129-149 smr(1) == mr over a whole solve
    solve_case("smr_s1_nx5", "sstep", "smr", a5, rhs5, x05, dict(s=1, tol=1e-4, max_iterations=500), "test_sstep.cpp:129-149")
    solve_case("mr_nx5", "standard", "mr", a5, rhs5, x05, dict(tol=1e-4, max_iterations=500), "test_sstep.cpp:129-149")
    # :151-189 somin(s=1,k=4) == omin(4) (unpreconditioned half; ILU(0) is out of scope)
    solve_case("somin_s1_k4_nx7", "sstep", "somin", a7, rhs7, x07, dict(s=1, k=4, tol=1e-6), "test_sstep.cpp:151-189")
    solve_case("omin_k4_nx7", "standard", "omin", a7, rhs7, x07, dict(k=4, tol=1e-6), "test_sstep.cpp:151-189")
    # :191-220 somin(s=2,k=1) vs s-GCR on the symmetric problem, f from mt19937(15)
    a7s, _, _ = discretize(7, 0.0, 0.0, symmetric=True)
    f15 = MT(15).draw(49)
    z49 = np.zeros(49)
    solve_case("somin_s2_k1_sym", "sstep", "somin", a7s, f15, z49, dict(s=2, k=1, tol=1e-30, max_iterations=12), "test_sstep.cpp:191-220")
    solve_case("sgcr_s2_sym", "sstep", "somin", a7s, f15, z49, dict(s=2, unbounded_window=True, tol=1e-30, max_iterations=12), "test_sstep.cpp:191-220")
    # :222-238 monotone residuals with debug checks
    solve_case("somin_s2_k2_debug_nx7", "sstep", "somin", a7, rhs7, x07, dict(s=2, k=2, tol=1e-6, debug_checks=True), "test_sstep.cpp:222-238")
    # :313-336 sgmres(s=1) shares gmres history
    solve_case("sgmres_s1_m5_nx7", "sstep", "sgmres", a7, rhs7, x07, dict(s=1, m=5, tol=1e-6, max_iterations=5000), "test_sstep.cpp:313-336")
    solve_case("gmres_m5_nx7", "standard", "gmres", a7, rhs7, x07, dict(m=5, tol=1e-6, max_iterations=5000), "test_sstep.cpp:313-336")
    # :338-368 Remark 4.1: sgmres(s=2,m=4) vs gmres(8), dense 40, mt19937(33)
    mt = MT(33)
    d40 = CsrMatrix.from_dense(mt.dense(40, 4.0))
    f40 = mt.draw(40)
    solve_case("sgmres_s2_m4_dense40", "sstep", "sgmres", d40, f40, np.zeros(40), dict(s=2, m=4, tol=1e-30, max_iterations=24), "test_sstep.cpp:338-368")
    solve_case("gmres_m8_dense40", "standard", "gmres", d40, f40, np.zeros(40), dict(m=8, tol=1e-30, max_iterations=24), "test_sstep.cpp:338-368")
    # :370-405 matvec budgets
    solve_case("sgmres_s2_m3_nx7_budget", "sstep", "sgmres", a7, rhs7, x07, dict(s=2, m=3, tol=1e-30, max_iterations=18), "test_sstep.cpp:370-387")
    solve_case("somin_s3_k2_nx7_budget", "sstep", "somin", a7, rhs7, x07, dict(s=3, k=2, tol=1e-6), "test_sstep.cpp:389-405")
    # :407-457 degenerate I+N operator: fallback recovery and basis-collapse report
    inil = nilpotent_plus_identity(24)
    solve_case("sgmres_s6_m2_nilpotent", "sstep", "sgmres", inil, MT(55).draw(24), np.zeros(24), dict(s=6, m=2, tol=1e-10), "test_sstep.cpp:407-434")
    solve_case("somin_s6_k2_nilpotent", "sstep", "somin", inil, MT(56).draw(24), np.zeros(24), dict(s=6, k=2, tol=1e-12), "test_sstep.cpp:436-457")
    # ---------------- test_accounting.cpp
    solve_case("somin_s2_k2_nx7_audit", "sstep", "somin", a7, rhs7, x07, dict(s=2, k=2, tol=1e-6), "test_accounting.cpp:101-118")
    solve_case("sgmres_s2_m2_nx7_audit", "sstep", "sgmres", a7, rhs7, x07, dict(s=2, m=2, tol=1e-30, max_iterations=12), "test_accounting.cpp:120-141")
    # ---------------- sarnoldi KATs (:240-311)
    mt = MT(19)
    d25 = CsrMatrix.from_dense(mt.dense(25, 3.0))
    v25 = mt.draw(25)
    mt = MT(21)
    d30 = CsrMatrix.from_dense(mt.dense(30, 2.0))
    v30 = mt.draw(30)
    e0 = np.zeros(9)
    e0[0] = 2.0
    for nm, (a, v, s, m) in {"sarnoldi_s1_m6_dense25": (d25, v25, 1, 6), "sarnoldi_s3_m1_nx3": (a3, e0, 3, 1),
                             "sarnoldi_s2_m3_dense30": (d30, v30, 2, 3), "sarnoldi_s3_m5_dense30": (d30, v30, 3, 5)}.items():
        b = REF.sarnoldi(a, v, s, m)
        h, steps, happy = REF.arnoldi(a, v, m) if s == 1 else (np.zeros((1, 1)), 0, False)
        save(nm, dict(offs=a.offs, cols=a.cols, vals=a.vals, v1=v, blocks=b["blocks"], grams=b["grams"],
                      hess=b["hess"], next_seed=b["next_seed"], arnoldi_h=h),
             dict(type="sarnoldi", s=s, m_blocks=m, next_seed_norm=b["next_seed_norm"], counter=list(b["counter"]),
                  ref="test_sstep.cpp:240-311"))
    # ---------------- test_block.cpp:49-60 krylov_block recurrence (paper problem nx=3, beta 1, gamma 50)
    e1 = np.zeros(9)
    e1[0] = 1.0
    kb = REF.krylov_block(a3, e1, 4)
    save("krylov_block_nx3_s4", dict(offs=a3.offs, cols=a3.cols, vals=a3.vals, v=e1, blocks=kb),
         dict(type="krylov_block", s=4, ref="test_block.cpp:49-60"))
    # ---------------- test_small_dense.cpp KATs (Gram solver / Cholesky / Hessenberg LSQ)
    gram_cases = {"identity3": (np.eye(3), np.array([[0.0], [1.0], [0.0]])),
                  "diag": (np.diag([4.0, 9.0]), np.array([[8.0], [27.0]])),
                  "indefinite_ldlt": (np.array([[1.0, 2.0], [2.0, 1.0]]), np.array([[3.0], [5.0]])),
                  "singular": (np.ones((2, 2)), None), "zero1": (np.zeros((1, 1)), None)}
    mt = MT(5)
    for t in range(6):
        u = mt.draw(40).reshape(4, 10)
        w = u @ u.T
        w = (w + w.T) / 2
        gram_cases[f"spd{t}"] = (w, mt.draw(4).reshape(4, 1))
    near = np.array([[1.0, 1.0 - 1e-9], [1.0 - 1e-9, 1.0]])
    gram_cases["near_singular_chol"] = (near, np.array([[1.0], [2.0]]))
    gram = {}
    for nm, (w, rhs) in gram_cases.items():
        try:
            x, ldlt, piv = REF.gram_solve(w, rhs)
            gram[nm] = dict(w=w.tolist(), rhs=None if rhs is None else rhs.tolist(), x=x.tolist(), ldlt=ldlt,
                            pivots=piv.tolist(), error=None)
        except OracleError as e:
            gram[nm] = dict(w=w.tolist(), rhs=None if rhs is None else rhs.tolist(), x=None, ldlt=None,
                            pivots=None, error=str(e))
    mt = MT(7)
    g = np.zeros((7, 6))
    for j in range(6):
        for i in range(j + 2):
            g[i, j] = mt.draw(1)[0]
    y, res = REF.hessenberg_lsq(g, 1.5)
    gdef = np.array([[1.0, 2.0], [0.0, 0.0], [0.0, 0.0]])
    try:
        REF.hessenberg_lsq(gdef, 1.0)
        lsq_err = None
    except OracleError as e:
        lsq_err = str(e)
    chol = REF.cholesky_upper(np.array([[4.0, 2.0], [2.0, 3.0]]))
    try:
        REF.cholesky_upper(np.array([[1.0, 2.0], [2.0, 1.0]]))
        chol_err = None
    except OracleError as e:
        chol_err = str(e)
    manifest["small_dense"] = dict(type="small_dense", gram=gram, lsq=dict(g=g.tolist(), beta=1.5, y=y.tolist(), residual=res),
                                   lsq_deficient=dict(g=gdef.tolist(), error=lsq_err),
                                   chol=dict(w=[[4.0, 2.0], [2.0, 3.0]], r=chol.tolist()),
                                   chol_indef=dict(error=chol_err), ref="test_small_dense.cpp:44-210")
    # ---------------- reduced BASELINE configurations (h^2-scaled stencils)
    stencil_case("C1_somin_s4_k2_128", "somin", 2, 128, 10.0, dict(s=4, k=2, max_iterations=200), rel_tol=1e-8,
                 ref_source="BASELINE configs[0]")
    stencil_case("C1op_sgmres_s2_m5_128", "sgmres", 2, 128, 10.0, dict(s=2, m=5), rel_tol=1e-8,
                 ref_source="SURVEY 8(c) strict s-GMRES anchor 2-GMRES(5)")
    stencil_case("C2shape_sgmres_s4_m10_64", "sgmres", 2, 64, 50.0, dict(s=4, m=10), rel_tol=1e-8,
                 ref_source="BASELINE configs[1] at 64^2")
    for s in (1, 2, 4):
        stencil_case(f"C3shape_somin_s{s}_k2_24", "somin", 3, 24, 20.0, dict(s=s, k=2, tol=0.0, max_iterations=60),
                     ref_source="BASELINE configs[2] at 24^3, 60 fixed s-steps")
    stencil_case("C3shape_somin_s8_k2_16", "somin", 3, 16, 20.0, dict(s=8, k=2, tol=0.0, max_iterations=20),
                 ref_source="BASELINE configs[2] s=8 at 16^3 (breakdown class)")
    stencil_case("C4shape_sgmres_s8_m8_64", "sgmres", 2, 64, 50.0, dict(s=8, m=8, tol=0.0, max_iterations=64),
                 ref_source="BASELINE configs[3] at 64^2 (breakdown class)")
    stencil_case("C5shape_somin_s8_k2_16vark", "somin", 3, 16, 20.0, dict(s=8, k=2, tol=0.0, max_iterations=10),
                 ref_source="BASELINE configs[4] at 16^3, variable k", variable_k=True)
    stencil_case("C5shape_somin_s2_k2_16vark", "somin", 3, 16, 20.0, dict(s=2, k=2, tol=0.0, max_iterations=40),
                 ref_source="variable-k operator, s=2 (converging class)", variable_k=True)

    with open(os.path.join(OUT, "manifest.json"), "w") as fh:
        json.dump(manifest, fh, indent=1, sort_keys=True)
    print(f"wrote {len(manifest)} golden cases to {OUT}")


if __name__ == "__main__":
    main()
