"""Pin the CPU oracle (oracle/skrylov_oracle.c, a restatement) to the reference.

* against tests/golden (generated from the unmodified reference): always;
* against oracle/_ref/libskref.so live, when it was built here.
Bit-exact equality is required: the restatement follows the reference's arithmetic order.
"""
import numpy as np
import pytest

from golden_util import MANIFEST, case, matrix, names
from oracle import Oracle, OracleError

PORT = Oracle("port")
HAVE_REF = Oracle.available("reference")


def _run(orc, meta, arr):
    a = matrix(arr)
    cfg = dict(meta["cfg"])
    if meta["kind"] == "sstep":
        return orc.sstep(meta["method"], a, arr["f"], arr["x0"], **cfg)
    return orc.standard(meta["method"], a, arr["f"], arr["x0"], **cfg)


@pytest.mark.parametrize("name", names("solve"))
def test_port_matches_golden_solve(name):
    meta, arr = case(name)
    res = _run(PORT, meta, arr)
    assert np.array_equal(np.array(res.residual_history), arr["history"])
    assert np.array_equal(res.x, arr["x"])
    assert np.array_equal(np.array(res.op_history, dtype=np.uint64).reshape(-1, 5), arr["op_history"])
    assert tuple(int(v) for v in arr["op_counts"]) == res.op_counts
    assert res.iterations == meta["iterations"] and res.cycles == meta["cycles"]
    assert res.converged == meta["converged"]
    assert res.breakdown == meta["breakdown"]
    assert res.fallback_cycles == meta["fallback_cycles"]
    assert res.notes == meta["notes"]
    assert res.steady_iteration == meta["steady_iteration"]


@pytest.mark.parametrize("name", names("sarnoldi"))
def test_port_matches_golden_sarnoldi(name):
    meta, arr = case(name)
    b = PORT.sarnoldi(matrix(arr), arr["v1"], meta["s"], meta["m_blocks"])
    for key in ("blocks", "grams", "hess", "next_seed"):
        assert np.array_equal(b[key], arr[key]), key
    assert b["next_seed_norm"] == meta["next_seed_norm"]
    assert list(b["counter"]) == meta["counter"]


@pytest.mark.parametrize("name", names("smr_step"))
def test_port_matches_golden_smr_step(name):
    meta, arr = case(name)
    x, r, co, cnt = PORT.smr_step(matrix(arr), arr["x0"], arr["r0"], meta["s"])
    assert np.array_equal(x, arr["x"]) and np.array_equal(r, arr["r"]) and np.array_equal(co, arr["coeffs"])
    assert list(cnt) == meta["counter"]


def test_port_matches_golden_krylov_block():
    meta, arr = case("krylov_block_nx3_s4")
    a = matrix(arr)
    kb = PORT.krylov_block(a, arr["v"], meta["s"])
    assert np.array_equal(kb, arr["blocks"])
    for j in range(meta["s"] - 1):  # test_block.cpp:49-60: each column is spmv of the previous, bit-exactly
        assert np.array_equal(kb[j + 1], PORT.spmv(a, kb[j]))


def test_port_matches_golden_small_dense():
    sd = MANIFEST["small_dense"]
    for nm, g in sd["gram"].items():
        w = np.array(g["w"])
        rhs = None if g["rhs"] is None else np.array(g["rhs"])
        if g["error"] is not None:
            with pytest.raises(OracleError) as ei:
                PORT.gram_solve(w, rhs)
            assert str(ei.value) == g["error"], nm
            continue
        x, ldlt, piv = PORT.gram_solve(w, rhs)
        assert np.array_equal(x, np.array(g["x"])), nm
        assert ldlt == g["ldlt"] and np.array_equal(piv, np.array(g["pivots"])), nm
    y, res = PORT.hessenberg_lsq(np.array(sd["lsq"]["g"]), sd["lsq"]["beta"])
    assert np.array_equal(y, np.array(sd["lsq"]["y"])) and res == sd["lsq"]["residual"]
    with pytest.raises(OracleError) as ei:
        PORT.hessenberg_lsq(np.array(sd["lsq_deficient"]["g"]), 1.0)
    assert str(ei.value) == sd["lsq_deficient"]["error"]
    assert np.array_equal(PORT.cholesky_upper(np.array(sd["chol"]["w"])), np.array(sd["chol"]["r"]))
    with pytest.raises(OracleError) as ei:
        PORT.cholesky_upper(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert str(ei.value) == sd["chol_indef"]["error"]


def test_reference_kats_hold_in_golden():
    """The reference's own cross-method KATs, evaluated on the golden outputs."""
    from golden_util import rel_diff
    # somin(s=1,k=4) == omin(4)  (test_sstep.cpp:151-189, 1e-12)
    a = case("somin_s1_k4_nx7")[1]["history"]
    b = case("omin_k4_nx7")[1]["history"]
    assert len(a) == len(b) and all(rel_diff(u, v) <= 1e-12 for u, v in zip(a, b))
    # sgmres(s=1) == gmres (:313-336, 1e-10)
    a = case("sgmres_s1_m5_nx7")[1]["history"]
    b = case("gmres_m5_nx7")[1]["history"]
    assert len(a) == len(b) and all(rel_diff(u, v) <= 1e-10 for u, v in zip(a, b))
    # Remark 4.1 (:338-368, 1e-6)
    a = case("sgmres_s2_m4_dense40")[1]["history"]
    b = case("gmres_m8_dense40")[1]["history"]
    for u, v in zip(a, b):
        if u < 1e-9 * a[0]:
            break
        assert rel_diff(u, v) <= 1e-6
    # matvec budgets (:370-405)
    oh = case("sgmres_s2_m3_nx7_budget")[1]["op_history"].astype(np.int64)
    assert all(d == 2 * 4 for d in np.diff(oh[:, 1]))
    oh = case("somin_s3_k2_nx7_budget")[1]["op_history"].astype(np.int64)
    assert all(d == 3 for d in np.diff(oh[:, 1]))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (no /root/reference here)")
@pytest.mark.parametrize("name", names("solve"))
def test_port_matches_reference_live(name):
    meta, arr = case(name)
    ref = Oracle("reference")
    r1, r2 = _run(PORT, meta, arr), _run(ref, meta, arr)
    assert r1.residual_history == r2.residual_history
    assert np.array_equal(r1.x, r2.x)
    assert r1.op_history == r2.op_history and r1.breakdown == r2.breakdown and r1.notes == r2.notes


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (no /root/reference here)")
@pytest.mark.parametrize("conv,dim,nx,variable_k", [(10.0, 2, 9, False), (20.0, 3, 5, False), (20.0, 3, 5, True)])
def test_stencil_csr_generator_consistent(conv, dim, nx, variable_k):
    """orc_stencil_apply (matrix free) == CSR spmv bitwise, both orders ascending-column."""
    from paper_2001_04886_b200.problems import convection_diffusion, splitmix64_uniform
    st = convection_diffusion(dim, nx, conv, variable_k=variable_k)
    k = PORT.lognormal(7, st.n) if variable_k else None
    a = PORT.stencil_csr(dim, st.nx, st.ny, st.nz, st.coef, kcell=k, ch2=st.ch2)
    x = splitmix64_uniform(3, st.n)
    y1 = PORT.stencil_apply(dim, st.nx, st.ny, st.nz, st.coef, x, kcell=k, ch2=st.ch2)
    assert np.array_equal(y1, PORT.spmv(a, x))
    assert np.array_equal(y1, Oracle("reference").spmv(a, x))
