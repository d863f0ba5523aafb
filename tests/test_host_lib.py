"""CPU-only checks of the product library: it loads, exports exactly the C ABI declared in
include/skrylov_b200.h, its host small-dense code (the same source that runs inside the
scalar kernels) reproduces the reference bit for bit, and GPU calls fail loudly without a
GPU (no CPU fallback)."""
import os
import re

import numpy as np
import pytest

from golden_util import MANIFEST

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lib():
    from paper_2001_04886_b200 import _lib
    return _lib


def test_library_exports_every_declared_symbol():
    L = _lib().lib()
    header = open(os.path.join(ROOT, "include", "skrylov_b200.h")).read()
    declared = set(re.findall(r"\b(skc_[a-z_0-9]+)\s*\(", header))
    assert declared, "no declarations parsed"
    for name in sorted(declared):
        assert hasattr(L, name), name
    assert declared == set(_lib().EXPORTS)


def test_version_string():
    assert b"sm_100a" in _lib().lib().skc_version()


def test_gpu_call_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2001_04886_b200 import Context, CudaError
    with pytest.raises(CudaError):
        Context(0)


def test_host_gram_solver_matches_reference_bitwise():
    from paper_2001_04886_b200 import BreakdownError, gram_solve
    for nm, g in MANIFEST["small_dense"]["gram"].items():
        w = np.array(g["w"])
        rhs = None if g["rhs"] is None else np.array(g["rhs"])
        if g["error"] is not None:
            with pytest.raises(BreakdownError) as ei:
                gram_solve(w, rhs)
            assert str(ei.value) == g["error"], nm
            continue
        x, ldlt, piv = gram_solve(w, rhs)
        assert np.array_equal(x, np.array(g["x"])), nm
        assert ldlt == g["ldlt"], nm
        assert np.array_equal(piv, np.array(g["pivots"])), nm


def test_host_cholesky_and_hessenberg_match_reference_bitwise():
    from paper_2001_04886_b200 import BreakdownError, cholesky_upper, hessenberg_lsq
    sd = MANIFEST["small_dense"]
    assert np.array_equal(cholesky_upper(np.array(sd["chol"]["w"])), np.array(sd["chol"]["r"]))
    with pytest.raises(BreakdownError) as ei:
        cholesky_upper(np.array([[1.0, 2.0], [2.0, 1.0]]))
    assert str(ei.value) == sd["chol_indef"]["error"]
    y, res = hessenberg_lsq(np.array(sd["lsq"]["g"]), sd["lsq"]["beta"])
    assert np.array_equal(y, np.array(sd["lsq"]["y"])) and res == sd["lsq"]["residual"]
    with pytest.raises(BreakdownError) as ei:
        hessenberg_lsq(np.array(sd["lsq_deficient"]["g"]), 1.0)
    assert str(ei.value) == sd["lsq_deficient"]["error"]
    with pytest.raises(ValueError):
        hessenberg_lsq(np.zeros((2, 2)), 1.0)  # rows must exceed cols


def test_rhs_generator_matches_oracle():
    from oracle import Oracle
    from paper_2001_04886_b200 import splitmix64_uniform
    o = Oracle("port")
    for seed, n, off in [(1, 10, 0), (20010486, 1000, 0), (7, 500, 12345)]:
        assert np.array_equal(splitmix64_uniform(seed, n, off), o.uniform(seed, n, off))
    u = splitmix64_uniform(3, 100000)
    assert u.min() >= -1.0 and u.max() < 1.0 and abs(u.mean()) < 0.01


def test_operator_coefficients():
    from paper_2001_04886_b200 import convection_diffusion
    st = convection_diffusion(2, 128, 10.0)
    h = 1.0 / 129.0
    assert st.coef[3] == 4.0 and st.coef[2] == -1.0 - 10.0 * h / 2.0 and st.coef[4] == -1.0 + 10.0 * h / 2.0
    st3 = convection_diffusion(3, 256, 20.0)
    assert st3.coef[3] == 6.0 and st3.n == 256 ** 3


def test_lognormal_field_matches_oracle_generator():
    """The product's k-field generator (skc_fill_lognormal) gives the oracle's bits."""
    from oracle import Oracle
    from paper_2001_04886_b200.problems import lognormal_k
    a = lognormal_k(4886, 5000)
    b = Oracle("port").lognormal(4886, 5000)
    assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
