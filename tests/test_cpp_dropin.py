"""The C++ drop-in header (include/skrylov_b200/sstep.hpp) compiles and links against the
library on CPU; on a GPU it solves like a reference caller would."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2001_04886_b200")


def build(tmp_path):
    exe = os.path.join(str(tmp_path), "drop_in")
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "drop_in.cpp"), "-L", LIBDIR, "-lskrylov_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_drop_in_header_builds(tmp_path):
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_drop_in_solves(tmp_path):
    exe = build(tmp_path)
    out = json.loads(subprocess.run([exe, "64"], check=True, capture_output=True, text=True).stdout)
    assert out["somin_converged"] and out["sgmres_converged"] and out["invalid_s_throws"]
    assert out["somin_true_residual"] <= out["tol"] * (1 + 1e-6)


def build_ref_caller(tmp_path):
    exe = os.path.join(str(tmp_path), "ref_caller")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "ref_caller.cpp"), "-L", LIBDIR, "-lskrylov_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_reference_style_caller_builds(tmp_path):
    """Caller code in the reference's namespace and types (skrylov::SparseMatrix, as_operator,
    LinearOperator, SStepBasis with DirectionBlock / Matrix, a dispatch_method-style
    dispatcher) compiles unchanged against include/skrylov_b200/skrylov.hpp."""
    assert os.path.exists(build_ref_caller(tmp_path))


@pytest.mark.gpu
def test_reference_style_caller_solves(tmp_path):
    exe = build_ref_caller(tmp_path)
    out = json.loads(subprocess.run([exe, "48"], check=True, capture_output=True, text=True).stdout)
    for m in ("somin", "sgcr", "sgmres", "smr"):
        assert out[m]["converged"], m
        assert out[m]["true_residual"] <= out["tol"] * (1 + 1e-6), m
    assert out["smr_step"]["coeffs"] == 3 and out["smr_step"]["matvecs"] == 3
    sa = out["sarnoldi"]
    assert (sa["blocks"], sa["width"], sa["hess_rows"], sa["hess_cols"]) == (4, 3, 15, 12)
    assert sa["avug_rel"] <= 1e-8 and sa["gram0_trace"] > 0.0
    assert out["host_closure_rejected"] and out["invalid_s_throws"]
