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
