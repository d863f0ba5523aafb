"""The benchmark driver layer (bench.hpp, matrix_market.hpp, problem.hpp) around the device
solvers: the paper problem's assembly, run configurations, Matrix Market I/O, the sweep and its
report emission.  Modelled on test_bench.cpp; the sweep's cells are checked against the
reference driver's own run of them (tests/golden/sweep.json, make_golden_sweep.py).
"""
import json
import os

import numpy as np
import pytest

from golden_util import case
from paper_2001_04886_b200 import accounting as acc
from paper_2001_04886_b200 import sweep as sw

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "sweep.json")))


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def small_sweep_config():
    """test_bench.cpp:29-42."""
    return sw.parse_run_config({
        "problem": {"nx": [5, 7], "beta": 1.0, "gamma": 50.0},
        "methods": [{"method": "omin", "s": 1, "k": 4, "precond": "ilu0"},
                    {"method": "somin", "s": 2, "k": 2, "precond": "ilu0"},
                    {"method": "gmres", "s": 1, "m": 10, "precond": "ilu0"},
                    {"method": "sgmres", "s": 2, "m": 5, "precond": "ilu0"}],
        "termination": 1e-6, "audit": "bounded"})


# ------------------------------------------------------------------ CPU
def test_discretize_bit_identical_to_reference():
    """problem.hpp:129-203 assembled by the library (skc_discretize) against the reference's
    arrays at nx = 7 (accounting.json), 16 and 64 (the ILU(0) and driver fixtures)."""
    from paper_2001_04886_b200 import discretize
    pr = json.load(open(os.path.join(ROOT, "tests", "golden", "accounting.json")))["problem"]
    p = discretize(7)
    assert np.array_equal(p.row_offsets, np.array(pr["offs"], np.uint64))
    assert np.array_equal(p.col_indices, np.array(pr["cols"], np.uint64))
    for got, want in ((p.values, pr["vals"]), (p.rhs, pr["rhs"]), (p.x0, pr["x0"])):
        assert np.array_equal(_bits(got), _bits(np.array(want)))
    for nx in (16, 64):
        meta, arr = case(f"ilu0_T61_nx{nx}")
        p = discretize(nx)
        assert np.array_equal(p.row_offsets, arr["offs"]) and np.array_equal(p.col_indices, arr["cols"])
        assert np.array_equal(_bits(p.values), _bits(arr["vals"]))
    meta, arr = case("solve_linear_sgmres_s2_m5_T61_nx64_ilu0")
    p = discretize(64)
    assert np.array_equal(_bits(p.rhs), _bits(arr["f"])) and np.array_equal(_bits(p.x0), _bits(arr["x0"]))
    # the analytic solution is what the discretization converges to (second order)
    assert np.abs(p.u_true).max() > 0.1
    with pytest.raises(ValueError, match="nx must be at least 1"):
        discretize(0)


def test_method_labels_and_run_config():
    """bench.hpp:43-71, :208-258; test_bench.cpp:192-199 (validation)."""
    rc = small_sweep_config()
    assert [m.label() for m in rc.methods] == ["s=1,k=4", "s=2,k=2", "s=1,m=10", "s=2,m=5"]
    assert [m.k_or_m() for m in rc.methods] == [4, 2, 10, 5]
    assert all(m.precondition for m in rc.methods) and rc.settings.audit is acc.AuditMode.bounded
    assert rc.problems == [(5, 1.0, 50.0), (7, 1.0, 50.0)]
    assert sw.MethodSpec("smr", s=3).label() == "s=3,mr" and sw.MethodSpec("sgcr", s=2).label() == "s=2,gcr"
    assert sw.parse_method({"method": "gmres", "precond": True}).precondition
    assert not sw.parse_method({"method": "gmres", "precond": "none"}).precondition
    with pytest.raises(ValueError, match="at least one method"):
        sw.parse_run_config({"problem": {"nx": 5}, "methods": []})
    with pytest.raises(ValueError, match="must be positive"):
        sw.parse_run_config({"problem": {"nx": 5}, "methods": [{"method": "gmres"}], "termination": -1.0})


def _cell(label, method, s=1, **rep):
    from paper_2001_04886_b200 import SolveReport
    return sw.CellResult(problem_label=label, method=sw.MethodSpec(method, s=s),
                         outcome=sw.SolveOutcome(report=SolveReport(**rep)))


def test_table_markers_and_layout():
    """bench.hpp:303-361; test_bench.cpp:145-160 (DIV / ERR markers)."""
    div = _cell("9", "omin", converged=False, iterations=17, breakdown="divergence: residual grew beyond 10x")
    err = sw.CellResult(problem_label="9", method=sw.MethodSpec("gmres"), error="assembly failed")
    t = sw.emit_table_text([div, err], "iterations")
    # std::setw(wid) left-aligned, wid = max(9, longest label + 2) = 10
    assert t.splitlines()[0] == "dimension | s=1,k=4   | s=1,m=10  "
    assert t.splitlines()[1] == "9         | DIV(17)   | ERR       "
    assert "cells: iterations\n" in t and "-- missing cell." in t
    brk = _cell("9", "somin", s=2, converged=False, iterations=4, breakdown="gram matrix singular")
    cap = _cell("11", "somin", s=2, converged=False, iterations=100)
    ok = _cell("11", "omin", converged=True, iterations=12, op_counts=(1, 13, 2, 3, 4))
    t = sw.emit_table_text([brk, cap, ok], "opcounts")
    lines = t.splitlines()
    assert lines[1].split("|")[1].strip() == "BRK(4)" and lines[2].split("|")[1].strip() == "MAX(100)"
    assert lines[2].split("|")[2].strip() == "13" and lines[1].split("|")[2].strip() == "--"
    assert "cells: operator applications (matvecs)" in t


def test_csv_and_json_schema():
    """bench.hpp:364-429; test_bench.cpp:120-133."""
    ok = _cell("7", "sgmres", converged=True, iterations=10, cycles=1, op_counts=(114, 14, 78, 16, 3),
               final_residual=0.1, residual_history=[1.0, 0.1])
    err = sw.CellResult(problem_label="7", method=sw.MethodSpec("omin"), error="no device path")
    csv = sw.emit_table_csv([ok, err])
    lines = csv.splitlines()
    assert lines[0] == ("nx,method,s,k_or_m,preconditioned,iterations,matvecs,dotprods,updates,"
                        "final_residual,converged,breakdown")
    assert lines[1] == "7,sgmres,1,10,0,10,14,114,78,0.10000000000000001,1,"
    assert lines[2] == "7,omin,1,4,0,,,,,,0,no device path"
    assert csv.count("\n") == 3
    j = sw.report_to_json(ok)
    assert list(j) == ["nx", "problem", "method", "s", "k_or_m", "preconditioned", "iterations", "cycles",
                       "matvecs", "dotprods", "updates", "termination_dots", "stored_vectors", "final_residual",
                       "converged", "breakdown", "fallback_cycles", "residual_history", "audit"]
    assert j["audit"] is None and j["matvecs"] == 14 and j["stored_vectors"] == 16
    assert sw.report_to_json(err) == {"nx": 0, "problem": "7", "method": "omin", "s": 1, "k_or_m": 4,
                                      "preconditioned": False, "error": "no device path"}


def test_matrix_market_round_trip_and_errors(tmp_path):
    from paper_2001_04886_b200 import discretize
    p = discretize(5)
    path = str(tmp_path / "a.mtx")
    sw.write_matrix_market(path, p.row_offsets, p.col_indices, p.values)
    offs, cols, vals = sw.read_matrix_market(path)
    assert np.array_equal(offs, p.row_offsets) and np.array_equal(cols, p.col_indices)
    assert np.array_equal(_bits(vals), _bits(p.values))
    bad = tmp_path / "b.mtx"
    for text, msg in (("%%MatrixMarket matrix array real general\n", "expected 'matrix coordinate"),
                      ("%%MatrixMarket matrix coordinate real general\n% c\n2 2 1\n3 1 1.0\n", "out of range"),
                      ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n1 1 2.0\n", "duplicate"),
                      ("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n", "truncated")):
        bad.write_text(text)
        with pytest.raises(ValueError, match=msg):
            sw.read_matrix_market(str(bad))


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_sweep_matches_reference_driver():
    """test_bench.cpp:94-118 on the device: the cells with a device path reproduce the reference
    driver's run (iterations, op counters and history exactly, residuals to 1e-9), audit clean;
    the standard Orthomin cells are error cells; repeated sweeps give identical reports."""
    from paper_2001_04886_b200 import Context
    ctx = Context(0)
    rc = small_sweep_config()
    cells = sw.run_sweep(ctx, rc)
    assert len(cells) == 8
    gold = {(c["nx"], c["method"]): c for c in GOLD["cells"]}
    for c in cells:
        if c.method.method == "omin":
            assert c.error and "no device path" in c.error
            continue
        assert not c.error, c.error
        g = gold[(c.nx, c.method.method)]
        rep = c.outcome.report
        assert rep.iterations == g["iterations"] and rep.converged == g["converged"]
        assert list(rep.op_counts) == g["op_counts"]
        assert [list(h) for h in rep.op_history] == g["op_history"]
        assert abs(rep.final_residual - g["final_residual"]) <= 1e-9 * max(1.0, g["final_residual"]) + 1e-12
        assert c.outcome.audit is not None and c.outcome.audit.ok
    t = sw.emit_table_text(cells, "iterations")
    assert "s=1,k=4" in t and "s=2,k=2" in t and "s=1,m=10" in t and "s=2,m=5" in t
    assert "\n5 " in t and "\n7 " in t
    again = sw.run_sweep(ctx, rc)
    strip = lambda j: {k: v for k, v in j.items() if k != "residual_history"}  # noqa: E731
    for a, b in zip(cells, again):
        assert strip(sw.report_to_json(a)) == strip(sw.report_to_json(b))
    assert sw.emit_table_csv(cells).count("\n") == len(cells) + 1


@pytest.mark.gpu
def test_external_matrix_market_problem(tmp_path):
    """test_bench.cpp:173-190."""
    from paper_2001_04886_b200 import Context, discretize
    p = discretize(5)
    path = str(tmp_path / "ext.mtx")
    sw.write_matrix_market(path, p.row_offsets, p.col_indices, p.values)
    rc = sw.parse_run_config({"problem": {"matrix_market": path},
                              "methods": [{"method": "gmres", "m": 10, "precond": "ilu0"}], "termination": 1e-8})
    cells = sw.run_sweep(Context(0), rc)
    assert len(cells) == 1 and not cells[0].error and cells[0].outcome.report.converged
