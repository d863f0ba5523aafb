"""Op-count accounting (accounting.hpp:54-191; the driver's run_audit, bench.hpp:126-143).

CPU: the Python (paper_2001_04886_b200.accounting) and C++ (include/skrylov_b200/accounting.hpp)
predictions, slacks and audit verdicts against the reference's own outputs
(tests/golden/accounting.json, written by make_golden_accounting.py from oracle/_ref), plus the
published points test_accounting.cpp:28-55 checks.  GPU: the device solvers' op histories on the
reference tests' problem equal the reference's, and audit to the same verdicts.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2001_04886_b200 import accounting as acc

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "accounting.json")))
PRED = {0: lambda a: acc.predicted_omin(*a), 1: lambda a: acc.predicted_gmres(*a).gmres,
        2: lambda a: acc.predicted_gmres(*a).sgmres, 3: lambda a: acc.somin_audit_slack(*a),
        4: lambda a: acc.gmres_audit_slack(), 5: lambda a: acc.sgmres_audit_slack(*a)}
MODES = {0: acc.AuditMode.exact, 1: acc.AuditMode.bounded, 2: acc.AuditMode.off}


def _verdict(v):
    return dict(ok=v.ok, matvecs_exact=v.matvecs_exact, dotprods_exact=v.dotprods_exact,
                updates_exact=v.updates_exact, diffs=list(v.diffs))


def test_published_points():
    """test_accounting.cpp:28-55."""
    c1 = acc.predicted_omin(4, 4, 1)
    assert (c1[acc.DOT], c1[acc.UPD], c1[acc.MV]) == (6, 10, 1)
    c2 = acc.predicted_omin(2, 2, 2)
    assert (c2[acc.DOT], c2[acc.MV]) == (11, 2)
    assert acc.predicted_omin(0, 1, 1)[acc.DOT] == 2
    p1 = acc.predicted_gmres(10, 1)
    assert (p1.gmres[acc.DOT], p1.gmres[acc.MV]) == (65, 11)
    assert acc.predicted_gmres(5, 2).sgmres[acc.MV] == 12
    assert acc.predicted_gmres(1, 1).gmres[acc.DOT] == 2


def test_predictions_match_reference():
    for p in GOLD["predict"]:
        assert list(PRED[p["kind"]](p["args"])) == p["out"], p


@pytest.mark.parametrize("case", GOLD["audit"], ids=[a["name"] for a in GOLD["audit"]])
def test_audit_matches_reference(case):
    v = acc.audit(case["hist"], case["steady"], tuple(case["predicted"]), MODES[case["mode"]], tuple(case["slack"]))
    assert _verdict(v) == case["verdict"]


def test_audit_mode_parsing_and_run_audit_dispatch():
    """bench.hpp:252-256 (strings) and :126-143 (which table each method is audited against)."""
    assert acc.AuditMode.parse("exact") is acc.AuditMode.exact
    assert acc.AuditMode.parse("bounded") is acc.AuditMode.bounded
    assert acc.AuditMode.parse("anything") is acc.AuditMode.off

    class Rep:
        op_history = [(0, 0, 0, 0, 0), (0, 6, 0, 0, 0)]
        steady_iteration = 0
    assert acc.run_audit(Rep, "sgmres", s=2, m=2, mode="bounded").ok  # s(m+1) = 6 matvecs per cycle
    assert not acc.run_audit(Rep, "sgmres", s=1, m=2, mode="bounded").ok  # s = 1: GMRES(m) table, 3 matvecs
    assert acc.run_audit(Rep, "smr", s=2, mode="bounded") is None
    assert acc.run_audit(Rep, "sgmres", s=2, m=2, mode="off") is None


def _cxx_exe(tmp_path):
    exe = os.path.join(str(tmp_path), "accounting_check")
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "accounting_check.cpp"), "-o", exe], check=True)
    return exe


def test_cxx_header_matches_reference(tmp_path):
    exe = _cxx_exe(tmp_path)
    lines = []
    for p in GOLD["predict"]:
        a = list(p["args"]) + [0] * (3 - len(p["args"]))
        lines.append(f"P {p['kind']} {a[0]} {a[1]} {a[2]}")
    for c in GOLD["audit"]:
        rows = " ".join(" ".join(str(v) for v in r) for r in c["hist"])
        lines.append(f"A {len(c['hist'])} {c['steady']} {c['mode']} {' '.join(map(str, c['predicted']))} "
                     f"{' '.join(map(str, c['slack']))} {rows}")
    out = subprocess.run([exe], input="\n".join(lines) + "\n", capture_output=True, text=True, check=True)
    it = iter(out.stdout.splitlines())
    for p in GOLD["predict"]:
        assert [int(v) for v in next(it).split()] == p["out"], p
    for c in GOLD["audit"]:
        ok, mv, dp, up, nd = (int(v) for v in next(it).split())
        got = dict(ok=bool(ok), matvecs_exact=bool(mv), dotprods_exact=bool(dp), updates_exact=bool(up),
                   diffs=[next(it) for _ in range(nd)])
        assert got == c["verdict"], c["name"]


# ------------------------------------------------------------------ GPU
DEVICE_SOLVES = [s for s in GOLD["solves"] if s["method"] != "omin"]  # (standard Orthomin has no device path)


@pytest.mark.gpu
@pytest.mark.parametrize("case", DEVICE_SOLVES, ids=[s["name"] for s in DEVICE_SOLVES])
def test_device_solves_audit_like_reference(case):
    """test_accounting.cpp:80-133 on the GPU: the device solvers record the reference's op
    history interval for interval, and the driver's audit gives the reference's verdict."""
    from paper_2001_04886_b200 import Context, SolverConfig, SStepConfig, gmres_solve, sgmres_solve, somin_solve
    pr = GOLD["problem"]
    op = Context(0).csr(np.array(pr["offs"], np.uint64), np.array(pr["cols"], np.uint64), np.array(pr["vals"]))
    x = np.array(pr["x0"])
    cfg = case["cfg"]
    if case["method"] == "gmres":
        rep = gmres_solve(op, np.array(pr["rhs"]), x, SolverConfig(method="gmres", **cfg))
    else:
        fn = somin_solve if case["method"] == "somin" else sgmres_solve
        rep = fn(op, np.array(pr["rhs"]), x, SStepConfig(**cfg))
    assert rep.iterations == case["iterations"] and rep.converged == case["converged"]
    assert [list(h) for h in rep.op_history] == case["op_history"]
    assert rep.steady_iteration == case["steady"]
    v = acc.audit(rep.op_history, rep.steady_iteration, tuple(case["predicted"]), MODES[case["mode"]],
                  tuple(case["slack"]))
    assert _verdict(v) == case["verdict"] and v.ok and v.matvecs_exact
    s = cfg.get("s", 1)
    v2 = acc.run_audit(rep, case["method"], s=s, k=cfg.get("k", 0), m=cfg.get("m", 0), mode="bounded")
    assert _verdict(v2) == case["verdict"]
