"""Op-count accounting: the published per-iteration / per-cycle vector-operation costs of the
methods and the audit of a report's counter deltas against them (accounting.hpp:54-191).

Counters are 5-tuples in report.hpp:35-41 order: (dotprods, matvecs, vec_updates,
stored_vectors, termination_dots) -- the layout of SolveReport.op_counts / op_history.
Arithmetic follows the reference's std::size_t: unsigned 64-bit, differences wrap.
Termination inner products are never audited (they are tallied separately by the solvers).
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field

_MASK = (1 << 64) - 1
DOT, MV, UPD, STORED, TERM = range(5)


class AuditMode(enum.Enum):
    exact = 0
    bounded = 1
    off = 2

    @classmethod
    def parse(cls, v) -> "AuditMode":
        """An AuditMode, or the run-config string (bench.hpp:252-256: anything but "exact" /
        "bounded" is off)."""
        if isinstance(v, AuditMode):
            return v
        return {"exact": cls.exact, "bounded": cls.bounded}.get(v, cls.off)


def _counter(dotprods=0, matvecs=0, vec_updates=0, stored_vectors=0, termination_dots=0) -> tuple:
    return (dotprods & _MASK, matvecs & _MASK, vec_updates & _MASK, stored_vectors & _MASK,
            termination_dots & _MASK)


def counter_delta(a, b) -> tuple:
    """report.hpp:43-51 `a - b`: wrapping differences, stored_vectors taken from a (a peak)."""
    return ((a[DOT] - b[DOT]) & _MASK, (a[MV] - b[MV]) & _MASK, (a[UPD] - b[UPD]) & _MASK, a[STORED],
            (a[TERM] - b[TERM]) & _MASK)


def predicted_omin(j: int, k: int, s: int) -> tuple:
    """accounting.hpp:54-70: cost of iteration j of (s-)Orthomin(k).  s = 1 in steady state
    (j >= k) is the classic k+2 dots / 2k+2 updates / 1 Mv; otherwise the table's formulas."""
    s2, tri = s * s, s * (s + 1) // 2
    if s == 1 and j >= k:
        dots, upd = k + 2, 2 * k + 2
    else:
        dots = min((j + 1) * s2 + tri, k * s2 + tri)
        upd = min(2 * (j + 1) * s2 + s, 2 * k * s2 + tri)
    return _counter(dots, s, upd, 2 * k * s + s + 1)


@dataclass(frozen=True)
class PredictedGmresCosts:
    gmres: tuple   # one cycle of GMRES(s m)
    sgmres: tuple  # one cycle of s-GMRES(m)


def predicted_gmres(m: int, s: int) -> PredictedGmresCosts:
    """accounting.hpp:77-92: published one-cycle costs of GMRES(sm) and s-GMRES(m)."""
    ms = m * s
    g = _counter(ms + ms * (ms + 1) // 2, ms + 1, (ms * ms + ms) // 2 + 2 * ms, ms + 1)
    sg = _counter(m * (m - 1) * s * s // 2 + s * (s + 1) // 2 + s, s * (m + 1), m * (m + 1) * s * s,
                  s * (m + 1) * m // 2 + m)
    return PredictedGmresCosts(g, sg)


def somin_audit_slack(s: int) -> tuple:
    """accounting.hpp:97-102: the (A P)^T r dots and the folded block updates, per iteration."""
    return _counter(dotprods=s, vec_updates=2 * s)


def gmres_audit_slack() -> tuple:
    """accounting.hpp:106-111: cycle-leading scaling and restart subtraction, per cycle."""
    return _counter(vec_updates=2)


def sgmres_audit_slack(m: int, s: int) -> tuple:
    """accounting.hpp:116-132: the margin of explicit Gram products, the cross-block safeguard
    and one worst-case reorthogonalization pass over the published dot count, per cycle."""
    tri = s * (s + 1) // 2
    mine = s * m * (m + 1) // 2 + m
    mine += m * tri
    mine += (2 * s * (s - 1) + s * s) * (m - 1) * m // 2 + (m - 1) * s
    table = m * (m - 1) * s * s // 2 + tri + s
    return _counter(dotprods=mine - table if mine > table else 0, vec_updates=2)


@dataclass
class AuditReport:
    """accounting.hpp:134-140."""
    ok: bool = True
    matvecs_exact: bool = True
    dotprods_exact: bool = True
    updates_exact: bool = True
    diffs: list = field(default_factory=list)


def audit(op_history, steady_iteration: int, predicted, mode=AuditMode.exact, slack=(0, 0, 0, 0, 0)) -> AuditReport:
    """accounting.hpp:149-191: check the counter deltas of op_history against a per-interval
    prediction.  Intervals before steady_iteration (growing window) need only stay at or below
    the prediction; steady ones match exactly (exact mode) or stay within prediction + slack
    (bounded mode).  Operator applications are exact in every mode.  `op_history` is a
    SolveReport's list of 5-tuples (or anything indexable the same way)."""
    mode = AuditMode.parse(mode)
    out = AuditReport()
    hist = [tuple(int(v) for v in row) for row in op_history]
    if mode is AuditMode.off or len(hist) < 2:
        return out
    p = predicted

    def complain(iv, name, got, want, rel):
        out.ok = False
        out.diffs.append(f"interval {iv}: {name} {got} {rel} {want}")

    for t in range(1, len(hist)):
        d = counter_delta(hist[t], hist[t - 1])
        iv = t - 1
        steady = iv >= steady_iteration
        if d[MV] != p[MV]:
            out.matvecs_exact = False
        if steady:
            if d[DOT] != p[DOT]:
                out.dotprods_exact = False
            if d[UPD] != p[UPD]:
                out.updates_exact = False
        if mode is AuditMode.exact:
            rel = "!=" if steady else ">"
            bad = (lambda g, w: g != w) if steady else (lambda g, w: g > w)
            if bad(d[DOT], p[DOT]):
                complain(iv, "dotprods", d[DOT], p[DOT], rel)
            if bad(d[UPD], p[UPD]):
                complain(iv, "vec_updates", d[UPD], p[UPD], rel)
        else:
            wd, wu = (p[DOT] + slack[DOT]) & _MASK, (p[UPD] + slack[UPD]) & _MASK
            if d[DOT] > wd:
                complain(iv, "dotprods", d[DOT], wd, ">")
            if d[UPD] > wu:
                complain(iv, "vec_updates", d[UPD], wu, ">")
        if d[MV] != p[MV]:
            complain(iv, "matvecs", d[MV], p[MV], "!=")
    return out


def run_audit(report, method: str, s: int = 1, k: int = 0, m: int = 0, mode=AuditMode.bounded):
    """bench.hpp:126-143: the prediction and slack the driver audits each method against;
    None for mode off and for the methods without a published table (mr, smr, gcr, sgcr)."""
    mode = AuditMode.parse(mode)
    if mode is AuditMode.off:
        return None
    if method == "omin":
        pred, sl = predicted_omin(k, k, 1), somin_audit_slack(1)
    elif method == "somin":
        pred, sl = predicted_omin(k, k, s), somin_audit_slack(s)
    elif method == "gmres" or (method == "sgmres" and s <= 1):  # s = 1 shares the GMRES path
        pred, sl = predicted_gmres(m, 1).gmres, gmres_audit_slack()
    elif method == "sgmres":
        pred, sl = predicted_gmres(m, s).sgmres, sgmres_audit_slack(m, s)
    else:
        return None
    return audit(report.op_history, report.steady_iteration, pred, mode, sl)
