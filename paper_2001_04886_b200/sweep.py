"""The reference's benchmark driver around the solvers (bench.hpp, matrix_market.hpp): run
configurations, the problem x method sweep on the GPU, and its report emission (iteration /
op-count text tables, CSV, per-cell JSON), so reference users keep their tables and scripts.

Every cell runs through `solve_linear` (ILU(0) right preconditioning, true-residual check,
op-count audit) on the device.  Methods without a device path (the standard mr / omin / gcr
solvers, outside the s-step hot path) become error cells ("ERR"), as any failing cell does in
the reference sweep.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field, replace

import numpy as np

from .accounting import AuditMode, AuditReport
from .sstep import SStepConfig, discretize, solve_linear

SSTEP_FAMILY = ("smr", "somin", "sgcr", "sgmres")


@dataclass
class MethodSpec:
    """bench.hpp:43-71."""
    method: str = ""
    s: int = 1
    k: int = 4
    m: int = 10
    precondition: bool = False

    def sstep_family(self) -> bool:
        return self.method in SSTEP_FAMILY

    def label(self) -> str:
        """Column label of the iteration table, e.g. "s=2,k=2" or "s=1,m=10"."""
        if self.method == "mr":
            return "mr"
        if self.method == "smr":
            return f"s={self.s},mr"
        if self.method in ("gcr", "sgcr"):
            return f"s={self.s},gcr"
        if self.method in ("omin", "somin"):
            return f"s={self.s},k={self.k}"
        return f"s={self.s},m={self.m}"

    def k_or_m(self) -> int:
        if self.method in ("gmres", "sgmres"):
            return self.m
        if self.method in ("mr", "smr"):
            return 0
        return self.k


@dataclass
class SolveSettings:
    """bench.hpp:73-79."""
    tol: float = 1e-6
    strict_termination: bool = False  # literal reading: ||r||_2 < tol^2
    max_iterations: int = 100000
    audit: AuditMode = AuditMode.off
    debug_checks: bool = False


@dataclass
class SolveOutcome:
    """bench.hpp:81-85."""
    x: np.ndarray | None = None
    report: object = None  # sstep.SolveReport
    audit: AuditReport | None = None


@dataclass
class CellResult:
    """bench.hpp:200-206."""
    problem_label: str = ""
    nx: int = 0  # 0 for external matrices
    method: MethodSpec = field(default_factory=MethodSpec)
    outcome: SolveOutcome | None = None
    error: str = ""


@dataclass
class RunConfig:
    """bench.hpp:193-198: problems (nx values with beta / gamma) or one Matrix Market file."""
    problems: list = field(default_factory=list)  # [(nx, beta, gamma)]
    matrix_market: str = ""
    methods: list = field(default_factory=list)
    settings: SolveSettings = field(default_factory=SolveSettings)
    output: str = ""


def _require(ok, msg):
    if not ok:
        raise ValueError(msg)


def parse_method(j: dict) -> MethodSpec:
    """bench.hpp:208-222."""
    ms = MethodSpec(method=j["method"])
    for key in ("s", "k", "m"):
        if key in j:
            setattr(ms, key, int(j[key]))
    if "precond" in j:
        p = j["precond"]
        ms.precondition = p == "ilu0" if isinstance(p, str) else bool(p)
    return ms


def parse_run_config(j: dict | str) -> RunConfig:
    """bench.hpp:224-258 (a dict, or a JSON string)."""
    if isinstance(j, str):
        j = json.loads(j)
    rc = RunConfig()
    prob = j["problem"]
    if "matrix_market" in prob:
        rc.matrix_market = prob["matrix_market"]
    else:
        beta, gamma = float(prob.get("beta", 1.0)), float(prob.get("gamma", 50.0))
        nx = prob["nx"]
        rc.problems = [(int(v), beta, gamma) for v in (nx if isinstance(nx, list) else [nx])]
    rc.methods = [parse_method(mj) for mj in j["methods"]]
    _require(len(rc.methods) > 0, "run config: at least one method required")
    if "termination" in j:
        rc.settings.tol = float(j["termination"])
    _require(rc.settings.tol > 0, "run config: termination threshold must be positive")
    if "strict_termination" in j:
        rc.settings.strict_termination = bool(j["strict_termination"])
    if "max_iterations" in j:
        rc.settings.max_iterations = int(j["max_iterations"])
    if "audit" in j:
        rc.settings.audit = AuditMode.parse(j["audit"])
    if "output" in j:
        rc.output = j["output"]
    return rc


# ------------------------------------------------------------------ Matrix Market (matrix_market.hpp)
def _read_mm(path: str):
    try:
        fh = open(path)
    except OSError:
        raise ValueError("matrix market: cannot open " + path) from None
    with fh:
        header = fh.readline()
        _require(header != "", "matrix market: empty stream")
        _require(header.split()[:5] == ["%%MatrixMarket", "matrix", "coordinate", "real", "general"],
                 "matrix market: expected 'matrix coordinate real general' header")
        line = fh.readline()
        while line and (line.rstrip("\n") == "" or line[0] == "%"):  # comments and empty lines
            line = fh.readline()
        try:
            rows, cols, nnz = (int(v) for v in line.split()[:3])
        except ValueError:
            raise ValueError("matrix market: bad size line") from None
        toks = fh.read().split()
    _require(len(toks) >= 3 * nnz, "matrix market: truncated entry list")
    ent = []
    for t in range(nnz):
        i, j, v = int(toks[3 * t]), int(toks[3 * t + 1]), float(toks[3 * t + 2])
        _require(1 <= i <= rows and 1 <= j <= cols, "matrix market: entry index out of range")
        ent.append((i - 1, j - 1, v))
    ent.sort(key=lambda e: (e[0], e[1]))
    for a, b in zip(ent, ent[1:]):
        _require((a[0], a[1]) != (b[0], b[1]), "from_triplets: duplicate entry")
    offs = np.zeros(rows + 1, np.uint64)
    for i, _, _ in ent:
        offs[i + 1] += 1
    offs = np.cumsum(offs, dtype=np.uint64)
    return rows, cols, (offs, np.array([e[1] for e in ent], np.uint64), np.array([e[2] for e in ent], np.float64))


def read_matrix_market(path: str):
    """matrix_market.hpp: a 'matrix coordinate real general' file -> (row_offsets, col_indices,
    values), entries sorted by (row, column) as from_triplets does (sparse.hpp:67-93)."""
    return _read_mm(path)[2]


def write_matrix_market(path: str, row_offsets, col_indices, values) -> None:
    """matrix_market.hpp: one 1-based 'i j %.17g' line per stored entry, rows in order."""
    n = len(row_offsets) - 1
    with open(path, "w") as out:
        out.write("%%MatrixMarket matrix coordinate real general\n")
        out.write(f"{n} {n} {len(values)}\n")
        for i in range(n):
            for p in range(int(row_offsets[i]), int(row_offsets[i + 1])):
                out.write(f"{i + 1} {int(col_indices[p]) + 1} {float(values[p]):.17g}\n")


# ------------------------------------------------------------------ the sweep
def run_cell(ctx, a, f, x0, ms: MethodSpec, st: SolveSettings) -> SolveOutcome:
    """bench.hpp:149-191 solve_linear with the cell's method spec and settings."""
    threshold = st.tol * st.tol if st.strict_termination else st.tol
    cfg = SStepConfig(s=ms.s, k=ms.k, m=ms.m, tol=threshold, max_iterations=st.max_iterations,
                      precondition=ms.precondition, debug_checks=st.debug_checks)
    audit = None if st.audit is AuditMode.off else st.audit
    x, rep = solve_linear(ctx, a[0], a[1], a[2], f, x0, ms.method, cfg, precondition=ms.precondition,
                          audit=audit)
    return SolveOutcome(x=x, report=rep, audit=rep.audit)


def run_sweep(ctx, rc: RunConfig) -> list:
    """bench.hpp:260-301: every problem x method cell on the device; failures are recorded per
    cell and the sweep continues; cells follow config order (repeatable runs give identical
    reports)."""
    inst = []
    if rc.matrix_market:
        n, ncols, a = _read_mm(rc.matrix_market)
        _require(n == ncols, "sweep: external matrix must be square")
        # manufactured unit solution f = A 1 (the device CSR product keeps spmv's row order and
        # separate rounding, so f is the reference's bit for bit)
        f = ctx.csr(*a).apply(np.ones(n))
        x0 = 0.05 * (np.arange(1, n + 1) % 50).astype(np.float64)  # initial_guess
        inst.append((rc.matrix_market, 0, a, f, x0))
    else:
        for nx, beta, gamma in rc.problems:
            p = discretize(nx, beta, gamma)
            inst.append((str(nx), nx, (p.row_offsets, p.col_indices, p.values), p.rhs, p.x0))
    cells = []
    for label, nx, a, f, x0 in inst:
        for ms in rc.methods:
            cell = CellResult(problem_label=label, nx=nx, method=replace(ms))
            try:
                cell.outcome = run_cell(ctx, a, f, x0, ms, rc.settings)
            except Exception as e:  # noqa: BLE001 -- recorded per cell, as the reference does
                cell.error = str(e)
            cells.append(cell)
    return cells


# ------------------------------------------------------------------ reports
def _cell_text(cell: CellResult, opcounts: bool) -> str:
    if cell.error:
        return "ERR"
    if cell.outcome is None:
        return "--"
    rep = cell.outcome.report
    value = rep.op_counts[1] if opcounts else rep.iterations
    if rep.converged:
        return str(value)
    if rep.breakdown and rep.breakdown.startswith("divergence"):
        return f"DIV({rep.iterations})"
    if rep.breakdown:
        return f"BRK({rep.iterations})"
    return f"MAX({rep.iterations})"


def emit_table_text(cells: list, layout: str = "iterations") -> str:
    """bench.hpp:320-361: rows = problem dimensions, columns = methods, cells = iteration counts
    ("iterations") or operator applications ("opcounts")."""
    opcounts = layout == "opcounts"
    rows, columns = [], []
    for c in cells:
        if c.problem_label not in rows:
            rows.append(c.problem_label)
        if c.method.label() not in columns:
            columns.append(c.method.label())

    def lookup(r, col):
        for c in cells:
            if c.problem_label == r and c.method.label() == col:
                return _cell_text(c, opcounts)
        return "--"

    wid = max([9] + [len(c) + 2 for c in columns])
    out = "dimension".ljust(wid) + "".join("| " + c.ljust(wid) for c in columns) + "\n"
    for r in rows:
        out += r.ljust(wid) + "".join("| " + lookup(r, c).ljust(wid) for c in columns) + "\n"
    out += "\n" + ("cells: operator applications (matvecs)\n" if opcounts else "cells: iterations\n")
    out += ("counting: Omin/MR families report outer iterations (one s-step each);\n"
            "          the GMRES family reports inner steps summed over cycles.\n"
            "markers: DIV(n) diverged, BRK(n) breakdown, MAX(n) iteration cap, ERR failed,\n"
            "         -- missing cell.\n")
    return out


def _g17(v: float) -> str:
    return "%.17g" % v


def emit_table_csv(cells: list) -> str:
    """bench.hpp:364-385: one line per cell."""
    out = ("nx,method,s,k_or_m,preconditioned,iterations,matvecs,dotprods,updates,"
           "final_residual,converged,breakdown\n")
    for c in cells:
        out += f"{c.problem_label},{c.method.method},{c.method.s},{c.method.k_or_m()},{int(c.method.precondition)},"
        if c.outcome is not None:
            rep = c.outcome.report
            out += (f"{rep.iterations},{rep.op_counts[1]},{rep.op_counts[0]},{rep.op_counts[2]},"
                    f"{_g17(rep.final_residual)},{int(rep.converged)},{rep.breakdown or ''}")
        else:
            out += f",,,,,0,{c.error}"
        out += "\n"
    return out


def report_to_json(cell: CellResult) -> dict:
    """bench.hpp:387-429: the per-cell report object (keys in the reference's order)."""
    j = {"nx": cell.nx, "problem": cell.problem_label, "method": cell.method.method, "s": cell.method.s,
         "k_or_m": cell.method.k_or_m(), "preconditioned": cell.method.precondition}
    if cell.error:
        j["error"] = cell.error
        return j
    rep = cell.outcome.report
    j.update({"iterations": rep.iterations, "cycles": rep.cycles, "matvecs": rep.op_counts[1],
              "dotprods": rep.op_counts[0], "updates": rep.op_counts[2], "termination_dots": rep.op_counts[4],
              "stored_vectors": rep.op_counts[3], "final_residual": rep.final_residual,
              "converged": rep.converged, "breakdown": rep.breakdown, "fallback_cycles": rep.fallback_cycles,
              "residual_history": list(rep.residual_history)})
    if rep.notes:
        j["notes"] = list(rep.notes)
    a = cell.outcome.audit
    j["audit"] = None if a is None else {"ok": a.ok, "matvecs_exact": a.matvecs_exact,
                                         "dotprods_exact": a.dotprods_exact, "updates_exact": a.updates_exact,
                                         "diffs": list(a.diffs)}
    return j
