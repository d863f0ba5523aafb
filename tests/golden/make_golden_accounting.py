"""Write tests/golden/accounting.json from the UNMODIFIED reference (oracle/_ref).

    make -C oracle && python tests/golden/make_golden_accounting.py

Contents:
  * "predict": every prediction / slack function of accounting.hpp:54-132 over a grid of
    (j, k, s) and (m, s);
  * "audit": audit() verdicts (accounting.hpp:149-191) -- the reference's own test_accounting.cpp
    cases (histories from the reference solvers on discretize(nx=7)), the structured-diff case,
    and seeded synthetic histories around the predictions in all three modes;
  * "solves": the reference test cases' problem (discretize(7): CSR, rhs, x0), configurations,
    op histories and verdicts, so the GPU solvers' reports can be audited the same way.
"""
from __future__ import annotations

import ctypes as C
import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import Counter  # noqa: E402

spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
mg = importlib.util.module_from_spec(spec)
spec.loader.exec_module(mg)
REF = mg.REF
L = REF.lib
L.ref_accounting_predict.argtypes = [C.c_int32, C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(Counter)]
L.ref_audit.argtypes = [C.POINTER(Counter), C.c_uint64, C.c_uint64, C.POINTER(Counter), C.c_int32,
                        C.POINTER(Counter), C.POINTER(C.c_int32), C.c_char_p, C.c_uint64]


def predict(kind, a=0, b=0, c=0):
    out = Counter()
    L.ref_accounting_predict(kind, a, b, c, C.byref(out))
    return list(out.as_tuple())


def ref_audit(hist, steady, pred, mode, slack):
    arr = (Counter * max(1, len(hist)))(*[Counter(*row) for row in hist])
    flags = (C.c_int32 * 4)()
    buf = C.create_string_buffer(1 << 16)
    L.ref_audit(arr, len(hist), steady, Counter(*pred), mode, Counter(*slack), flags, buf, len(buf))
    d = buf.value.decode()
    return dict(ok=bool(flags[0]), matvecs_exact=bool(flags[1]), dotprods_exact=bool(flags[2]),
                updates_exact=bool(flags[3]), diffs=d.split("\n") if d else [])


def main():
    pred = []
    for s in range(1, 9):
        for k in range(1, 6):
            for j in range(0, 7):
                pred.append(dict(kind=0, args=[j, k, s], out=predict(0, j, k, s)))
        pred.append(dict(kind=3, args=[s], out=predict(3, s)))
        for m in range(1, 13):
            pred.append(dict(kind=1, args=[m, s], out=predict(1, m, s)))
            pred.append(dict(kind=2, args=[m, s], out=predict(2, m, s)))
            pred.append(dict(kind=5, args=[m, s], out=predict(5, m, s)))
    pred.append(dict(kind=4, args=[], out=predict(4)))

    audits, solves = [], []
    a, rhs, x0 = mg.discretize(7)
    # test_accounting.cpp:57-133: the reference's own audit cases
    cases = [(f"omin_k{k}", "standard", "omin", dict(k=k, tol=1e-6), (0, k, k, 1), None, 0) for k in (1, 2, 4)]
    cases += [("gmres_m5", "standard", "gmres", dict(m=5, tol=1e-6, max_iterations=2000), (1, 5, 1), (4,), 1),
              ("somin_s2_k2", "sstep", "somin", dict(s=2, k=2, tol=1e-6), (0, 2, 2, 2), (3, 2), 1),
              ("sgmres_s2_m2", "sstep", "sgmres", dict(s=2, m=2, tol=1e-30, max_iterations=12), (2, 2, 2), (5, 2, 2), 1)]
    for name, fam, method, cfg, pk, sk, mode in cases:
        res = getattr(REF, fam)(method, a, rhs, x0, **cfg)
        p = predict(*pk)
        sl = predict(*sk) if sk else [0] * 5
        hist = [list(h) for h in res.op_history]
        v = ref_audit(hist, res.steady_iteration, p, mode, sl)
        audits.append(dict(name="ref_" + name, hist=hist, steady=res.steady_iteration, predicted=p, mode=mode,
                           slack=sl, verdict=v))
        solves.append(dict(name=name, family=fam, method=method, cfg=cfg, mode=mode, predicted=p, slack=sl,
                           iterations=res.iterations, converged=res.converged, op_history=hist,
                           steady=res.steady_iteration, verdict=v))
    # test_accounting.cpp:160-178: structured diffs
    hist = [[0] * 5, [10, 1, 4, 0, 0]]
    audits.append(dict(name="structured_diffs", hist=hist, steady=0, predicted=[6, 1, 4, 0, 0], mode=0,
                       slack=[0] * 5, verdict=ref_audit(hist, 0, [6, 1, 4, 0, 0], 0, [0] * 5)))
    # seeded synthetic histories: deltas at, just below and just above the prediction
    rng = np.random.default_rng(2001_04886)
    for i in range(120):
        p = [int(v) for v in rng.integers(0, 40, 5)]
        sl = [int(v) for v in rng.integers(0, 4, 5)]
        n = int(rng.integers(0, 7))
        steady = int(rng.integers(0, 5))
        mode = int(rng.integers(0, 3))
        hist, cur = [], [int(v) for v in rng.integers(0, 100, 5)]
        for t in range(n):
            if t:
                d = [max(0, p[c] + int(rng.integers(-2, 3)) * int(rng.random() < 0.4)) for c in range(5)]
                cur = [cur[c] + d[c] for c in range(5)]
                cur[3] = int(rng.integers(0, 50))  # stored_vectors: a peak, not a delta
            hist.append(list(cur))
        audits.append(dict(name=f"synthetic_{i}", hist=hist, steady=steady, predicted=p, mode=mode, slack=sl,
                           verdict=ref_audit(hist, steady, p, mode, sl)))
    out = dict(ref="accounting.hpp:54-191 via oracle/_ref/libskref.so (unmodified reference headers)",
               predict=pred, audit=audits, solves=solves,
               problem=dict(nx=7, offs=a.offs.tolist(), cols=a.cols.tolist(), vals=a.vals.tolist(),
                            rhs=rhs.tolist(), x0=x0.tolist()))
    with open(os.path.join(HERE, "accounting.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print(len(pred), "predictions,", len(audits), "audits,",
          sum(not x["verdict"]["ok"] for x in audits), "failing verdicts")


if __name__ == "__main__":
    main()
