"""Write tests/golden/sweep.json: the reference driver (oracle/_ref, bench.hpp:149-191
solve_linear) on the cells of the reference's own small sweep (test_bench.cpp:29-42:
nx 5 and 7, beta 1, gamma 50, ILU(0), termination 1e-6) that have a device path
(s-Omin s=2 k=2, GMRES m=10, s-GMRES s=2 m=5).

    make -C oracle && python tests/golden/make_golden_sweep.py
"""
from __future__ import annotations

import importlib.util
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
mg = importlib.util.module_from_spec(spec)
spec.loader.exec_module(mg)


def main():
    cells = []
    for nx in (5, 7):
        a, rhs, x0 = mg.discretize(nx, 1.0, 50.0)
        for method, cfg in (("somin", dict(s=2, k=2)), ("gmres", dict(s=1, m=10)), ("sgmres", dict(s=2, m=5))):
            full = dict(s=2, k=4, m=10)
            full.update(cfg)
            res = mg.REF.solve_linear(method, a, rhs, x0, precondition=True, tol=1e-6, max_iterations=100000, **full)
            cells.append(dict(nx=nx, method=method, cfg=full, iterations=res.iterations, cycles=res.cycles,
                              converged=res.converged, breakdown=res.breakdown, op_counts=list(res.op_counts),
                              op_history=[list(h) for h in res.op_history], steady=res.steady_iteration,
                              final_residual=res.final_residual, fallback_cycles=res.fallback_cycles))
            print(nx, method, res.iterations, res.converged, res.op_counts)
    with open(os.path.join(HERE, "sweep.json"), "w") as fh:
        json.dump(dict(ref="bench.hpp:149-191 solve_linear via oracle/_ref on test_bench.cpp:29-42's sweep",
                       cells=cells), fh, indent=0)


if __name__ == "__main__":
    main()
