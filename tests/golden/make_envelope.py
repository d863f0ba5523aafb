"""Measure the reference's own summation-order envelope for every golden solve case.

The oracle restatement is run with its dot products switched to a blocked/tree order
(orc_set_dot_mode(1): 8-lane partials per 1024-element chunk + pairwise tree, the kind of
order any GPU reduction uses) and compared with the reference output stored in the
fixture.  The GPU parity tests accept max(protocol bound, 10 x envelope) for chaotic
cases, as SURVEY.md 8(c) prescribes.  Writes tests/golden/envelope.json.
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

from golden_util import GOLDEN, case, matrix, names  # noqa: E402
from oracle import Oracle  # noqa: E402
from parity_util import rel_hist, rel_vec  # noqa: E402


MODES = {1: "blocked tree", 2: "reversed", 3: "compensated"}


def main():
    orc = Oracle("port")
    env = {}
    for name in names("solve"):
        meta, arr = case(name)
        a = matrix(arr)
        e = dict(hist50=0.0, x=0.0, rho1=0.0, modes={})
        base = None
        if meta["kind"] == "sstep" and meta["method"] == "sgmres" and meta["cfg"].get("s", 1) > 1:
            base = orc.sstep(meta["method"], a, arr["f"], arr["x0"], **meta["cfg"])  # mode 0 == reference
        for mode in MODES:
            orc.set_dot_mode(mode)
            if meta["kind"] == "sstep":
                r = orc.sstep(meta["method"], a, arr["f"], arr["x0"], **meta["cfg"])
            else:
                r = orc.standard(meta["method"], a, arr["f"], arr["x0"], **meta["cfg"])
            h = rel_hist(r.residual_history, arr["history"])
            xv = rel_vec(r.x, arr["x"])
            e["modes"][MODES[mode]] = dict(hist50=h, x=xv, iterations=r.iterations, breakdown=r.breakdown)
            e["hist50"] = max(e["hist50"], h)
            e["x"] = max(e["x"], xv)
            if base is not None and base.block_rho and r.block_rho:
                u, v = base.block_rho[0], r.block_rho[0]
                e["rho1"] = max(e["rho1"], abs(u - v) / max(abs(u), abs(v)))
        orc.set_dot_mode(0)
        env[name] = e
        print(name, f"hist50={e['hist50']:.2e} x={e['x']:.2e}")
    json.dump(env, open(os.path.join(GOLDEN, "envelope.json"), "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
