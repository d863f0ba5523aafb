"""Print GPU-vs-reference parity metrics for every golden solve case (run on a GPU box).

    python tools/parity_report.py [--json out.json]
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "oracle"), os.path.join(ROOT, "tests")]

from golden_util import names  # noqa: E402
from parity_util import run_gpu_case, summarize  # noqa: E402


def main():
    from paper_2001_04886_b200 import Context
    ctx = Context(0)
    rows = {}
    for name in names("solve"):
        for pref in (True, False):
            try:
                meta, arr, rep, x, op = run_gpu_case(ctx, name, prefer_stencil=pref)
                s = summarize(meta, arr, rep, x)
                s["op_kind"] = op.kind
            except Exception as e:  # report, don't stop
                s = dict(error=f"{type(e).__name__}: {e}")
            key = name + ("" if pref else "[csr]")
            rows[key] = s
            print(key, json.dumps(s, default=str))
            if "stencil" not in __import__("golden_util").MANIFEST[name]:
                break
    if len(sys.argv) > 2 and sys.argv[1] == "--json":
        json.dump(rows, open(sys.argv[2], "w"), indent=1, default=str)


if __name__ == "__main__":
    main()
