"""Run one golden GPU parity case (debugging aid): python tools/run_case.py <name> [csr]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")):
    sys.path.insert(0, p)
from paper_2001_04886_b200 import Context  # noqa: E402
from parity_util import run_gpu_case  # noqa: E402

ctx = Context(0)
meta, arr, rep, x, op = run_gpu_case(ctx, sys.argv[1], len(sys.argv) < 3)
print("iterations", rep.iterations, "ref", meta["iterations"], "breakdown", rep.breakdown, flush=True)
