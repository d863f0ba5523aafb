"""Run one restart cycle of the C2 workload (for ncu captures / launch lists)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2001_04886_b200 import Context, SStepConfig, convection_diffusion, sgmres_solve, splitmix64_uniform  # noqa: E402

cycles = int(sys.argv[1]) if len(sys.argv) > 1 else 1
st = convection_diffusion(2, 1024, 50.0)
f = splitmix64_uniform(20010486, st.n)
ctx = Context(0)
op = ctx.stencil(st)
x = np.zeros(st.n)
rep = sgmres_solve(op, f, x, SStepConfig(s=4, m=10, tol=0.0, max_iterations=40 * cycles))
print("cycles", rep.cycles, "iterations", rep.iterations, "launches", ctx.launch_count(), "rn", rep.final_residual)
