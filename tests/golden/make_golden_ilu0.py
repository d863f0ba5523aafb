"""Add the ILU(0) golden cases to tests/golden/ from the UNMODIFIED reference (oracle/_ref).

    make -C oracle && python tests/golden/make_golden_ilu0.py

Cases (appended to manifest.json; the other cases are left untouched):
  * ilu0_T61_nx{16,64}: the paper's Table 6.1 problem (problem.hpp discretize, beta = 1,
    gamma = 50, 1/h^2 scaling) -- ilu0_factor values in A's pattern, z = ilu0_apply(r) and
    A z (the right-preconditioned operator applied to r), ilu0.hpp:45-146;
  * ilu0_zero_pivot / ilu0_no_diagonal: the factorization's two error paths;
  * solve_linear_*: the reference driver flow (bench.hpp:149-191) with and without ILU(0)
    right preconditioning around s-Omin and s-GMRES on the same problem.
"""
from __future__ import annotations

import importlib.util
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import CsrMatrix, Oracle, OracleError  # noqa: E402
from paper_2001_04886_b200.problems import splitmix64_uniform  # noqa: E402

sys.path.insert(0, os.path.dirname(HERE))
from parity_util import rel_hist  # noqa: E402

spec = importlib.util.spec_from_file_location("make_golden", os.path.join(HERE, "make_golden.py"))
mg = importlib.util.module_from_spec(spec)
spec.loader.exec_module(mg)
REF = Oracle("reference")


def main():
    manifest = json.load(open(os.path.join(HERE, "manifest.json")))

    def save(name, arrays, meta):
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **arrays)
        manifest[name] = meta

    for nx in (16, 64):
        a, rhs, x0 = mg.discretize(nx, 1.0, 50.0)
        lu = REF.ilu0_factor(a)
        r = splitmix64_uniform(7, a.n)
        z = REF.ilu0_apply(a, lu, r)
        save(f"ilu0_T61_nx{nx}", dict(offs=a.offs, cols=a.cols, vals=a.vals, lu=lu, r=r, z=z, az=REF.spmv(a, z)),
             dict(type="ilu0", nx=nx, ref="ilu0.hpp:45-146 on problem.hpp discretize(nx, beta=1, gamma=50)"))
    # error paths: a pivot below 1e-14 max|diag| (row 1 eliminates column 0), a missing diagonal
    for name, dense in (("ilu0_zero_pivot", [[1e-20, 1.0, 0.0], [1.0, 1.0, 0.0], [0.0, 1.0, 2.0]]),
                        ("ilu0_no_diagonal", [[1.0, 1.0, 0.0], [1.0, 0.0, 1.0], [0.0, 1.0, 2.0]])):
        a = CsrMatrix.from_dense(np.array(dense))  # (non-zeros only: row 2 of the second has no diagonal)
        try:
            REF.ilu0_factor(a)
            err, status = None, 0
        except OracleError as e:
            err, status = str(e), e.status
        save(name, dict(offs=a.offs, cols=a.cols, vals=a.vals), dict(type="ilu0_error", error=err, status=status,
                                                                       ref="ilu0.hpp:52-79"))
    # the driver flow (bench.hpp:149-191)
    a, rhs, x0 = mg.discretize(64, 1.0, 50.0)
    r0 = rhs - REF.spmv(a, x0)
    tol = 1e-8 * float(np.linalg.norm(r0))
    for name, method, cfg, prec in (
            ("solve_linear_somin_s2_k2_T61_nx64_ilu0", "somin", dict(s=2, k=2), True),
            ("solve_linear_sgmres_s2_m5_T61_nx64_ilu0", "sgmres", dict(s=2, m=5), True),
            ("solve_linear_somin_s4_k2_T61_nx64_ilu0", "somin", dict(s=4, k=2), True),
            ("solve_linear_sgmres_s2_m5_T61_nx64_plain", "sgmres", dict(s=2, m=5), False)):
        cfg = dict(cfg, tol=tol, max_iterations=2000)
        res = REF.solve_linear(method, a, rhs, x0, precondition=prec, **cfg)
        arrays = dict(offs=a.offs, cols=a.cols, vals=a.vals, f=rhs, x0=x0, x=res.x,
                      history=np.array(res.residual_history),
                      op_history=np.array(res.op_history, dtype=np.uint64).reshape(-1, 5),
                      op_counts=np.array(res.op_counts, dtype=np.uint64))
        save(name, arrays, dict(type="solve_linear", method=method, cfg=cfg, precondition=prec,
                                converged=res.converged, iterations=res.iterations, cycles=res.cycles,
                                final_residual=res.final_residual, steady_iteration=res.steady_iteration,
                                breakdown=res.breakdown, fallback_cycles=res.fallback_cycles, notes=res.notes,
                                ref="bench.hpp:149-191 driver flow around sstep.hpp on discretize(64, 1, 50)"))
        # the reference's own summation-order sensitivity: the oracle restatement's driver flow
        # (bit-identical to the reference's in its sequential order) with its dots in the other
        # orders (as make_envelope.py does for the solver cases)
        port = Oracle("port")
        base = port.solve_linear(method, a, rhs, x0, precondition=prec, **cfg).residual_history
        env = 0.0
        for mode in (1, 2, 3):
            port.set_dot_mode(mode)
            h = port.solve_linear(method, a, rhs, x0, precondition=prec, **cfg).residual_history
            env = max(env, rel_hist(h[:-1], base[:-1]))
        port.set_dot_mode(0)
        manifest[name]["envelope_hist50"] = env
        print(name, res.converged, res.iterations, res.breakdown, manifest[name].get("envelope_hist50"))
    json.dump(manifest, open(os.path.join(HERE, "manifest.json"), "w"), indent=1, sort_keys=True)
    extra_cases()


def _digest(v):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(v, dtype=np.float64).tobytes()).hexdigest()


def extra_cases():
    """Grid shapes the strip-wavefront solves hand off on: a rectangular 80 x 37
    grid (three strips, a partial last one), a 3D 7-point grid (level schedule), and a
    tridiagonal matrix above the strip path's old cooperative-grid limit (n = 160000, detected
    as an nx = n, ny = 1 grid).  The large case stores only sha256 digests of the reference's
    factor / solve / operator bits; its inputs are regenerated from the port's stencil builder
    and the splitmix64 stream."""
    from paper_2001_04886_b200.problems import convection_diffusion
    manifest = json.load(open(os.path.join(HERE, "manifest.json")))
    port = Oracle("port")
    for name, (dim, nx, ny, nz, conv) in {"ilu0_rect_80x37": (2, 80, 37, 1, 50.0),
                                           "ilu0_3d_12": (3, 12, 12, 12, 20.0)}.items():
        st = convection_diffusion(dim, nx, conv, ny=ny, nz=nz if dim == 3 else None)
        a = port.stencil_csr(dim, st.nx, st.ny, st.nz, st.coef, ch2=st.ch2)
        lu = REF.ilu0_factor(a)
        r = splitmix64_uniform(7, a.n)
        z = REF.ilu0_apply(a, lu, r)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), offs=a.offs, cols=a.cols, vals=a.vals, lu=lu, r=r, z=z,
                            az=REF.spmv(a, z))
        manifest[name] = dict(type="ilu0", grid=[nx, ny, nz], ref="ilu0.hpp:45-146 on the h^2-scaled stencil")
    # tridiagonal, n = 160000 (1D convection-diffusion, h^2-scaled)
    n = 160000
    h = 1.0 / (n + 1.0)
    lo, hi = -1.0 - 50.0 * h / 2.0, -1.0 + 50.0 * h / 2.0
    trip = []
    offs = [0]
    cols, vals = [], []
    for i in range(n):
        if i > 0:
            cols.append(i - 1), vals.append(lo)
        cols.append(i), vals.append(2.0)
        if i + 1 < n:
            cols.append(i + 1), vals.append(hi)
        offs.append(len(cols))
    a = CsrMatrix(np.array(offs, np.uint64), np.array(cols, np.uint64), np.array(vals))
    lu = REF.ilu0_factor(a)
    r = splitmix64_uniform(7, n)
    z = REF.ilu0_apply(a, lu, r)
    manifest["ilu0_tridiag_160000"] = dict(type="ilu0_digest", n=n, conv=50.0, rhs_seed=7,
                                           lu_sha256=_digest(lu), z_sha256=_digest(z), az_sha256=_digest(REF.spmv(a, z)),
                                           ref="ilu0.hpp:45-146 on a tridiagonal 1D convection-diffusion matrix")
    json.dump(manifest, open(os.path.join(HERE, "manifest.json"), "w"), indent=1, sort_keys=True)
    print("extra ILU(0) cases written")


if __name__ == "__main__":
    if sys.argv[1:] == ["extra"]:
        extra_cases()
    else:
        main()
