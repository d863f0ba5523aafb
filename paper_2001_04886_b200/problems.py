"""Seeded synthetic inputs for the BASELINE configurations (ours).

The reference assembles the paper's Section 5 problem with 1/h^2 scaling
(problem.hpp:138-199).  BASELINE's configurations are instead constant- or
variable-coefficient convection-diffusion stencils; SURVEY.md 8(c) measured that the
1/h^2 scaling makes the monomial s=4 basis collapse, so the operators here are
scaled by h^2: diagonal 4 (2D) / 6 (3D), off-diagonals -1 -+ c h/2.  Coefficient
values are computed once here and handed, bit for bit, to both the GPU library and
the CPU oracle.

Right-hand sides are counter-based: element i is output i+1 of the splitmix64
stream seeded with ``seed``, mapped to U[-1, 1).  This is identical in numpy here,
in the oracle (orc_fill_uniform) and on the device.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)


def splitmix64_uniform(seed: int, n: int, offset: int = 0) -> np.ndarray:
    """U[-1,1) draws, element i = splitmix64 output number offset+i+1 of `seed`."""
    with np.errstate(over="ignore"):
        idx = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + idx * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return 2.0 * u - 1.0


def lognormal_k(seed: int, n: int) -> np.ndarray:
    """Per-cell k = exp(N(0,1)) of the variable-coefficient operator (Box-Muller on splitmix64
    draws, glibc math on the host; see skc_fill_lognormal)."""
    import ctypes as C
    from . import _lib
    out = np.zeros(n)
    _lib.check(_lib.lib().skc_fill_lognormal(seed, n, out.ctypes.data_as(C.POINTER(C.c_double))))
    return out


@dataclass(frozen=True)
class Stencil:
    """h^2-scaled 5-point (dim 2) / 7-point (dim 3) convection-diffusion operator.

    coef = (-z, -y, -x, C, +x, +y, +z): the reference's ascending-column order for
    natural (x fastest) ordering (sparse.hpp:141-145).  With ``variable_k`` the
    diffusion is -div(k grad u), k per cell, harmonic-mean faces and the cell's own k
    on boundary faces; ``ch2`` = c h / 2 is the convection half-coefficient.
    """

    dim: int
    nx: int
    ny: int
    nz: int
    coef: tuple
    ch2: float = 0.0
    variable_k: bool = False

    @property
    def n(self) -> int:
        return self.nx * self.ny * (self.nz if self.dim == 3 else 1)


def convection_diffusion(dim: int, nx: int, conv: float, ny: int | None = None,
                         nz: int | None = None, variable_k: bool = False) -> Stencil:
    ny = nx if ny is None else ny
    nz = (nx if nz is None else nz) if dim == 3 else 1
    h = 1.0 / (nx + 1.0)
    ch2 = conv * h / 2.0
    lo, hi = -1.0 - ch2, -1.0 + ch2
    diag = 4.0 if dim == 2 else 6.0
    if dim == 2:
        coef = (0.0, lo, lo, diag, hi, hi, 0.0)
    else:
        coef = (lo, lo, lo, diag, hi, hi, hi)
    return Stencil(dim, nx, ny, nz, coef, ch2, variable_k)


# BASELINE.json "configs" (restated in SURVEY.md 8(d)); k=2 is the reference default window.
CONFIGS = {
    "C1": dict(method="somin", dim=2, nx=128, conv=10.0, s=4, k=2, rel_tol=1e-8, max_iterations=200, csr=True),
    "C2": dict(method="sgmres", dim=2, nx=1024, conv=50.0, s=4, m=10, rel_tol=1e-8),
    "C3": dict(method="somin", dim=3, nx=256, conv=20.0, s_list=(1, 2, 4, 8), k=2, fixed_steps=100),
    "C4": dict(method="sgmres", dim=2, nx=16384, conv=50.0, s=8, m=8, fixed_steps=50),
    "C5": dict(method="somin", dim=3, nx=512, conv=20.0, s=8, k=2, fixed_steps=50, variable_k=True),
}

RHS_SEED = 20010486
K_SEED = 4886
