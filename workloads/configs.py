"""Config table: BASELINE.json configs[0..4] (C1..C5) plus small test variants.

Axis 0 is the first listed dimension, the slowest in memory and the column /
beam axis.  `levels` counts the finest level
(r10: 64x32 with L=3 -> 32x16 -> 16x8).
"""

from __future__ import annotations

from dataclasses import dataclass, field, replace
from math import prod


@dataclass(frozen=True)
class Config:
    name: str
    nel: tuple            # element counts, axis 0 first
    nrhs: int             # state + adjoint right-hand sides
    levels: int
    bc: str = "base"      # "base": all DOFs on node plane i0 = 0 fixed
    load: str = "top"     # "top": unit total load on plane i0 = N0 along -axis 0
                          # "edge": unit total load on edge {i0=N0, i1=0} along -axis 1
    nphi: int = 0         # number of phi vectors for G(u) phi timing (C3: 12)
    seed: int = 1000      # numpy default_rng seed (r9: 1000 + k for config Ck)
    E0: float = 1.0
    Emin: float = 1e-6
    nu: float = 0.3
    penal: float = 3.0
    rmin: float = 2.0     # density filter radius (elements)
    beta: float = 2.0     # Heaviside projection sharpness (Eq. 1)
    eta: float = 0.5      # Heaviside projection threshold (Eq. 1)
    rhs_rmin: float = 4.0 # adjoint-field filter radius (node lattice)
    tol: float = 1e-10

    @property
    def dim(self) -> int:
        return len(self.nel)


CONFIGS = {
    # BASELINE.json:7  (64x32 Q4 has 2,145 nodes / 4,290 DOFs)
    "C1": Config("C1", (64, 32), 1, 3, seed=1001),
    # BASELINE.json:8
    "C2": Config("C2", (480, 240), 13, 5, seed=1002),
    # BASELINE.json:9 (also times G(u) phi for 12 phi)
    "C3": Config("C3", (1920, 960), 13, 7, nphi=12, seed=1003),
    # BASELINE.json:10 (cantilever: face x=0 clamped, line load on bottom edge of face x=end)
    # nphi: G(u) phi over the config's 6 adjoint fields (reading r16; full-size 3D G parity, bench step)
    "C4": Config("C4", (96, 48, 48), 7, 4, load="edge", nphi=6, seed=1004),
    # BASELINE.json:11 (column: base clamped, uniform top pressure)
    "C5": Config("C5", (256, 128, 128), 7, 5, nphi=6, seed=1005),
    # bounded CPU-baseline sample of C5 (same recipe, BCs, load and 7 RHS at 1/64 of the elements)
    "C5s": Config("C5s", (64, 32, 32), 7, 3, nphi=6, seed=1005),
    # small variants used by the parity tests (same recipes, oracle-friendly sizes)
    "T2a": Config("T2a", (32, 16), 3, 3, nphi=3, seed=2001),
    "T2b": Config("T2b", (40, 24), 5, 3, nphi=2, seed=2002),          # ragged tiles
    "T2c": Config("T2c", (96, 64), 4, 4, nphi=2, seed=2003),
    "T3a": Config("T3a", (16, 8, 8), 3, 3, nphi=2, seed=3001),
    "T3b": Config("T3b", (24, 12, 12), 3, 3, load="edge", nphi=2, seed=3002),
    "T3c": Config("T3c", (40, 24, 16), 2, 3, nphi=2, seed=3003),       # ragged tiles
    "T3d": Config("T3d", (48, 24, 24), 7, 4, load="edge", nphi=2, seed=3004),
    # coarsest level of C5's size (n_L = 4131 -> padded 4160): the large-level Gauss-Jordan path
    "T3e": Config("T3e", (32, 16, 16), 2, 2, seed=3005),
    # axis 2 wider than one 32-element column tile: the column-cluster fine kernels (h8t.cu CX) with
    # a full last tile (N2 = 64, the grid's last node column right of it) and a ragged one (N2 = 70)
    "T3f": Config("T3f", (8, 12, 64), 3, 3, nphi=2, seed=3006),
    "T3g": Config("T3g", (8, 10, 70), 2, 2, nphi=2, seed=3007),
    # last column tile owning 7 node columns (n2 = 37 = 30 + 7): the stacked-row tail tile of the
    # fine kernels (h8t.cu TAIL), 3 tail row tiles of 21 rows over n1 = 45 (ragged)
    "T3h": Config("T3h", (8, 44, 36), 3, 3, nphi=2, seed=3008),
}


def get_config(name: str, **overrides) -> Config:
    cfg = CONFIGS[name]
    return replace(cfg, **overrides) if overrides else cfg


def n_elems(nel) -> int:
    return prod(nel)


def n_nodes(nel) -> int:
    return prod(n + 1 for n in nel)


def n_dofs(nel) -> int:
    return len(nel) * n_nodes(nel)


def level_dims(nel, levels: int):
    """Element counts of every level (finest first); factor-2 coarsening.

    SPEC.md:36-44 build_hierarchy: requires divisibility by 2^(levels-1)."""
    f = 1 << (levels - 1)
    if levels < 1 or any(n % f for n in nel):
        raise ValueError(f"dims {nel} not divisible by 2^(levels-1) = {f}")
    return [tuple(n >> l for n in nel) for l in range(levels)]
