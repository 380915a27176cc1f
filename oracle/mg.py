"""Nested hierarchy, transfer operators and Galerkin products (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md:146 "Let Omega_l be the coarsest discretization ... I^j_{j+1}, I^{j+1}_j
the interpolation and restriction operators between two consecutive levels";
PAPER.md:155 / Alg. 2 l.5 (:705) Galerkin projection K^l = I^1_l K I^l_1.
Factor-2 coarsening, bilinear/trilinear nodal interpolation, restriction = P^T
(SPEC.md:29-33, :70-71).  Boundary conditions: a coarse DOF is fixed
iff its coincident fine DOF is fixed; P is masked on both sides, P_m = F_f P F_c.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp


def level_dims(nel, levels):
    f = 1 << (levels - 1)
    if any(n % f for n in nel):
        raise ValueError("NonDivisibleDims")
    return [tuple(n >> l for n in nel) for l in range(levels)]


def prolongation_1d(nc: int) -> sp.csr_matrix:
    """(2nc+1) x (nc+1) linear interpolation on a node line: weight 1 at coincident
    nodes, 1/2 at midpoints (hat functions)."""
    nf = 2 * nc
    rows, cols, vals = [], [], []
    for I in range(nc + 1):
        rows.append(2 * I); cols.append(I); vals.append(1.0)
        if I > 0:
            rows.append(2 * I - 1); cols.append(I); vals.append(0.5)
        if I < nc:
            rows.append(2 * I + 1); cols.append(I); vals.append(0.5)
    return sp.csr_matrix((vals, (rows, cols)), shape=(nf + 1, nc + 1))


def prolongation(nel_c, dim=None) -> sp.csr_matrix:
    """DOF prolongation coarse -> fine (unmasked): kron over axes (axis 0 slowest) x I_d."""
    dim = len(nel_c) if dim is None else dim
    P = prolongation_1d(nel_c[0])
    for n in nel_c[1:]:
        P = sp.kron(P, prolongation_1d(n), format="csr")
    return sp.kron(P, sp.eye(dim), format="csr")


def coarse_fixed(nel_f, fixed_f) -> np.ndarray:
    """Coarse DOF fixed iff coincident fine DOF fixed."""
    dim = len(nel_f)
    g = np.asarray(fixed_f).reshape(tuple(n + 1 for n in nel_f) + (dim,))
    sl = tuple(slice(0, None, 2) for _ in nel_f)
    return np.ascontiguousarray(g[sl]).reshape(-1)


def masked_prolongation(nel_c, fixed_f, fixed_c) -> sp.csr_matrix:
    P = prolongation(nel_c)
    return (sp.diags(1.0 - np.asarray(fixed_f, float)) @ P @ sp.diags(1.0 - np.asarray(fixed_c, float))).tocsr()


def galerkin(A_f, Pm, fixed_c, row_blocks=1) -> sp.csr_matrix:
    """A_c = Pm^T A_f Pm + (I - F_c)  (Alg. 2 l.5).
    row_blocks > 1 forms the same product as sum_b Pm[rows_b]^T (A_f[rows_b] Pm) over bands of
    fine rows, so that the fine-by-coarse intermediate never exists whole (C5 size)."""
    if row_blocks <= 1:
        return (Pm.T @ A_f @ Pm + sp.diags(np.asarray(fixed_c, float))).tocsr()
    n = A_f.shape[0]
    Ac = sp.diags(np.asarray(fixed_c, float)).tocsr()
    for b in range(row_blocks):
        r0, r1 = b * n // row_blocks, (b + 1) * n // row_blocks
        Ac = (Ac + Pm[r0:r1].T @ (A_f[r0:r1] @ Pm)).tocsr()
    return Ac


class Hierarchy:
    """All levels' operators for a K with Dirichlet identity rows (A_0 = K_bc)."""

    def __init__(self, nel, K_bc, fixed, levels, row_blocks=1):
        self.dims = level_dims(nel, levels)
        self.A = [K_bc.tocsr()]
        self.fixed = [np.asarray(fixed)]
        self.P = []
        for l in range(1, levels):
            fc = coarse_fixed(self.dims[l - 1], self.fixed[-1])
            Pm = masked_prolongation(self.dims[l], self.fixed[-1], fc)
            self.P.append(Pm)
            self.fixed.append(fc)
            self.A.append(galerkin(self.A[-1], Pm, fc, row_blocks if l == 1 else 1))
