"""Sparse assembly of K and G (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md:99 "The global elastic stiffness matrix K = K[x] and the global stress
stiffness matrix G = G[x, u(x)] ... are assembled from the elemental ones
K_e[x_e] = E_kappa(x_e) K_e0 and G_e = E_sigma(x_e) G_e0[u_e(x_e)]".
Dirichlet conditions: fixed rows/cols of K become identity;
fixed rows/cols of G become zero.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import fem


def node_strides(nel):
    nn = [n + 1 for n in nel]
    strides = [1] * len(nn)
    for k in range(len(nn) - 2, -1, -1):
        strides[k] = strides[k + 1] * nn[k + 1]
    return strides


def element_dofs(nel) -> np.ndarray:
    """(m, d*2^d) global DOF indices of each element (elements in C order)."""
    dim = len(nel)
    strides = node_strides(nel)
    grids = np.meshgrid(*[np.arange(n) for n in nel], indexing="ij")
    base = sum(g.reshape(-1) * s for g, s in zip(grids, strides))
    offs = np.array([sum(int(b) * s for b, s in zip(bits, strides)) for bits in fem.local_nodes(dim)])
    nodes = base[:, None] + offs[None, :]                                   # (m, 2^d)
    return (dim * nodes[:, :, None] + np.arange(dim)[None, None, :]).reshape(len(base), -1)


def _coo(edofs, Ke_flat, n):
    nl = edofs.shape[1]
    rows = np.repeat(edofs, nl, axis=1).reshape(-1)
    cols = np.tile(edofs, (1, nl)).reshape(-1)
    return sp.coo_matrix((Ke_flat.reshape(-1), (rows, cols)), shape=(n, n)).tocsr()


def assemble_K_raw(nel, E, nu=0.3, element="std") -> sp.csr_matrix:
    """K = sum_e E_e A_e^T K0 A_e, no boundary conditions."""
    dim = len(nel)
    K0 = fem.element_stiffness_of(element, dim, nu)
    edofs = element_dofs(nel)
    n = dim * int(np.prod([m + 1 for m in nel]))
    vals = np.asarray(E, dtype=np.float64)[:, None] * K0.reshape(1, -1)
    return _coo(edofs, vals, n)


def assemble_K_raw_slabs(nel, E, nu=0.3, element="std", planes=8) -> sp.csr_matrix:
    """The same sum as `assemble_K_raw`, built one band of node planes (axis 0) at a time so that
    the COO triplets of a 12.8M-DOF grid (C5: 2.4e9 of them) never exist at once.  Rows of node
    planes [a, b) receive contributions only from element planes [a-1, b), so each band is
    assembled from those elements' entries restricted to its own rows; the bands are stacked."""
    dim = len(nel)
    K0 = fem.element_stiffness_of(element, dim, nu)
    E = np.asarray(E, dtype=np.float64).reshape(tuple(nel))
    n = dim * int(np.prod([m + 1 for m in nel]))
    plane = dim * int(np.prod([m + 1 for m in nel[1:]]))      # DOFs per node plane
    eplane = int(np.prod(nel[1:]))                            # elements per element plane
    edofs = element_dofs(nel)
    nl = edofs.shape[1]
    blocks = []
    for a in range(0, nel[0] + 1, planes):
        b = min(a + planes, nel[0] + 1)
        e0, e1 = max(a - 1, 0), min(b, nel[0])
        ed = edofs[e0 * eplane:e1 * eplane]
        vals = E.reshape(-1)[e0 * eplane:e1 * eplane, None] * K0.reshape(1, -1)
        rows = np.repeat(ed, nl, axis=1).reshape(-1)
        cols = np.tile(ed, (1, nl)).reshape(-1)
        keep = (rows >= a * plane) & (rows < b * plane)
        blk = sp.coo_matrix((vals.reshape(-1)[keep], (rows[keep] - a * plane, cols[keep])),
                            shape=((b - a) * plane, n)).tocsr()
        del vals, rows, cols, keep
        blocks.append(blk)
    return sp.vstack(blocks, format="csr")


def apply_dirichlet(A: sp.csr_matrix, fixed, identity: bool) -> sp.csr_matrix:
    free = 1.0 - np.asarray(fixed, dtype=np.float64)
    F = sp.diags(free)
    out = F @ A @ F
    if identity:
        out = out + sp.diags(np.asarray(fixed, dtype=np.float64))
    return out.tocsr()


def apply_dirichlet_inplace(A: sp.csr_matrix, fixed, identity: bool) -> sp.csr_matrix:
    """`apply_dirichlet` for matrices too large to copy: the same F A F (+ I - F), formed by
    scaling the stored entries by free[row] * free[col] in place and, for identity=True, setting
    the (structurally present) diagonal of every fixed row to 1."""
    free = 1.0 - np.asarray(fixed, dtype=np.float64)
    n = A.shape[0]
    step = 1 << 20
    for r0 in range(0, n, step):
        r1 = min(r0 + step, n)
        s, e = A.indptr[r0], A.indptr[r1]
        rows = np.repeat(np.arange(r0, r1), np.diff(A.indptr[r0:r1 + 1]))
        A.data[s:e] *= free[rows] * free[A.indices[s:e]]
    if identity:
        for r in np.flatnonzero(free == 0.0):
            s, e = A.indptr[r], A.indptr[r + 1]
            j = s + np.flatnonzero(A.indices[s:e] == r)
            if len(j) != 1:
                raise ValueError("diagonal entry of a fixed row is not stored")
            A.data[j] = 1.0
    return A


def assemble_K(nel, E, fixed, nu=0.3, element="std") -> sp.csr_matrix:
    """Fine-grid K with fixed rows/cols replaced by identity."""
    return apply_dirichlet(assemble_K_raw(nel, E, nu, element), fixed, identity=True)


def assemble_K_large(nel, E, fixed, nu=0.3, element="std") -> sp.csr_matrix:
    """`assemble_K` with the memory-light steps above (same entries; used at C5 size)."""
    return apply_dirichlet_inplace(assemble_K_raw_slabs(nel, E, nu, element), fixed, identity=True)


def element_geometric_batch(dim, u_e, nu=0.3):
    """G_e0[u_e] for a batch of elements: (m, d*2^d, d*2^d)."""
    sig = fem.centroid_stress(dim, u_e, nu)                      # (m, d, d)
    S = np.einsum("eij,ijab->eab", sig, fem.geometric_H(dim))     # (m, na, na)
    m, na = S.shape[0], S.shape[1]
    G = np.einsum("eab,cd->eacbd", S, np.eye(dim)).reshape(m, na * dim, na * dim)
    return G


def assemble_G(nel, Es, u, fixed, nu=0.3) -> sp.csr_matrix:
    """G(u) = sum_e Es_e A_e^T G_e0[u_e] A_e; fixed rows/cols zero.
    u is taken with its fixed DOFs as given (they are 0 for a solution)."""
    dim = len(nel)
    edofs = element_dofs(nel)
    n = dim * int(np.prod([m + 1 for m in nel]))
    Ge = element_geometric_batch(dim, np.asarray(u)[edofs], nu)
    Ge *= np.asarray(Es, dtype=np.float64)[:, None, None]
    return apply_dirichlet(_coo(edofs, Ge, n), fixed, identity=False)
