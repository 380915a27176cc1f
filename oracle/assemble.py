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


def apply_dirichlet(A: sp.csr_matrix, fixed, identity: bool) -> sp.csr_matrix:
    free = 1.0 - np.asarray(fixed, dtype=np.float64)
    F = sp.diags(free)
    out = F @ A @ F
    if identity:
        out = out + sp.diags(np.asarray(fixed, dtype=np.float64))
    return out.tocsr()


def assemble_K(nel, E, fixed, nu=0.3, element="std") -> sp.csr_matrix:
    """Fine-grid K with fixed rows/cols replaced by identity."""
    return apply_dirichlet(assemble_K_raw(nel, E, nu, element), fixed, identity=True)


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
