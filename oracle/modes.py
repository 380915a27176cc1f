"""Multilevel approximation of buckling modes (oracle; TEST INFRASTRUCTURE ONLY).
SURVEY.md 8(f) NEXT-2; the four steps of PAPER.md:146-175 (Sec. 2.1, Eq. 6-8):

 1. coarse eigenproblem (K^l + lambda^l G^l) psi^l = 0 with K^l, G^l the Galerkin projections of
    the fine operators (Eq. 6, :153-157), q lowest positive lambda^l;
 2. Psi^j = I^j_{j+1} Psi^{j+1} down to the fine level (:160);
 3. fine BVP K Phi~ = G Psi (Eq. 7, :163-167);
 4. Rayleigh quotients lambda~_i = -phi~_i^T K phi~_i / phi~_i^T G phi~_i (Eq. 8, :170-175);
    the modes are returned normalised as phi~_i^T K phi~_i = 1, and
    `eigen_residual` gives y = (K + lambda~_1 G) phi~_1 (Eq. 7).

K^l = P^T K P + (I - F_l) (identity on fixed coarse DOFs, like the multigrid hierarchy) and
G^l = P^T G P with P the composition of the masked prolongations; the coarse
eigenproblem is solved densely on the free coarse DOFs (scipy eigh of (-G^l, K^l)).
"""

from __future__ import annotations

import numpy as np
import scipy.linalg as sla

from . import assemble, solve
from .mg import Hierarchy


def multilevel_modes(nel, E, Es, fixed, u, levels, q, nu=0.3, element="std"):
    """Returns (lam_coarse (q,), Psi (q, n), Phi (q, n), lam_tilde (q,)); Phi K-normalised."""
    K = assemble.assemble_K(nel, E, fixed, nu, element)
    G = assemble.assemble_G(nel, Es, u, fixed, nu)
    H = Hierarchy(nel, K, fixed, levels)
    Pt = None                                    # fine <- coarsest composition
    for P in H.P:
        Pt = P if Pt is None else Pt @ P
    fixed_L = H.fixed[-1]
    if Pt is None:                               # levels == 1: the coarse problem is the fine one
        KL, GL = K.toarray(), G.toarray()
    else:
        KL = (Pt.T @ K @ Pt).toarray() + np.diag(np.asarray(fixed_L, float))
        GL = (Pt.T @ G @ Pt).toarray()
    free = np.where(np.asarray(fixed_L) == 0)[0]
    th, V = sla.eigh(-GL[np.ix_(free, free)], KL[np.ix_(free, free)])
    order = np.argsort(-th)[:q]                  # largest theta = 1 / lambda, lambda > 0 smallest
    lam_c = 1.0 / th[order]
    PsiL = np.zeros((q, KL.shape[0]))
    PsiL[:, free] = V[:, order].T
    Psi = PsiL if Pt is None else np.asarray((Pt @ PsiL.T).T)
    rhs = np.asarray((G @ Psi.T).T)
    Phi = solve.direct_solve(K, rhs, fixed)
    num = np.einsum("in,in->i", Phi, np.asarray((K @ Phi.T).T))
    den = np.einsum("in,in->i", Phi, np.asarray((G @ Phi.T).T))
    Phi = Phi / np.sqrt(num)[:, None]            # phi~^T K phi~ = 1
    return lam_c, Psi, Phi, -num / den


def eigen_residual(nel, E, Es, fixed, u, lam1, phi1, nu=0.3, element="std"):
    """Eq. 7: y = (K[x] + lambda~_1 G[x, u]) phi~_1, with the assembled K and G."""
    K = assemble.assemble_K(nel, E, fixed, nu, element)
    G = assemble.assemble_G(nel, Es, u, fixed, nu)
    return np.asarray(K @ phi1 + lam1 * (G @ phi1))
