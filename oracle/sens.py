"""Adjoint right-hand sides and buckling-load-factor sensitivities (oracle; TEST
INFRASTRUCTURE ONLY).  SURVEY.md 8(f) NEXT-1.

* `adjoint_rhs`: b_i = phi_i^T (grad_u G) phi_i, the right-hand side of the adjoint system
  K z_i = b_i, Eq. 5.  G(u) = F (sum_e Es_e A_e^T G_e0[u_e] A_e) F is
  linear in u, so d(phi^T G phi)/du_k is evaluated element by element as
  phi_e^T G_e0[e_q] phi_e with e_q the q-th local unit displacement (the definition of the
  gradient of a linear form, using `fem.element_geometric` as is).  b is returned on the free
  DOFs (zero on fixed DOFs, like every right-hand side of the solve).
* `element_terms`: per element e the three quadratic forms of Eq. 4 with unit
  moduli: k_e = phi_e^T K_e0 phi_e, g_e = phi_e^T G_e0[u_e] phi_e, kz_e = z_e^T K_e0 u_e
  (vectors masked to the free DOFs, since K's fixed rows/cols are identity and G's are zero).
* `eigen_sensitivity`: Eq. 4, d lambda / d x_e = dEk_e (k_e - lambda kz_e) + lambda dEs_e g_e, with
  dEk_e = d E_kappa / d x_e and dEs_e = d E_sigma / d x_e supplied by the caller (Eq. 2 :104-108);
  the filter / projection chain rule is outside the hot path.
"""

from __future__ import annotations

import numpy as np

from . import fem
from .assemble import element_dofs, element_geometric_batch


def adjoint_rhs(nel, Es, fixed, phi, nu=0.3):
    """b (n,) or (nphi, n) for phi (n,) or (nphi, n)."""
    phi = np.asarray(phi, dtype=np.float64)
    single = phi.ndim == 1
    phis = phi[None] if single else phi
    dim = len(nel)
    n = phis.shape[1]
    free = 1.0 - np.asarray(fixed, dtype=np.float64)
    edofs = element_dofs(nel)                                  # (m, d 2^d)
    nl = edofs.shape[1]
    # G_e0 at every local unit displacement: (nl, nl, nl), linear in u_e
    Gq = np.stack([fem.element_geometric(dim, np.eye(nl)[q], nu) for q in range(nl)])
    Es = np.asarray(Es, dtype=np.float64)
    out = []
    for ph in phis:
        pe = (ph * free)[edofs]                                 # (m, nl) masked phi_e
        c = np.einsum("ea,qab,eb->eq", pe, Gq, pe) * Es[:, None]
        b = np.zeros(n)
        np.add.at(b, edofs.reshape(-1), c.reshape(-1))
        out.append(b * free)
    return out[0] if single else np.stack(out)


def element_terms(nel, fixed, u, phi, z, nu=0.3):
    """(k, g, kz) each (m,) for one mode phi, its adjoint z and the state u."""
    dim = len(nel)
    free = 1.0 - np.asarray(fixed, dtype=np.float64)
    edofs = element_dofs(nel)
    K0 = fem.element_stiffness(dim, nu)
    pe = (np.asarray(phi, dtype=np.float64) * free)[edofs]
    ze = (np.asarray(z, dtype=np.float64) * free)[edofs]
    ue = np.asarray(u, dtype=np.float64)[edofs]
    uef = (np.asarray(u, dtype=np.float64) * free)[edofs]
    k = np.einsum("ea,ab,eb->e", pe, K0, pe)
    kz = np.einsum("ea,ab,eb->e", ze, K0, uef)
    g = np.einsum("ea,eab,eb->e", pe, element_geometric_batch(dim, ue, nu), pe)
    return k, g, kz


def eigen_sensitivity(nel, fixed, u, phi, z, lam, dEk, dEs, nu=0.3):
    """Eq. 4 for one simple eigenpair (lam, phi) with phi^T K phi = 1 and K z = adjoint_rhs."""
    k, g, kz = element_terms(nel, fixed, u, phi, z, nu)
    return np.asarray(dEk) * (k - lam * kz) + lam * np.asarray(dEs) * g
