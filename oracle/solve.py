"""Reference solutions of K u = f (oracle; TEST INFRASTRUCTURE ONLY).

Definition: the method reaches, up to its tolerance, exactly
u = K_ff^-1 f_f on free DOFs, u = 0 on fixed DOFs.  Passages: LA / state solve,
Alg. 1 l.2; adjoint solve, Eq. 5 (:133-136); fine BVP, Eq. 6
(:161-165); mgPCG / mgBPCG (:758-761).

* `direct_solve`: sparse LU (SuperLU, MMD_AT_PLUS_A) on the free-DOF block,
  plus one refinement step whose residual may be computed by an independent
  extended-precision element-by-element matvec (`ebe.matvec(..., longdouble)`).
* `mgpcg_solve`: plain preconditioned CG (one RHS at a time) with a geometric
  multigrid V-cycle built from scipy triple products (`mg.Hierarchy`), for the
  3D sizes where direct factorisation does not fit (SURVEY 8(c) "C4, C5").
  Run to a relative residual far below the product's 1e-10, so that its own
  error does not enter the 1e-8 parity budget.
"""

from __future__ import annotations

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .mg import Hierarchy


def direct_solve(K_bc, F, fixed, residual_fn=None):
    """Solve K_bc U = F for F (n,) or (R, n). residual_fn(U) -> F - K U (optional,
    used for the refinement step; default: the same sparse matrix in fp64)."""
    F = np.asarray(F, dtype=np.float64)
    single = F.ndim == 1
    F2 = F[None] if single else F
    free = np.flatnonzero(np.asarray(fixed) == 0)
    Kff = K_bc[free][:, free].tocsc()
    lu = spla.splu(Kff, permc_spec="MMD_AT_PLUS_A")
    U = np.zeros_like(F2)
    U[:, free] = lu.solve(np.ascontiguousarray(F2[:, free].T)).T
    Rres = residual_fn(U) if residual_fn is not None else F2 - (K_bc @ U.T).T
    U[:, free] += lu.solve(np.ascontiguousarray(np.asarray(Rres, np.float64)[:, free].T)).T
    return U[0] if single else U


class _VCycle:
    """Symmetric V(nu,nu) cycle, damped Jacobi, direct coarsest solve."""

    def __init__(self, H: Hierarchy, omega=0.6, nu=1):
        self.H, self.omega, self.nu = H, omega, nu
        self.Dinv = [1.0 / A.diagonal() for A in H.A]
        self.coarse = spla.splu(H.A[-1].tocsc())

    def apply(self, r, l=0):
        H = self.H
        if l == len(H.A) - 1:
            return self.coarse.solve(r)
        A, Di, w = H.A[l], self.Dinv[l], self.omega
        z = w * Di * r
        for _ in range(self.nu - 1):
            z = z + w * Di * (r - A @ z)
        rc = H.P[l].T @ (r - A @ z)
        z = z + H.P[l] @ self.apply(rc, l + 1)
        for _ in range(self.nu):
            z = z + w * Di * (r - A @ z)
        return z


def pcg(A, b, M, tol, maxit=2000):
    """Textbook PCG, zero initial guess, stop at ||r||/||b|| <= tol."""
    x = np.zeros_like(b)
    r = b.copy()
    nb = np.linalg.norm(b)
    if nb == 0.0:
        return x, 0
    z = M(r)
    p = z.copy()
    rz = r @ z
    for it in range(1, maxit + 1):
        q = A @ p
        alpha = rz / (p @ q)
        x += alpha * p
        r -= alpha * q
        if np.linalg.norm(r) <= tol * nb:
            return x, it
        z = M(r)
        rz_new = r @ z
        p = z + (rz_new / rz) * p
        rz = rz_new
    return x, maxit


def mgpcg_solve(nel, K_bc, F, fixed, levels, tol=1e-13, omega=0.6, nu=1, row_blocks=1):
    F = np.asarray(F, dtype=np.float64)
    single = F.ndim == 1
    F2 = F[None] if single else F
    H = Hierarchy(nel, K_bc, fixed, levels, row_blocks)
    V = _VCycle(H, omega, nu)
    U = np.zeros_like(F2)
    its = []
    for k in range(F2.shape[0]):
        U[k], it = pcg(K_bc, F2[k], V.apply, tol)
        its.append(it)
    return (U[0] if single else U), its
