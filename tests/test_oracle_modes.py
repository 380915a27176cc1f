"""Pins of the NEXT-2 oracle (oracle/modes.py): the degenerate one-level path
is the exact fine eigenproblem, the multilevel Rayleigh quotients bound the fine
eigenvalues from above and approach them, and the fundamental BLF of a uniform clamped-free
column approaches Euler's load."""

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import assemble, modes, solve
from workloads import get_config
from workloads.generate import fixed_mask, state_load


def column(nel, x, p=3.0, Emin=1e-6):
    cfg = get_config("T2a" if len(nel) == 2 else "T3a", nel=nel, nrhs=1)
    fixed = fixed_mask(cfg)
    f = state_load(cfg) * (1 - fixed)
    E = Emin + x ** p * (1 - Emin)
    Es = x ** p
    K = assemble.assemble_K(nel, E, fixed)
    u = solve.direct_solve(K, f, fixed)
    return E, Es, fixed, u, K


def fine_lambdas(nel, E, Es, fixed, u, K, q):
    G = assemble.assemble_G(nel, Es, u, fixed)
    free = np.where(fixed == 0)[0]
    th = sla.eigh(-G.toarray()[np.ix_(free, free)], K.toarray()[np.ix_(free, free)], eigvals_only=True)
    return np.sort(1.0 / th[th > 0])[:q]


@pytest.mark.parametrize("nel", [(16, 8), (4, 2, 2)])
def test_one_level_is_the_fine_eigenproblem(nel):
    rng = np.random.default_rng(7)
    x = rng.uniform(0.4, 1.0, int(np.prod(nel)))
    E, Es, fixed, u, K = column(nel, x)
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(nel, E, Es, fixed, u, 1, 4)
    ref = fine_lambdas(nel, E, Es, fixed, u, K, 4)
    assert np.allclose(lam_c, ref, rtol=1e-10) and np.allclose(lam_t, ref, rtol=1e-9)


@pytest.mark.parametrize("nel,levels", [((32, 16), 2), ((32, 16), 3), ((8, 4, 4), 2)])
def test_multilevel_quotients_bound_and_approach_the_fine_eigenvalues(nel, levels):
    rng = np.random.default_rng(3)
    x = rng.uniform(0.5, 1.0, int(np.prod(nel)))
    E, Es, fixed, u, K = column(nel, x)
    q = 3
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(nel, E, Es, fixed, u, levels, q)
    ref = fine_lambdas(nel, E, Es, fixed, u, K, q)
    assert lam_t[0] >= ref[0] * (1 - 1e-12)          # Rayleigh quotient >= lambda_1
    assert abs(lam_t[0] / ref[0] - 1) < 0.05          # the global mode is recovered within 5 %
    assert abs(lam_t[0] / ref[0] - 1) <= abs(lam_c[0] / ref[0] - 1) + 1e-12   # the fine BVP improves it


def test_uniform_column_approaches_euler():
    nel = (80, 8)
    x = np.ones(640)
    E, Es, fixed, u, K = column(nel, x, Emin=0.0)
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(nel, E, Es, fixed, u, 3, 1)
    L, h = 80.0, 8.0
    euler = np.pi ** 2 * (h ** 3 / 12.0) / (4 * L ** 2)   # E = 1, unit total load, clamped-free
    assert abs(lam_t[0] / euler - 1) < 0.02


@pytest.mark.parametrize("nel,levels", [((16, 8), 1), ((4, 2, 2), 1), ((32, 16), 3), ((8, 4, 4), 2)])
def test_k_normalisation_and_rayleigh_identity(nel, levels):
    """phi~_i^T K phi~_i = 1 and, with that normalisation, Eq. 8 reduces to
    lambda~_i = -1 / (phi~_i^T G phi~_i): pins the normalisation and the sign convention."""
    rng = np.random.default_rng(11)
    x = rng.uniform(0.4, 1.0, int(np.prod(nel)))
    E, Es, fixed, u, K = column(nel, x)
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(nel, E, Es, fixed, u, levels, 3)
    G = assemble.assemble_G(nel, Es, u, fixed)
    kk = np.einsum("in,in->i", Phi, (K @ Phi.T).T)
    gg = np.einsum("in,in->i", Phi, (G @ Phi.T).T)
    assert np.allclose(kk, 1.0, rtol=1e-12)
    assert np.allclose(lam_t, -1.0 / gg, rtol=1e-12)


@pytest.mark.parametrize("nel", [(16, 8), (4, 2, 2)])
def test_eigen_residual_vanishes_for_one_level(nel):
    """With one level the prolongated coarse modes are the exact fine modes, K Phi~ = G Psi gives
    Phi~ = -Psi / lambda, so the Eq. 7 residual of the first pair is zero (to rounding)."""
    rng = np.random.default_rng(5)
    x = rng.uniform(0.4, 1.0, int(np.prod(nel)))
    E, Es, fixed, u, K = column(nel, x)
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(nel, E, Es, fixed, u, 1, 2)
    y = modes.eigen_residual(nel, E, Es, fixed, u, lam_t[0], Phi[0])
    assert np.linalg.norm(y) <= 1e-9 * np.linalg.norm(K @ Phi[0])


@pytest.mark.parametrize("nel,levels", [((32, 16), 2), ((32, 16), 3), ((8, 4, 4), 2)])
def test_eigen_residual_is_orthogonal_to_its_mode(nel, levels):
    """lambda~_1 is the Rayleigh quotient of phi~_1, so phi~_1^T y = phi~^T K phi~ + lambda~ phi~^T G
    phi~ = 0 exactly, while y itself does not vanish once the coarse levels approximate (Eq. 7)."""
    rng = np.random.default_rng(9)
    x = rng.uniform(0.5, 1.0, int(np.prod(nel)))
    E, Es, fixed, u, K = column(nel, x)
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(nel, E, Es, fixed, u, levels, 2)
    y = modes.eigen_residual(nel, E, Es, fixed, u, lam_t[0], Phi[0])
    ky = np.linalg.norm(K @ Phi[0])
    assert abs(Phi[0] @ y) <= 1e-12 * ky * np.linalg.norm(Phi[0])
    assert np.linalg.norm(y) > 1e-8 * ky
