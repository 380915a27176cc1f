"""Pins of the NEXT-1 oracle (oracle/sens.py): adjoint right-hand side of Eq. 5 and the
eigenvalue sensitivity of Eq. 4, against finite differences of quantities
the oracle assembles independently (SURVEY.md 8(f) NEXT-1 pins)."""

import numpy as np
import pytest
import scipy.linalg as sla

from oracle import assemble, sens, solve
from workloads import get_config
from workloads.generate import fixed_mask, state_load


def column(nel, x, p=3.0, Emin=1e-6):
    """Clamped column under unit compression (the C1-C5 load case) with SIMP moduli of x."""
    cfg = get_config("T2a" if len(nel) == 2 else "T3a", nel=nel, nrhs=1)
    fixed = fixed_mask(cfg)
    f = state_load(cfg) * (1 - fixed)
    E = Emin + x ** p * (1 - Emin)
    Es = x ** p
    K = assemble.assemble_K(nel, E, fixed)
    u = solve.direct_solve(K, f, fixed)
    G = assemble.assemble_G(nel, Es, u, fixed)
    free = np.where(fixed == 0)[0]
    th, V = sla.eigh(-G.toarray()[np.ix_(free, free)], K.toarray()[np.ix_(free, free)])
    i = int(np.argmax(th))                       # smallest positive lambda = 1 / largest theta
    phi = np.zeros(len(f))
    phi[free] = V[:, i]                          # phi^T K phi = 1
    return dict(K=K, G=G, u=u, lam=1.0 / th[i], phi=phi, fixed=fixed, E=E, Es=Es)


@pytest.mark.parametrize("nel", [(6, 3), (3, 2, 2)])
def test_adjoint_rhs_is_the_gradient_of_phiGphi(nel):
    """G is linear in u, so a central difference with unit step is exact up to rounding."""
    rng = np.random.default_rng(11)
    m = int(np.prod(nel))
    x = rng.uniform(0.3, 1.0, m)
    P = column(nel, x)
    phi = rng.standard_normal(len(P["u"]))
    b = sens.adjoint_rhs(nel, P["Es"], P["fixed"], phi)
    n = len(P["u"])
    for k in np.where(P["fixed"] == 0)[0]:
        e = np.zeros(n)
        e[k] = 1.0
        fp = phi @ (assemble.assemble_G(nel, P["Es"], P["u"] + e, P["fixed"]) @ phi)
        fm = phi @ (assemble.assemble_G(nel, P["Es"], P["u"] - e, P["fixed"]) @ phi)
        assert abs(b[k] - (fp - fm) / 2) <= 1e-13 * (abs(b).max() + 1.0)
    assert np.all(b[P["fixed"] == 1] == 0.0)
    # Euler: the linear form reproduces itself, u . b = phi^T G(u) phi (u = 0 on fixed DOFs)
    assert abs(P["u"] @ b - phi @ (P["G"] @ phi)) <= 1e-12 * abs(phi @ (P["G"] @ phi))


@pytest.mark.parametrize("nel,p", [((12, 4), 3.0), ((4, 2, 2), 3.0)])
def test_eq4_sensitivity_vs_finite_differences_of_lambda(nel, p):
    """Eq. 4 with the adjoint of Eq. 5 reproduces d lambda / d x_e by central differences of the
    full pipeline (K(x), u(x), G(x, u), eigensolve).  Reading: Eq. 4 as printed is
    the derivative for modes with phi^T (-G) phi = 1; for the phi^T K phi = 1 normalisation of
    PAPER.md:122 it carries an extra factor lambda."""
    rng = np.random.default_rng(5)
    m = int(np.prod(nel))
    x = rng.uniform(0.4, 1.0, m)
    P = column(nel, x, p)
    lam, phi = P["lam"], P["phi"]
    b = sens.adjoint_rhs(nel, P["Es"], P["fixed"], phi)
    z = solve.direct_solve(P["K"], b, P["fixed"])
    dEk = p * x ** (p - 1) * (1 - 1e-6)
    dEs = p * x ** (p - 1)
    s = sens.eigen_sensitivity(nel, P["fixed"], P["u"], phi, z, lam, dEk, dEs)
    # G-normalised mode: Eq. 4 verbatim
    phiG = phi * np.sqrt(lam)
    zG = z * lam
    sG = sens.eigen_sensitivity(nel, P["fixed"], P["u"], phiG, zG, lam, dEk, dEs)
    assert np.allclose(sG, lam * s, rtol=1e-9, atol=1e-15)
    h = 1e-6
    for e in rng.choice(m, 6, replace=False):
        xp, xm = x.copy(), x.copy()
        xp[e] += h
        xm[e] -= h
        fd = (column(nel, xp, p)["lam"] - column(nel, xm, p)["lam"]) / (2 * h)
        assert abs(sG[e] - fd) <= 1e-5 * abs(fd) + 1e-12   # central-difference noise ~1e-6


def test_element_terms_sum_to_the_global_forms():
    rng = np.random.default_rng(2)
    nel = (8, 4)
    x = rng.uniform(0.3, 1.0, 32)
    P = column(nel, x)
    phi = rng.standard_normal(len(P["u"])) * (1 - P["fixed"])
    z = rng.standard_normal(len(P["u"])) * (1 - P["fixed"])
    k, g, kz = sens.element_terms(nel, P["fixed"], P["u"], phi, z)
    assert np.isclose(P["E"] @ k, phi @ (P["K"] @ phi), rtol=1e-13)
    assert np.isclose(P["Es"] @ g, phi @ (P["G"] @ phi), rtol=1e-12)
    assert np.isclose(P["E"] @ kz, z @ (P["K"] @ P["u"]), rtol=1e-12)
