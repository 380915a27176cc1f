"""Pins of the CPU oracle against what the paper and the mathematics fix (CPU only).

Every oracle function is tied to something other than itself:
closed forms, a second (quadrature-free) construction, exact patch solutions,
beam theory, Euler buckling, dense brute force, and DOF counts printed in the paper.
"""

import json
import os

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse as sp

from oracle import assemble, ebe, fem, mg, solve
from workloads import configs as wc

GOLD = os.path.join(os.path.dirname(__file__), "golden")
CCW = [(0, 0), (1, 0), (1, 1), (0, 1)]


# ---------------------------------------------------------------- element matrices

def kron_construction(dim, nu, plane_stress=True):
    """Quadrature-free K0 from 1-D matrices (SURVEY 8(c) 'K0 second construction'):
    K0[(a,i),(b,j)] = lam S_ij + mu S_ji + mu delta_ij sum_k S_kk,
    S_ij[a,b] = int dN_a/dx_i dN_b/dx_j as a product of 1-D integrals."""
    M = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    D = np.array([[1.0, -1.0], [-1.0, 1.0]])
    C = np.array([[-0.5, -0.5], [0.5, 0.5]])          # C[a,b] = int phi_a' phi_b
    mu = 1.0 / (2 * (1 + nu))
    lam = nu / (1 - nu * nu) if (dim == 2 and plane_stress) else nu / ((1 + nu) * (1 - 2 * nu))
    nodes = fem.local_nodes(dim)
    na = len(nodes)

    def S(i, j):
        out = np.ones((na, na))
        for a, ab in enumerate(nodes):
            for b, bb in enumerate(nodes):
                for k in range(dim):
                    if k == i and k == j:
                        f = D[ab[k], bb[k]]
                    elif k == i:
                        f = C[ab[k], bb[k]]
                    elif k == j:
                        f = C[bb[k], ab[k]]
                    else:
                        f = M[ab[k], bb[k]]
                    out[a, b] *= f
        return out

    Ss = {(i, j): S(i, j) for i in range(dim) for j in range(dim)}
    K = np.zeros((dim * na, dim * na))
    for i in range(dim):
        for j in range(dim):
            blk = lam * Ss[i, j] + mu * Ss[j, i]
            if i == j:
                blk = blk + mu * sum(Ss[k, k] for k in range(dim))
            K[i::dim, j::dim] = blk
    return K, Ss


def test_q4_k0_row_closed_form_and_golden():
    gold = np.loadtxt(os.path.join(GOLD, "q4_k0_row0.txt"))
    K = fem.element_stiffness(2, 0.3, nodes=CCW)
    assert np.allclose(K[0], gold, atol=5e-7)
    for nu in (0.25, 0.3, 0.4):
        K = fem.element_stiffness(2, nu, nodes=CCW)
        row = np.array([1 / 2 - nu / 6, 1 / 8 + nu / 8, -1 / 4 - nu / 12, -1 / 8 + 3 * nu / 8,
                        -1 / 4 + nu / 12, -1 / 8 - nu / 8, nu / 6, 1 / 8 - 3 * nu / 8]) / (1 - nu * nu)
        assert np.allclose(K[0], row, rtol=0, atol=1e-15)


@pytest.mark.parametrize("nu", [0.25, 0.3, 0.4])
def test_q4_k0_eigenvalues_closed_form(nu):
    ev = np.sort(np.linalg.eigvalsh(fem.element_stiffness(2, nu)))
    want = np.sort([0, 0, 0, (3 - nu) / (6 * (1 - nu * nu)), (3 - nu) / (6 * (1 - nu * nu)),
                    1 / (1 + nu), 1 / (1 + nu), 1 / (1 - nu)])
    assert np.allclose(ev, want, atol=1e-14)


@pytest.mark.parametrize("dim", [2, 3])
@pytest.mark.parametrize("nu", [0.2, 0.3, 0.45])
def test_k0_second_construction(dim, nu):
    Kq = fem.element_stiffness(dim, nu)
    Kk, _ = kron_construction(dim, nu)
    assert np.abs(Kq - Kk).max() < 1e-15 * 10


@pytest.mark.parametrize("nu", [0.25, 0.3, 0.4])
def test_h8_k0_properties(nu):
    K = fem.element_stiffness(3, nu)
    assert np.abs(K - K.T).max() < 1e-16
    assert np.abs(K.sum(axis=1)).max() < 1e-14
    ev = np.linalg.eigvalsh(K)
    assert np.sum(np.abs(ev) < 1e-12) == 6
    lam = nu / ((1 + nu) * (1 - 2 * nu))
    mu = 1 / (2 * (1 + nu))
    assert np.allclose(np.diag(K), (lam + 4 * mu) / 9)            # 0.235043 at nu = 0.3
    for want in (1 / (2 * (1 - 2 * nu)), mu, mu / 2, mu / 6, 2 * mu / 3, (lam + 4 * mu) / 18):
        assert np.min(np.abs(ev - want)) < 1e-12


def test_geometric_H_closed_form_and_kron():
    H = fem.geometric_H(2, nodes=CCW)
    Hxx = np.array([[2, -2, -1, 1], [-2, 2, 1, -1], [-1, 1, 2, -2], [1, -1, -2, 2]]) / 6
    Hyy = np.array([[2, 1, -1, -2], [1, 2, -2, -1], [-1, -2, 2, 1], [-2, -1, 1, 2]]) / 6
    Hs = np.array([[1, 0, -1, 0], [0, -1, 0, 1], [-1, 0, 1, 0], [0, 1, 0, -1]]) / 2
    assert np.allclose(H[0, 0], Hxx, atol=1e-15)
    assert np.allclose(H[1, 1], Hyy, atol=1e-15)
    assert np.allclose(H[0, 1] + H[1, 0], Hs, atol=1e-15)
    for dim in (2, 3):
        _, Ss = kron_construction(dim, 0.3)
        H = fem.geometric_H(dim)
        for i in range(dim):
            for j in range(dim):
                assert np.abs(H[i, j] - Ss[i, j]).max() < 1e-15


# ---------------------------------------------------------------- assembly

def rigid_modes(nel):
    dim = len(nel)
    grids = np.meshgrid(*[np.arange(n + 1, dtype=float) for n in nel], indexing="ij")
    X = np.stack([g.reshape(-1) for g in grids], axis=1)
    modes = []
    for c in range(dim):
        v = np.zeros((X.shape[0], dim)); v[:, c] = 1; modes.append(v.reshape(-1))
    pairs = [(0, 1)] if dim == 2 else [(0, 1), (0, 2), (1, 2)]
    for i, j in pairs:
        v = np.zeros((X.shape[0], dim)); v[:, i] = -X[:, j]; v[:, j] = X[:, i]; modes.append(v.reshape(-1))
    return np.stack(modes)


@pytest.mark.parametrize("nel", [(6, 4), (3, 2, 2)])
def test_rigid_null_space_and_spd(nel):
    rng = np.random.default_rng(5)
    E = rng.uniform(0.1, 1.0, int(np.prod(nel)))
    K = assemble.assemble_K_raw(nel, E).toarray()
    assert np.abs(K - K.T).max() < 1e-15
    ev = np.linalg.eigvalsh(K)
    nz = 3 if len(nel) == 2 else 6
    assert np.sum(ev < 1e-10 * ev.max()) == nz
    R = rigid_modes(nel)
    assert np.abs(K @ R.T).max() < 1e-13
    # clamped base -> SPD on free DOFs
    fixed = np.zeros(K.shape[0], np.uint8)
    fixed.reshape(tuple(n + 1 for n in nel) + (len(nel),))[0] = 1
    free = fixed == 0
    np.linalg.cholesky(K[np.ix_(free, free)])


@pytest.mark.parametrize("nel", [(4, 3), (2, 2, 2), (5, 3)])
def test_direct_solve_vs_dense_brute_force(nel):
    rng = np.random.default_rng(7)
    dim = len(nel)
    E = rng.uniform(1e-3, 1.0, int(np.prod(nel)))
    n = dim * int(np.prod([m + 1 for m in nel]))
    fixed = np.zeros(n, np.uint8)
    fixed.reshape(tuple(m + 1 for m in nel) + (dim,))[0] = 1
    K = assemble.assemble_K(nel, E, fixed)
    F = rng.standard_normal((2, n)) * (1 - fixed)
    U = solve.direct_solve(K, F, fixed)
    Ud = np.linalg.solve(K.toarray(), F.T).T
    assert np.abs(U - Ud).max() <= 1e-13 * np.abs(Ud).max()
    # manufactured solution
    us = rng.standard_normal(n) * (1 - fixed)
    u = solve.direct_solve(K, K @ us, fixed)
    assert np.linalg.norm(u - us) <= 1e-11 * np.linalg.norm(us)


def _uniform_compression_case(nel, p=0.7, nu=0.3):
    """Roller supports + uniform traction p on the top face: the exact elasticity
    solution is linear (u0 = -p x0 / E, u_k = nu p x_k / E in plane stress / 3D), which
    bilinear/trilinear elements reproduce exactly (patch test)."""
    dim = len(nel)
    nsh = tuple(m + 1 for m in nel)
    fixed = np.zeros(nsh + (dim,), np.uint8)
    fixed[0, ..., 0] = 1                         # axial roller on the base
    idx = [0] + [slice(None)] * (dim - 1)
    for k in range(1, dim):                      # u_k = 0 on base nodes with x_k = 0
        sl = [0] + [slice(None)] * (dim - 1)
        sl[k] = 0
        fixed[tuple(sl) + (k,)] = 1
    fixed = fixed.reshape(-1)
    f = np.zeros(nsh + (dim,))
    w = None
    for m in nel[1:]:
        t = np.full(m + 1, 1.0); t[0] = t[-1] = 0.5
        w = t if w is None else np.multiply.outer(w, t)
    f[nel[0], ..., 0] = -p * w
    grids = np.meshgrid(*[np.arange(m + 1, dtype=float) for m in nel], indexing="ij")
    uex = np.zeros(nsh + (dim,))
    lat = nu if dim == 3 else nu           # lateral strain factor (plane stress: nu; 3D: nu)
    uex[..., 0] = -p * grids[0]
    for k in range(1, dim):
        uex[..., k] = lat * p * grids[k]
    return fixed, f.reshape(-1), uex.reshape(-1)


@pytest.mark.parametrize("nel", [(8, 5), (4, 3, 2)])
def test_patch_uniform_compression_exact(nel):
    fixed, f, uex = _uniform_compression_case(nel)
    E = np.ones(int(np.prod(nel)))
    K = assemble.assemble_K(nel, E, fixed)
    u = solve.direct_solve(K, f, fixed)
    assert np.abs(u - uex).max() < 1e-12
    # G under the exact uniform stress sigma = diag(-p, 0, ..): G = -p * assembled(H_00 kron I)
    p = 0.7
    G = assemble.assemble_G(nel, E, u, fixed).toarray()
    dim = len(nel)
    edofs = assemble.element_dofs(nel)
    _, Ss = kron_construction(dim, 0.3)
    Ge = np.kron(Ss[0, 0], np.eye(dim)) * (-p)
    n = len(f)
    Gw = np.zeros((n, n))
    for e in range(edofs.shape[0]):
        Gw[np.ix_(edofs[e], edofs[e])] += Ge
    free = 1.0 - fixed
    Gw = Gw * free[:, None] * free[None, :]
    assert np.abs(G - Gw).max() < 1e-12


def _cantilever_tip(nel, element="std"):
    dim = len(nel)
    nsh = tuple(m + 1 for m in nel)
    fixed = np.zeros(nsh + (dim,), np.uint8)
    fixed[0] = 1
    f = np.zeros(nsh + (dim,))
    w = None
    for m in nel[1:]:
        t = np.full(m + 1, 1.0 / m); t[0] = t[-1] = 0.5 / m
        w = t if w is None else np.multiply.outer(w, t)
    f[nel[0], ..., 1] = -w                        # unit total tip shear along -axis 1
    fixed = fixed.reshape(-1)
    K = assemble.assemble_K(nel, np.ones(int(np.prod(nel))), fixed, element=element)
    u = solve.direct_solve(K, f.reshape(-1), fixed).reshape(nsh + (dim,))
    delta = -np.sum(u[nel[0], ..., 1] * w)        # load-weighted tip deflection
    L, h = nel[0], nel[1]
    b = nel[2] if dim == 3 else 1.0
    nu = 0.3
    I = b * h ** 3 / 12.0
    Gs = 1.0 / (2 * (1 + nu))
    timo = L ** 3 / (3 * I) + L / ((5.0 / 6.0) * Gs * b * h)
    return delta / timo


def test_cantilever_vs_timoshenko_q4():
    r1 = _cantilever_tip((80, 8))
    r2 = _cantilever_tip((160, 16))
    assert 0.98 < r1 < 1.0 and 0.99 < r2 < 1.0 and r2 > r1


def test_cantilever_vs_timoshenko_h8():
    r1 = _cantilever_tip((40, 4, 4))
    r2 = _cantilever_tip((80, 8, 8))
    assert 0.93 < r1 < 1.0 and 0.97 < r2 < 1.0 and r2 > r1


@pytest.mark.parametrize("nel,tol", [((80, 8), 0.02), ((40, 4, 4), 0.06)])
def test_euler_buckling_column(nel, tol):
    """Clamped-free column, unit total axial compression, uniform E = Es = 1:
    lambda_1 of (K + lambda G) phi = 0 (Alg. 1 l.4, Eq. 3) vs Euler pi^2 EI / (4 L^2)."""
    dim = len(nel)
    nsh = tuple(m + 1 for m in nel)
    fixed = np.zeros(nsh + (dim,), np.uint8); fixed[0] = 1; fixed = fixed.reshape(-1)
    f = np.zeros(nsh + (dim,))
    w = None
    for m in nel[1:]:
        t = np.full(m + 1, 1.0 / m); t[0] = t[-1] = 0.5 / m
        w = t if w is None else np.multiply.outer(w, t)
    f[nel[0], ..., 0] = -w
    E = np.ones(int(np.prod(nel)))
    K = assemble.assemble_K(nel, E, fixed)
    u = solve.direct_solve(K, f.reshape(-1), fixed)
    G = assemble.assemble_G(nel, E, u, fixed)
    free = np.flatnonzero(fixed == 0)
    Kd = K[free][:, free].toarray(); Gd = G[free][:, free].toarray()
    mu = sla.eigh(-Gd, Kd, eigvals_only=True, subset_by_index=[len(free) - 1, len(free) - 1])
    lam1 = 1.0 / mu[0]
    L, h = nel[0], nel[1]
    I = h ** 3 / 12.0 if dim == 2 else min(nel[2] * h ** 3, h * nel[2] ** 3) / 12.0
    euler = np.pi ** 2 * I / (4 * L ** 2)
    assert abs(lam1 / euler - 1) < tol


def test_G_properties():
    nel = (5, 4)
    rng = np.random.default_rng(3)
    dim, m = 2, 20
    n = dim * 30
    fixed = np.zeros(n, np.uint8)
    Es = rng.uniform(0, 1, m)
    u, v = rng.standard_normal(n), rng.standard_normal(n)
    G = lambda w: assemble.assemble_G(nel, Es, w, fixed).toarray()
    assert np.abs(G(np.zeros(n))).max() == 0
    assert np.abs(G(2 * u + v) - 2 * G(u) - G(v)).max() < 1e-13
    Gu = G(u)
    assert np.abs(Gu - Gu.T).max() < 1e-15
    for r in rigid_modes(nel):
        assert np.abs(G(r)).max() < 1e-13
    for nel3 in [(2, 3, 2)]:
        R3 = rigid_modes(nel3)
        n3 = R3.shape[1]
        for r in R3:
            assert np.abs(assemble.assemble_G(nel3, np.ones(12), r, np.zeros(n3, np.uint8)).toarray()).max() < 1e-13


def test_ebe_routes_match_assembled():
    for nel in [(7, 5), (3, 4, 2)]:
        rng = np.random.default_rng(11)
        dim = len(nel)
        n = dim * int(np.prod([m + 1 for m in nel]))
        E = rng.uniform(1e-3, 1, int(np.prod(nel)))
        fixed = (rng.random(n) < 0.1).astype(np.uint8)
        x = rng.standard_normal((2, n))
        K = assemble.assemble_K(nel, E, fixed)
        y = (K @ x.T).T
        assert np.abs(ebe.matvec(nel, E, fixed, x) - y).max() < 1e-13
        yl = ebe.matvec(nel, E, fixed, x[0], dtype=np.longdouble)
        assert np.abs(np.asarray(yl, float) - y[0]).max() < 1e-13
        nodes = np.array([0, 3, n // dim - 1, n // (2 * dim)])
        rows = ebe.matvec_rows(nel, E, fixed, x[1], nodes)
        assert np.abs(rows - y[1].reshape(-1, dim)[nodes]).max() < 1e-13
        u = rng.standard_normal(n)
        G = assemble.assemble_G(nel, E, u, fixed)
        assert np.abs(ebe.stress_stiffness_apply(nel, E, fixed, u, x) - (G @ x.T).T).max() < 1e-13


# ---------------------------------------------------------------- hierarchy, transfers, Galerkin

def test_hierarchy_paper_counts():
    g = json.load(open(os.path.join(GOLD, "paper_dof_counts.json")))
    for c in g["2d"]:
        nel = tuple(c["nel"])
        n = wc.n_dofs(nel)
        assert abs(n / c["dofs_approx"] - 1) < c["rel"]
        dims = mg.level_dims(nel, c["levels"])
        assert wc.n_elems(nel) == c["cut"] * wc.n_elems(dims[-1])
        assert abs(n / wc.n_dofs(dims[-1]) / c["cut"] - 1) < 0.03   # "cut ... 16 and 64 times" (approx.)
    c = g["3d"]
    nel = tuple(c["nel"])
    assert wc.n_elems(nel) == c["elements"]
    assert wc.n_dofs(nel) == c["dofs"]
    dims = mg.level_dims(nel, c["levels"])
    assert wc.n_dofs(dims[-1]) == c["coarse_dofs"]
    assert wc.level_dims(nel, c["levels"]) == dims
    with pytest.raises(ValueError):
        mg.level_dims((30, 15), 2)
    with pytest.raises(ValueError):
        wc.level_dims((30, 15), 2)


@pytest.mark.parametrize("nelc", [(3, 2), (2, 2, 3)])
def test_prolongation_reproduces_linear_fields(nelc):
    dim = len(nelc)
    nelf = tuple(2 * m for m in nelc)
    P = mg.prolongation(nelc)
    rng = np.random.default_rng(2)
    a, B = rng.standard_normal(dim), rng.standard_normal((dim, dim))

    def lin(nel, h):
        grids = np.meshgrid(*[np.arange(m + 1) * h for m in nel], indexing="ij")
        X = np.stack([g.reshape(-1) for g in grids], 1)
        return (a[None] + X @ B.T).reshape(-1)

    assert np.abs(P @ lin(nelc, 2.0) - lin(nelf, 1.0)).max() < 1e-13
    # hat function: coarse unit vector -> bilinear hat of support 2h
    nc = dim * int(np.prod([m + 1 for m in nelc]))
    e = np.zeros(nc); e[dim * 1 + 0] = 1.0
    hat = (P @ e).reshape(tuple(m + 1 for m in nelf) + (dim,))[..., 0]
    assert hat.max() == 1.0 and set(np.unique(hat)) <= {0.0, 0.125, 0.25, 0.5, 1.0}


@pytest.mark.parametrize("nel", [(8, 4), (4, 4, 2)])
def test_galerkin_equals_rediscretised_for_coarse_constant_E(nel):
    """Nested conforming spaces: P^T K_h P is the FE stiffness of the coarse grid
    (h = 2) when E is constant on each coarse element; 3D stiffness scales as h^(d-2)."""
    dim = len(nel)
    rng = np.random.default_rng(4)
    nelc = tuple(m // 2 for m in nel)
    Ec = rng.uniform(0.1, 1, int(np.prod(nelc))).reshape(nelc)
    Ef = Ec
    for ax in range(dim):
        Ef = np.repeat(Ef, 2, axis=ax)
    n = dim * int(np.prod([m + 1 for m in nel]))
    fixed = np.zeros(n, np.uint8)
    fixed.reshape(tuple(m + 1 for m in nel) + (dim,))[0] = 1
    K = assemble.assemble_K(nel, Ef.reshape(-1), fixed)
    H = mg.Hierarchy(nel, K, fixed, 2)
    Kc = assemble.assemble_K(nelc, Ec.reshape(-1) * 2.0 ** (dim - 2), H.fixed[1])
    assert np.abs((H.A[1] - Kc).toarray()).max() < 1e-14
    assert np.abs((H.A[1] - H.A[1].T).toarray()).max() < 1e-15


def test_iterative_oracle_matches_direct():
    cfg = wc.get_config("T3a")
    from workloads import generate
    inp = generate(cfg, with_phi=False)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    Ud = solve.direct_solve(K, inp["rhs"], inp["fixed"])
    Ui, its = solve.mgpcg_solve(cfg.nel, K, inp["rhs"], inp["fixed"], cfg.levels, tol=1e-13)
    for k in range(cfg.nrhs):
        assert np.linalg.norm(Ui[k] - Ud[k]) <= 1e-11 * np.linalg.norm(Ud[k])
    assert max(its) < 100


# ---------------------------------------------------------------- NEXT-4: incompatible-mode element
@pytest.mark.parametrize("dim", [2, 3])
def test_wilson_element_properties(dim):
    """Condensed incompatible-mode K_e0: symmetric, PSD with
    exactly the rigid modes as null space, and strictly softer than the standard element on the
    pure-bending nodal pattern while equal on constant-strain (patch) patterns."""
    Kw = fem.element_stiffness_wilson(dim)
    K0 = fem.element_stiffness(dim)
    assert np.abs(Kw - Kw.T).max() < 1e-15
    ev = np.linalg.eigvalsh(Kw)
    nrig = 3 if dim == 2 else 6
    assert np.all(np.abs(ev[:nrig]) < 1e-13) and ev[nrig] > 1e-3
    nodes = fem.local_nodes(dim).astype(float)
    # pure bending about axis 1: u_0 = (x_0 - 1/2)(x_1 - 1/2), other components 0
    ub = np.zeros(dim * len(nodes))
    ub[0::dim] = (nodes[:, 0] - 0.5) * (nodes[:, 1] - 0.5)
    assert ub @ Kw @ ub < ub @ K0 @ ub * (1 - 1e-3)
    # constant strain u = A x: identical energy (incompatible modes pass the patch test)
    rng = np.random.default_rng(0)
    A = rng.standard_normal((dim, dim))
    uc = (nodes @ A.T).reshape(-1)
    assert abs(uc @ Kw @ uc - uc @ K0 @ uc) < 1e-12 * abs(uc @ K0 @ uc)


def test_wilson_pure_bending_is_exact_on_the_unit_square():
    """Plane stress pure bending sigma_xx = M y: the Wilson Q6 element represents it exactly, so
    the element energy of the exact nodal field equals the continuum energy (1/2 int sigma eps)."""
    nu = 0.3
    Kw = fem.element_stiffness_wilson(2, nu)
    nodes = fem.local_nodes(2).astype(float)
    # exact field for eps_xx = kappa (y - 1/2), eps_yy = -nu kappa (y - 1/2), gamma = 0:
    # u = kappa x (y - 1/2), v = -kappa x^2 / 2 - nu kappa (y - 1/2)^2 / 2 (up to rigid modes)
    kappa = 1.0
    x, y = nodes[:, 0], nodes[:, 1]
    u = np.zeros(8)
    u[0::2] = kappa * x * (y - 0.5)
    u[1::2] = -0.5 * kappa * x ** 2 - 0.5 * nu * kappa * (y - 0.5) ** 2
    # continuum energy: 1/2 int E eps_xx^2 dA (sigma_yy = 0), = 1/2 kappa^2 int (y - 1/2)^2 = kappa^2 / 24
    exact = kappa ** 2 / 24.0
    assert abs(0.5 * u @ Kw @ u - exact) < 1e-13
    # the standard element overestimates it (shear locking)
    K0 = fem.element_stiffness(2, nu)
    assert 0.5 * u @ K0 @ u > exact * 1.05


@pytest.mark.parametrize("nu", [0.0, 0.3, 0.45])
def test_wilson_pure_bending_is_exact_on_the_unit_cube(nu):
    """3D pure bending sigma_xx = E kappa (y - 1/2), all other stresses zero: the exact field
    u = kappa x (y - 1/2), v = -kappa x^2 / 2 - nu kappa ((y - 1/2)^2 - (z - 1/2)^2) / 2,
    w = -nu kappa (y - 1/2)(z - 1/2) lies in the trilinear + bubble space of the incompatible-mode
    hexahedron, so the condensed element energy of its nodal values equals the
    continuum energy 1/2 int sigma_xx eps_xx = kappa^2 / 24 on the unit cube (E = 1).  A wrong
    strain assignment of the bubble modes (e.g. the shear rows of B_i) changes this energy."""
    Kw = fem.element_stiffness_wilson(3, nu)
    nodes = fem.local_nodes(3).astype(float)
    kappa = 1.0
    x, y, z = nodes[:, 0], nodes[:, 1], nodes[:, 2]
    u = np.zeros(24)
    u[0::3] = kappa * x * (y - 0.5)
    u[1::3] = -0.5 * kappa * x ** 2 - 0.5 * nu * kappa * ((y - 0.5) ** 2 - (z - 0.5) ** 2)
    u[2::3] = -nu * kappa * (y - 0.5) * (z - 0.5)
    exact = kappa ** 2 / 24.0
    assert abs(0.5 * u @ Kw @ u - exact) < 1e-13
    # the same bending about the other axes (coordinate permutations) is exact too
    for perm in ((1, 2, 0), (2, 0, 1)):
        up = np.zeros(24)
        X = nodes[:, list(perm)]
        comp = np.array([[0, 1, 2]])[0][list(perm)]
        up[comp[0]::3] = kappa * X[:, 0] * (X[:, 1] - 0.5)
        up[comp[1]::3] = -0.5 * kappa * X[:, 0] ** 2 - 0.5 * nu * kappa * ((X[:, 1] - 0.5) ** 2 - (X[:, 2] - 0.5) ** 2)
        up[comp[2]::3] = -nu * kappa * (X[:, 1] - 0.5) * (X[:, 2] - 0.5)
        assert abs(0.5 * up @ Kw @ up - exact) < 1e-13
    # the standard trilinear element overestimates it (parasitic shear)
    K0 = fem.element_stiffness(3, nu)
    assert 0.5 * u @ K0 @ u > exact * 1.05


def test_wilson_cantilever_closer_to_beam_theory():
    """SURVEY 8(f) NEXT-4 pin: on a coarse cantilever the incompatible-mode element is closer to
    Timoshenko beam theory than the standard Q4."""
    r_std = _cantilever_tip((16, 2), "std")
    r_wil = _cantilever_tip((16, 2), "wilson")
    assert abs(1 - r_wil) < 0.2 * abs(1 - r_std)
    assert 0.97 < r_wil < 1.03
