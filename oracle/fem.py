"""Element matrices by Gauss quadrature (oracle; TEST INFRASTRUCTURE ONLY).

PAPER.md:99 "K_e[x_e] = E_kappa(x_e) K_e0 and G_e = E_sigma(x_e) G_e0[u_e]".
Element type: standard bilinear Q4 / trilinear H8 on the unit square / cube
(BASELINE.json:5 "standard Q4/H8 element stiffness entries";
plane stress, thickness 1, h = 1).

Local numbering used throughout the oracle: local node a <-> bits
(a_0, ..., a_{d-1}) with a = sum_k a_k 2^(d-1-k) (axis 0 most significant,
i.e. C order inside the element); local DOF = d*a + comp.
"""

from __future__ import annotations

import itertools

import numpy as np

GAUSS_1D = (0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0))  # 2-point rule on [0,1]


def local_nodes(dim: int) -> np.ndarray:
    """(2^d, d) array of local node bit offsets, C order."""
    return np.array(list(itertools.product((0, 1), repeat=dim)), dtype=np.int64)


def shape_grad(dim: int, xi, nodes=None) -> np.ndarray:
    """dN_a/dx_j at point xi on the unit element: array (n_nodes, d).
    N_a(x) = prod_k (x_k if a_k else 1 - x_k)."""
    nodes = local_nodes(dim) if nodes is None else np.asarray(nodes)
    g = np.ones((len(nodes), dim))
    for a, bits in enumerate(nodes):
        for j in range(dim):
            for k in range(dim):
                if k == j:
                    g[a, j] *= 1.0 if bits[k] else -1.0
                else:
                    g[a, j] *= xi[k] if bits[k] else 1.0 - xi[k]
    return g


def constitutive(dim: int, E: float = 1.0, nu: float = 0.3) -> np.ndarray:
    """D0 in Voigt notation.  2D plane stress [e00, e11, g01];
    3D [e00, e11, e22, g12, g02, g01] (engineering shear strains)."""
    if dim == 2:
        return E / (1.0 - nu * nu) * np.array([[1.0, nu, 0.0],
                                               [nu, 1.0, 0.0],
                                               [0.0, 0.0, (1.0 - nu) / 2.0]])
    lam = E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    D = np.zeros((6, 6))
    D[:3, :3] = lam
    D[np.arange(3), np.arange(3)] += 2.0 * mu
    D[3, 3] = D[4, 4] = D[5, 5] = mu
    return D


VOIGT_SHEAR = {2: [(0, 1)], 3: [(1, 2), (0, 2), (0, 1)]}


def strain_displacement(dim: int, xi, nodes=None) -> np.ndarray:
    """B(xi): Voigt strain = B @ u_e, u_e with local DOF d*a + comp."""
    g = shape_grad(dim, xi, nodes)
    na = g.shape[0]
    nv = 3 if dim == 2 else 6
    B = np.zeros((nv, dim * na))
    for a in range(na):
        for i in range(dim):
            B[i, dim * a + i] = g[a, i]                     # normal strains
        for s, (i, j) in enumerate(VOIGT_SHEAR[dim]):
            B[dim + s, dim * a + i] += g[a, j]              # du_i/dx_j
            B[dim + s, dim * a + j] += g[a, i]              # du_j/dx_i
    return B


def gauss_points(dim: int):
    for pt in itertools.product(GAUSS_1D, repeat=dim):
        yield np.array(pt), 0.5 ** dim


def element_stiffness(dim: int, nu: float = 0.3, E: float = 1.0, nodes=None) -> np.ndarray:
    """K_e0 = int B^T D0 B over the unit element, exact 2x2(x2) Gauss."""
    D = constitutive(dim, E, nu)
    n = dim * (2 ** dim)
    K = np.zeros((n, n))
    for xi, w in gauss_points(dim):
        B = strain_displacement(dim, xi, nodes)
        K += w * B.T @ D @ B
    return K


def element_stiffness_wilson(dim: int, nu: float = 0.3, E: float = 1.0) -> np.ndarray:
    """Incompatible-mode element (Wilson et al.; "Wilson quadrilaterals in 2D",
    hexahedra in 3D): the displacement field is enriched per
    component with the bubble modes M_k = 1 - xi_k^2 (xi_k = 2 x_k - 1 in [-1, 1], k < d), whose
    DOFs are condensed statically on the unit element (material constant per element):
        K_e0 = K_cc - K_ci K_ii^-1 K_ic,   K = int [B_c B_i]^T D0 [B_c B_i], exact 2x2(x2) Gauss.
    Incompatible DOF (comp c, mode k) has strain dM_k/dx_j = -4 (2 x_k - 1) delta_kj."""
    D = constitutive(dim, E, nu)
    na = 2 ** dim
    nv = 3 if dim == 2 else 6
    n, ninc = dim * na, dim * dim
    K = np.zeros((n + ninc, n + ninc))
    for xi, w in gauss_points(dim):
        Bc = strain_displacement(dim, xi)
        Bi = np.zeros((nv, ninc))
        for k in range(dim):
            dM = np.zeros(dim)
            dM[k] = -4.0 * (2.0 * xi[k] - 1.0)
            for c in range(dim):
                col = c * dim + k
                Bi[c, col] += dM[c]
                for s, (i, j) in enumerate(VOIGT_SHEAR[dim]):
                    if c == i:
                        Bi[dim + s, col] += dM[j]
                    if c == j:
                        Bi[dim + s, col] += dM[i]
        B = np.hstack([Bc, Bi])
        K += w * B.T @ D @ B
    Kcc, Kci, Kii = K[:n, :n], K[:n, n:], K[n:, n:]
    return Kcc - Kci @ np.linalg.solve(Kii, Kci.T)


def element_stiffness_of(element: str, dim: int, nu: float = 0.3) -> np.ndarray:
    """K_e0 of the element type: "std" (bilinear / trilinear) or "wilson" (incompatible modes)."""
    if element == "wilson":
        return element_stiffness_wilson(dim, nu)
    return element_stiffness(dim, nu)


def geometric_H(dim: int, nodes=None) -> np.ndarray:
    """H[i, j, a, b] = int dN_a/dx_i dN_b/dx_j over the unit element (exact Gauss)."""
    na = 2 ** dim
    H = np.zeros((dim, dim, na, na))
    for xi, w in gauss_points(dim):
        g = shape_grad(dim, xi, nodes)
        H += w * np.einsum("ai,bj->ijab", g, g)
    return H


def centroid_stress(dim: int, u_e: np.ndarray, nu: float = 0.3) -> np.ndarray:
    """sigma = D0 B(centroid) u_e as a symmetric d x d tensor (SPEC.md:153 /
    SURVEY r15: stress at the element centroid, tension positive).
    u_e: (..., d*2^d) -> (..., d, d)."""
    B = strain_displacement(dim, np.full(dim, 0.5))
    s = np.einsum("vk,...k->...v", constitutive(dim, 1.0, nu) @ B, u_e)
    T = np.zeros(u_e.shape[:-1] + (dim, dim))
    for i in range(dim):
        T[..., i, i] = s[..., i]
    for q, (i, j) in enumerate(VOIGT_SHEAR[dim]):
        T[..., i, j] = s[..., dim + q]
        T[..., j, i] = s[..., dim + q]
    return T


def element_geometric(dim: int, u_e: np.ndarray, nu: float = 0.3) -> np.ndarray:
    """G_e0[u_e] = (sum_ij sigma_ij H_ij) kron I_d.  The same for the
    incompatible-mode element: the bubble gradients vanish at the centroid, so the recovered
    incompatible DOFs do not change the centroid stress."""
    sig = centroid_stress(dim, u_e, nu)
    S = np.einsum("ij,ijab->ab", sig, geometric_H(dim))
    return np.kron(S, np.eye(dim))
