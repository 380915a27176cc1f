"""Element-by-element products on the structured grid (oracle; TEST INFRASTRUCTURE ONLY).

Same definitions as `assemble`, evaluated
without forming the sparse matrix, so that they reach sizes where assembly does
not fit (C3 residuals, C5), and in extended precision (np.longdouble) for the
direct solve's refinement residual (SURVEY 8(c) "C3: direct").

Dirichlet convention as in `assemble`: y = F K F x + (I - F) x for K and
y = F G F phi for G, F = diag(free).
"""

from __future__ import annotations

import numpy as np

from . import fem


def _slices(bits, nel):
    return tuple(slice(b, b + n) for b, n in zip(bits, nel))


def matvec(nel, E, fixed, x, nu=0.3, dtype=np.float64, element="std"):
    """y = K x for one vector x (n,) or a batch (R, n)."""
    x = np.asarray(x)
    if x.ndim == 2:
        return np.stack([matvec(nel, E, fixed, xi, nu, dtype, element) for xi in x])
    dim = len(nel)
    nsh = tuple(n + 1 for n in nel) + (dim,)
    K0 = fem.element_stiffness_of(element, dim, nu).astype(dtype)
    free = (1 - np.asarray(fixed).astype(dtype)).reshape(nsh)
    xg = x.astype(dtype).reshape(nsh) * free
    Eg = np.asarray(E).astype(dtype).reshape(tuple(nel) + (1,))
    bits = fem.local_nodes(dim)
    nl = dim * len(bits)
    # element DOF vectors x_e (local DOF d*a + comp), element products y_e = E_e K0 x_e, then the
    # gather-sum of y_e into the nodes of each element (K = sum_e E_e A_e^T K0 A_e)
    xe = np.concatenate([xg[_slices(bb, nel)] for bb in bits], axis=-1)          # (*nel, nl)
    ye = (xe.reshape(-1, nl) @ K0.T).reshape(xe.shape) * Eg
    y = np.zeros(nsh, dtype=dtype)
    for b, bb in enumerate(bits):
        y[_slices(bb, nel)] += ye[..., b * dim:(b + 1) * dim]
    y = y * free + (1 - free) * x.astype(dtype).reshape(nsh)
    return y.reshape(-1)


def matvec_rows(nel, E, fixed, x, nodes, nu=0.3, element="std"):
    """Rows of y = K x at the given node indices only: returns (len(nodes), d).
    Each row sums the 2^d adjacent elements one by one (sampled parity at full size)."""
    dim = len(nel)
    nn = np.array([n + 1 for n in nel])
    K0 = fem.element_stiffness_of(element, dim, nu)
    x = np.asarray(x, dtype=np.float64)
    fixed = np.asarray(fixed)
    E = np.asarray(E, dtype=np.float64)
    bits = fem.local_nodes(dim)
    strides_n = [int(np.prod(nn[k + 1:])) for k in range(dim)]
    strides_e = [int(np.prod(nel[k + 1:])) for k in range(dim)]
    out = np.zeros((len(nodes), dim))
    for s, p in enumerate(nodes):
        coords = np.array(np.unravel_index(int(p), tuple(nn)))
        pf = 1.0 - fixed[dim * p: dim * p + dim]
        acc = np.zeros(dim)
        for b, bb in enumerate(bits):
            ec = coords - bb
            if np.any(ec < 0) or np.any(ec >= np.array(nel)):
                continue
            e = int(sum(int(c) * st for c, st in zip(ec, strides_e)))
            xe = np.zeros(dim * len(bits))
            for a, ab in enumerate(bits):
                q = int(sum(int(c) * st for c, st in zip(ec + ab, strides_n)))
                xe[dim * a:dim * a + dim] = x[dim * q:dim * q + dim] * (1.0 - fixed[dim * q:dim * q + dim])
            acc += E[e] * (K0[b * dim:(b + 1) * dim] @ xe)
        out[s] = pf * acc + (1.0 - pf) * x[dim * p:dim * p + dim]
    return out


def stress_stiffness_apply(nel, Es, fixed, u, phi, nu=0.3):
    """y = G(u) phi for phi (n,) or (nphi, n), without assembling G."""
    phi = np.asarray(phi)
    dim = len(nel)
    nsh = tuple(n + 1 for n in nel) + (dim,)
    free = (1 - np.asarray(fixed).astype(np.float64)).reshape(nsh)
    ug = np.asarray(u, dtype=np.float64).reshape(nsh)
    bits = fem.local_nodes(dim)
    ue = np.concatenate([ug[_slices(bb, nel)] for bb in bits], axis=-1)   # (*nel, d*2^d)
    sig = fem.centroid_stress(dim, ue, nu) * np.asarray(Es, dtype=np.float64).reshape(tuple(nel) + (1, 1))
    H = fem.geometric_H(dim)
    S = np.einsum("...ij,ijab->...ab", sig, H)                           # (*nel, na, na)
    single = phi.ndim == 1
    phis = phi[None] if single else phi
    outs = []
    for ph in phis:
        pg = ph.reshape(nsh) * free
        pa = [pg[_slices(bb, nel)] for bb in bits]
        y = np.zeros(nsh)
        for b, bb in enumerate(bits):
            acc = np.zeros(tuple(nel) + (dim,))
            for a in range(len(bits)):
                acc += S[..., b, a][..., None] * pa[a]
            y[_slices(bb, nel)] += acc
        outs.append((y * free).reshape(-1))
    return outs[0] if single else np.stack(outs)
