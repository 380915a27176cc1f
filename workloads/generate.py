"""Seeded synthetic input recipe (BASELINE.json configs).

Everything here is *input preparation*: it produces the element moduli E_e,
stress moduli Es_e, the fixed-DOF mask and the right-hand sides that both the
oracle and the CUDA path receive.  Layout (SURVEY.md 8(b) conventions):

* vectors are RHS-major (nrhs, n); DOF index = d*node + comp;
* nodes in C order over (N0+1, N1+1[, N2+1]) (axis 0 slowest);
* E_e in C order over (N0, N1[, N2]);
* comp c is the displacement along axis c.
"""

from __future__ import annotations

import numpy as np
from scipy import ndimage, signal

from .configs import Config, n_dofs


def element_grid_shape(nel):
    return tuple(nel)


def node_grid_shape(nel):
    return tuple(n + 1 for n in nel)


def _cone_kernel(r: float, dim: int) -> np.ndarray:
    """Cone weights max(0, r - dist) on the integer lattice ("standard
    density filter"; cone shape per SPEC.md:183 / SURVEY r7)."""
    k = int(np.ceil(r)) - 1 if float(r).is_integer() else int(np.floor(r))
    ax = np.arange(-k, k + 1, dtype=np.float64)
    grids = np.meshgrid(*([ax] * dim), indexing="ij")
    dist = np.sqrt(sum(g * g for g in grids))
    return np.maximum(0.0, r - dist)


def cone_filter(field: np.ndarray, r: float, use_fft: bool = False) -> np.ndarray:
    """Normalised cone filter over in-domain neighbours (no padding)."""
    w = _cone_kernel(r, field.ndim)
    if use_fft:
        num = signal.fftconvolve(field, w, mode="same")
        den = signal.fftconvolve(np.ones_like(field), w, mode="same")
    else:
        num = ndimage.correlate(field, w, mode="constant", cval=0.0)
        den = ndimage.correlate(np.ones_like(field), w, mode="constant", cval=0.0)
    return num / den


def heaviside_projection(xt: np.ndarray, beta: float, eta: float) -> np.ndarray:
    """Eq. (1)."""
    tb = np.tanh(beta * eta)
    return (tb + np.tanh(beta * (xt - eta))) / (tb + np.tanh(beta * (1.0 - eta)))


def _trapezoid(nseg: int) -> np.ndarray:
    """Consistent nodal weights of a unit total load spread uniformly over nseg
    unit segments (ends 1/(2N), interior 1/N)."""
    w = np.full(nseg + 1, 1.0 / nseg)
    w[0] = w[-1] = 0.5 / nseg
    return w


def fixed_mask(cfg: Config) -> np.ndarray:
    """uint8 per DOF, 1 = fixed.  "base": every DOF on node plane i0 = 0."""
    nshape = node_grid_shape(cfg.nel)
    m = np.zeros(nshape + (cfg.dim,), dtype=np.uint8)
    if cfg.bc == "base":
        m[0] = 1
    else:
        raise ValueError(cfg.bc)
    return m.reshape(-1)


def state_load(cfg: Config) -> np.ndarray:
    """Unit total consistent load."""
    nshape = node_grid_shape(cfg.nel)
    f = np.zeros(nshape + (cfg.dim,))
    N0 = cfg.nel[0]
    if cfg.load == "top":
        # plane i0 = N0, along -axis 0 (compression); tensor trapezoid weights
        w = _trapezoid(cfg.nel[1])
        for nseg in cfg.nel[2:]:
            w = np.multiply.outer(w, _trapezoid(nseg))
        f[N0, ..., 0] = -w
    elif cfg.load == "edge":
        # edge {i0 = N0, i1 = 0, all i2}, along -axis 1
        assert cfg.dim == 3
        f[N0, 0, :, 1] = -_trapezoid(cfg.nel[2])
    else:
        raise ValueError(cfg.load)
    return f.reshape(-1)


def generate(cfg: Config, with_phi: bool = True) -> dict:
    """Build all inputs of config `cfg` from numpy default_rng(cfg.seed).

    Draw order: densities first (rng.random(nel), C order), then the
    adjoint fields k = 1..R-1 (rng.standard_normal((*nodes, d))).
    Returns dict with E, Es (m,), fixed (n,) uint8, rhs (R, n), phi (nphi, n).
    """
    rng = np.random.default_rng(cfg.seed)
    d = cfg.dim
    nshape = node_grid_shape(cfg.nel)
    n = n_dofs(cfg.nel)
    rho_raw = rng.random(cfg.nel)
    rho_f = cone_filter(rho_raw, cfg.rmin)
    rho = heaviside_projection(rho_f, cfg.beta, cfg.eta)
    rp = rho ** cfg.penal
    E = (cfg.Emin + rp * (cfg.E0 - cfg.Emin)).reshape(-1)      # Eq. 2, E_kappa
    Es = (rp * cfg.E0).reshape(-1)                              # Eq. 2, E_sigma
    fixed = fixed_mask(cfg)
    free = 1.0 - fixed
    rhs = np.empty((cfg.nrhs, n))
    rhs[0] = state_load(cfg) * free
    big = np.prod(nshape) > 200_000
    for k in range(1, cfg.nrhs):
        g = rng.standard_normal(nshape + (d,))
        sm = np.stack([cone_filter(g[..., c], cfg.rhs_rmin, use_fft=big) for c in range(d)], axis=-1)
        v = sm.reshape(-1) * free
        rhs[k] = v / np.linalg.norm(v)
    out = dict(cfg=cfg, E=np.ascontiguousarray(E), Es=np.ascontiguousarray(Es),
               fixed=fixed, rhs=rhs, rho=rho.reshape(-1))
    if with_phi and cfg.nphi:
        # r16: phi = the adjoint-RHS fields (smooth, unit norm); extra draws if R-1 < nphi
        phis = [rhs[1 + k] for k in range(min(cfg.nphi, cfg.nrhs - 1))]
        while len(phis) < cfg.nphi:
            g = rng.standard_normal(nshape + (d,))
            sm = np.stack([cone_filter(g[..., c], cfg.rhs_rmin, use_fft=big) for c in range(d)], axis=-1)
            v = sm.reshape(-1) * free
            phis.append(v / np.linalg.norm(v))
        out["phi"] = np.ascontiguousarray(np.stack(phis))
    return out


def rough_vectors(cfg: Config, nvec: int, seed_offset: int = 777, masked: bool = False) -> np.ndarray:
    """iid N(0,1) vectors (matvec parity is measured on rough inputs)."""
    rng = np.random.default_rng(cfg.seed + seed_offset)
    v = rng.standard_normal((nvec, n_dofs(cfg.nel)))
    if masked:
        v *= 1.0 - fixed_mask(cfg)
    return v
