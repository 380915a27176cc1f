"""NEXT-2 on the GPU: the multilevel mode approximation through
the C ABI against the pinned oracle pipeline (oracle/modes.py) -- coarse BLFs, fine Rayleigh
quotients and the fine mode shapes (up to sign)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, modes, solve  # noqa: E402
from workloads import generate, get_config  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@pytest.mark.parametrize("name,q", [("T2a", 3), ("T2c", 4), ("C1", 6), ("T3a", 3), ("T3b", 2)])
def test_multilevel_modes_parity(name, q):
    import paper_1909_13585_b200 as mg
    cfg = get_config(name)
    inp = generate(cfg)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    u = solve.direct_solve(K, inp["rhs"][0], inp["fixed"])
    lam_c, Psi, Phi, lam_t = modes.multilevel_modes(cfg.nel, inp["E"], inp["Es"], inp["fixed"], u, cfg.levels, q)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    P = torch.empty((q, Phi.shape[1]), dtype=torch.float64, device=DEV)
    y1 = torch.empty(Phi.shape[1], dtype=torch.float64, device=DEV)
    lt, lc, (ynorm, yrel) = mg.mg_multilevel_modes(h, to_dev(inp["Es"]), to_dev(u), q, P, y1=y1, with_residual=True)
    assert np.allclose(lc, lam_c, rtol=1e-9), (lc, lam_c)
    assert np.allclose(lt, lam_t, rtol=1e-9), (lt, lam_t)
    Pg = P.cpu().numpy()
    # K-normalised modes: phi~^T K phi~ = 1 on the GPU result, by the oracle's K
    assert np.allclose(np.einsum("in,in->i", Pg, (K @ Pg.T).T), 1.0, rtol=1e-10)
    for i in range(q):
        s = np.sign(Pg[i] @ Phi[i])
        assert np.linalg.norm(s * Pg[i] - Phi[i]) / np.linalg.norm(Phi[i]) < 1e-8
    # Eq. 7 residual of the first pair vs the oracle's (same sign convention as phi~_1)
    y = modes.eigen_residual(cfg.nel, inp["E"], inp["Es"], inp["fixed"], u, lam_t[0], Phi[0])
    s0 = np.sign(Pg[0] @ Phi[0])
    yg = y1.cpu().numpy()
    assert np.linalg.norm(s0 * yg - y) <= 1e-8 * np.linalg.norm(K @ Phi[0])
    assert abs(ynorm - np.linalg.norm(y)) <= 1e-8 * np.linalg.norm(K @ Phi[0])
    assert abs(yrel - np.linalg.norm(y) / np.linalg.norm(K @ Phi[0])) <= 1e-8
    assert abs(Pg[0] @ yg) <= 1e-10 * np.linalg.norm(K @ Pg[0]) * np.linalg.norm(Pg[0])   # phi~_1^T y = 0
