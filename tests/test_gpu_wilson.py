"""NEXT-4 on the GPU: the incompatible-mode element of the paper
 through the same kernels -- matvec and solve parity against the oracle with the
oracle's own condensed element (oracle/fem.element_stiffness_wilson, pinned by the exact pure
bending energy and the patch test), 2D and 3D, one and several slabs."""

import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, solve  # noqa: E402
from workloads import generate, get_config, rough_vectors  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@functools.lru_cache(maxsize=None)
def case(name):
    cfg = get_config(name)
    inp = generate(cfg)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"], element="wilson")
    return cfg, inp, K


def handle(name, nslab=1):
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    if nslab == 1:
        return mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels, element="wilson")
    return mg.mg_setup_dist(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels, nslab=nslab,
                            element="wilson")


def rel(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


@pytest.mark.parametrize("name,nslab", [("T2a", 1), ("T2b", 1), ("C2", 1), ("T3a", 1), ("T3c", 1), ("T2c", 3),
                                        ("T3b", 2)])
def test_wilson_matvec_parity(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    X = rough_vectors(cfg, 2)
    y = torch.empty((2, X.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_matvec(handle(name, nslab), 0, to_dev(X), y)
    assert rel(y.cpu().numpy(), (K @ X.T).T).max() < 1e-13


@pytest.mark.parametrize("name,nslab", [("T2a", 1), ("T2c", 1), ("T3a", 1), ("T3b", 1), ("T2b", 2), ("T3c", 2)])
def test_wilson_solve_parity(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    U = solve.direct_solve(K, inp["rhs"], inp["fixed"])
    x = torch.empty((cfg.nrhs, U.shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(handle(name, nslab), to_dev(inp["rhs"]), cfg.tol, x, raise_on_error=False)
    assert rep["status"] == "MG_OK", rep
    assert rel(x.cpu().numpy(), U).max() < 1e-8


def test_wilson_galerkin_levels():
    import paper_1909_13585_b200 as mg
    from oracle import mg as omg
    cfg, inp, K = case("T2c")
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    h = handle("T2c")
    rng = np.random.default_rng(3)
    for l in range(1, cfg.levels):
        n = H.A[l].shape[0]
        X = rng.standard_normal((2, n))
        y = torch.empty((2, n), dtype=torch.float64, device=DEV)
        mg.mg_matvec(h, l, to_dev(X), y)
        assert rel(y.cpu().numpy(), (H.A[l] @ X.T).T).max() < 1e-13
