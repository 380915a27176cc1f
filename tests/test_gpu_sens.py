"""NEXT-1 on the GPU: adjoint right-hand sides (Eq. 5) and element
sensitivities (Eq. 4) through the C ABI against the pinned oracle (oracle/sens.py)."""

import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, sens, solve  # noqa: E402
from workloads import generate, get_config, rough_vectors  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@functools.lru_cache(maxsize=None)
def case(name):
    cfg = get_config(name)
    return cfg, generate(cfg)


@pytest.mark.parametrize("name", ["T2a", "T2b", "C1", "T3a", "T3c"])
def test_adjoint_rhs_parity(name):
    import paper_1909_13585_b200 as mg
    cfg, inp = case(name)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    phi = rough_vectors(cfg, 3, seed_offset=41)
    b = torch.empty((3, phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_adjoint_rhs(h, to_dev(inp["Es"]), to_dev(phi), b)
    ref = sens.adjoint_rhs(cfg.nel, inp["Es"], inp["fixed"], phi)
    got = b.cpu().numpy()
    assert (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max() < 1e-13


@pytest.mark.parametrize("name", ["T2a", "T2c", "T3a", "T3b"])
def test_eigen_sensitivity_parity(name):
    import paper_1909_13585_b200 as mg
    cfg, inp = case(name)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    u = solve.direct_solve(K, inp["rhs"][0], inp["fixed"])
    phi = rough_vectors(cfg, 2, seed_offset=43)
    z = rough_vectors(cfg, 2, seed_offset=47)
    lam = [0.37, 1.9]
    rng = np.random.default_rng(9)
    dEk = rng.uniform(0.1, 3.0, len(inp["E"]))
    dEs = rng.uniform(0.1, 3.0, len(inp["E"]))
    out = torch.empty((2, len(inp["E"])), dtype=torch.float64, device=DEV)
    mg.mg_eigen_sensitivity(h, to_dev(dEk), to_dev(dEs), to_dev(u), to_dev(phi), to_dev(z), lam, out)
    got = out.cpu().numpy()
    for i in range(2):
        ref = sens.eigen_sensitivity(cfg.nel, inp["fixed"], u, phi[i], z[i], lam[i], dEk, dEs)
        assert np.abs(got[i] - ref).max() <= 1e-13 * np.abs(ref).max()


def test_adjoint_pipeline_on_gpu_matches_oracle():
    """phi -> b (GPU) -> z by mgcg_solve (GPU) -> Eq. 4 (GPU) equals the oracle pipeline."""
    import paper_1909_13585_b200 as mg
    cfg, inp = case("T2b")
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    u = solve.direct_solve(K, inp["rhs"][0], inp["fixed"])
    phi = inp["rhs"][1:3]                                   # smooth fields as stand-in modes
    b = torch.empty((2, phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_adjoint_rhs(h, to_dev(inp["Es"]), to_dev(phi), b)
    z = torch.empty_like(b)
    mg.mgcg_solve(h, b, 1e-10, z)
    rng = np.random.default_rng(4)
    dEk = rng.uniform(0.1, 3.0, len(inp["E"]))
    dEs = rng.uniform(0.1, 3.0, len(inp["E"]))
    lam = [0.5, 0.8]
    out = torch.empty((2, len(inp["E"])), dtype=torch.float64, device=DEV)
    mg.mg_eigen_sensitivity(h, to_dev(dEk), to_dev(dEs), to_dev(u), to_dev(phi), z, lam, out)
    bo = sens.adjoint_rhs(cfg.nel, inp["Es"], inp["fixed"], phi)
    zo = solve.direct_solve(K, bo, inp["fixed"])
    for i in range(2):
        ref = sens.eigen_sensitivity(cfg.nel, inp["fixed"], u, phi[i], zo[i], lam[i], dEk, dEs)
        assert np.abs(out.cpu().numpy()[i] - ref).max() <= 1e-8 * np.abs(ref).max()


@pytest.mark.parametrize("name,nslab", [("T2b", 3), ("T2c", 4), ("T3b", 3), ("T3d", 5)])
def test_next1_on_slabs_parity(name, nslab):
    """NEXT-1 on a slab decomposition (in-process slabs: the halo path NCCL ranks use): the
    adjoint right-hand sides and the Eq. 4 element sensitivities against the oracle, same bars."""
    import paper_1909_13585_b200 as mg
    cfg, inp = case(name)
    h = mg.mg_setup_dist(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels, nslab=nslab)
    phi = rough_vectors(cfg, 3, seed_offset=41)
    b = torch.empty((3, phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_adjoint_rhs(h, to_dev(inp["Es"]), to_dev(phi), b)
    ref = sens.adjoint_rhs(cfg.nel, inp["Es"], inp["fixed"], phi)
    got = b.cpu().numpy()
    assert (np.linalg.norm(got - ref, axis=1) / np.linalg.norm(ref, axis=1)).max() < 1e-13
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    u = solve.direct_solve(K, inp["rhs"][0], inp["fixed"])
    z = rough_vectors(cfg, 3, seed_offset=47)
    lam = [0.37, 1.9, 0.8]
    rng = np.random.default_rng(9)
    dEk = rng.uniform(0.1, 3.0, len(inp["E"]))
    dEs = rng.uniform(0.1, 3.0, len(inp["E"]))
    out = torch.empty((3, len(inp["E"])), dtype=torch.float64, device=DEV)
    mg.mg_eigen_sensitivity(h, to_dev(dEk), to_dev(dEs), to_dev(u), to_dev(phi), to_dev(z), lam, out)
    got = out.cpu().numpy()
    for i in range(3):
        ref = sens.eigen_sensitivity(cfg.nel, inp["fixed"], u, phi[i], z[i], lam[i], dEk, dEs)
        assert np.abs(got[i] - ref).max() <= 1e-13 * np.abs(ref).max()
