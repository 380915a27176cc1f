"""Slab decomposition on one GPU: nslab slabs in one handle exchange their
ghost planes by device copies, through the same code path NCCL ranks use for remote
neighbours.  Every result must match the CPU oracle to the single-GPU bars, and the
preconditioner must equal the undecomposed one up to summation order."""

import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, solve  # noqa: E402
from workloads import generate, get_config, rough_vectors  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@functools.lru_cache(maxsize=None)
def case(name):
    cfg = get_config(name)
    inp = generate(cfg)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    return cfg, inp, K


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def rel(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


def handle(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    return mg.mg_setup_dist(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels, nslab=nslab)


# (config, slabs): uneven splits, 2D and 3D, slabs down to one coarsest layer
SLAB_CASES = [("T2b", 2), ("T2b", 3), ("T2c", 4), ("C2", 4), ("T3a", 2), ("T3b", 3), ("T3c", 4), ("T3d", 5), ("T3f", 2)]


@pytest.mark.parametrize("name,nslab", SLAB_CASES)
def test_slab_matvec_parity_rough(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    h = handle(name, nslab)
    X = rough_vectors(cfg, 3)
    y = torch.empty((3, X.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_matvec(h, 0, to_dev(X), y)
    assert rel(y.cpu().numpy(), (K @ X.T).T).max() < 1e-13


@pytest.mark.parametrize("name,nslab", SLAB_CASES)
def test_slab_vcycle_equals_single_slab(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    A = rough_vectors(cfg, 2, seed_offset=31, masked=True)
    Z1 = torch.empty((2, A.shape[1]), dtype=torch.float64, device=DEV)
    Zs = torch.empty_like(Z1)
    mg.mg_vcycle(handle(name, 1), to_dev(A), Z1)
    mg.mg_vcycle(handle(name, nslab), to_dev(A), Zs)
    assert rel(Zs.cpu().numpy(), Z1.cpu().numpy()).max() < 1e-11


@pytest.mark.parametrize("name,nslab", SLAB_CASES)
def test_slab_solve_parity_direct(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    U = solve.direct_solve(K, inp["rhs"], inp["fixed"])
    h = handle(name, nslab)
    x = torch.empty((cfg.nrhs, U.shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x, raise_on_error=False)
    assert rep["status"] == "MG_OK", rep
    assert rel(x.cpu().numpy(), U).max() < 1e-8
    res = inp["rhs"] - (K @ x.cpu().numpy().T).T
    assert (np.linalg.norm(res, axis=1) / np.linalg.norm(inp["rhs"], axis=1)).max() <= 2 * cfg.tol
    # same preconditioner => same iteration counts as one slab (up to rounding at the threshold)
    x1 = torch.empty_like(x)
    rep1 = mg.mgcg_solve(handle(name, 1), to_dev(inp["rhs"]), cfg.tol, x1)
    assert all(abs(a - b) <= 1 for a, b in zip(rep["iters"], rep1["iters"]))


@pytest.mark.parametrize("name,nslab", [("T2b", 3), ("T3a", 2), ("T3c", 4)])
def test_slab_stress_stiffness_parity(name, nslab):
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    h = handle(name, nslab)
    u = rough_vectors(cfg, 1, seed_offset=5)[0]
    phi = rough_vectors(cfg, 2, seed_offset=9)
    y = torch.empty((2, phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.stress_stiffness_apply(h, to_dev(inp["Es"]), to_dev(u), to_dev(phi), y)
    G = assemble.assemble_G(cfg.nel, inp["Es"], u, inp["fixed"])
    assert rel(y.cpu().numpy(), (G @ phi.T).T).max() < 1e-13


def test_dist_single_slab_is_mg_setup_bitwise():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2c")
    rhs = to_dev(inp["rhs"])
    x0 = torch.empty_like(rhs)
    x1 = torch.empty_like(rhs)
    mg.mgcg_solve(mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels), rhs, 1e-10, x0)
    mg.mgcg_solve(handle("T2c", 1), rhs, 1e-10, x1)
    assert torch.equal(x0, x1)


def test_slab_update_modulus_and_host_buffers():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T3b")
    h = handle("T3b", 3)
    E2 = inp["E"][::-1].copy()
    mg.mg_update_modulus(h, to_dev(E2))
    K2 = assemble.assemble_K(cfg.nel, E2, inp["fixed"])
    U = solve.direct_solve(K2, inp["rhs"], inp["fixed"])
    xh = np.empty_like(inp["rhs"])
    mg.mgcg_solve(h, np.ascontiguousarray(inp["rhs"]), 1e-10, xh)
    assert rel(xh, U).max() < 1e-8


_STAGE_SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_1909_13585_b200 as mg
from workloads import generate, get_config
out = {}
for name, nslab in %(cases)r:
    cfg = get_config(name)
    inp = generate(cfg)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    h = mg.mg_setup_dist(cfg.nel, d(inp["E"]), d(inp["fixed"]), cfg.levels, nslab=nslab)
    x = torch.empty((cfg.nrhs, inp["rhs"].shape[1]), dtype=torch.float64, device="cuda")
    mg.mgcg_solve(h, d(inp["rhs"]), 1e-10, x)
    out[name + str(nslab)] = x.cpu().numpy().tobytes().hex()
print(json.dumps(out))
"""


def test_packed_halo_messages_bitwise():
    """MG_COMM_STAGE=1 routes the in-process neighbour exchanges through the packed-message path
    of the cross-rank exchange (all vectors of a boundary plane packed into one contiguous
    message, moved, unpacked); data movement only, so the solves are bitwise those of the direct
    plane copies."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cases = [("T2b", 3), ("C2", 4), ("T3b", 3), ("T3d", 5)]
    res = {}
    for st in ("0", "1"):
        p = subprocess.run([sys.executable, "-c", _STAGE_SCRIPT % {"root": root, "cases": cases}],
                           env=dict(os.environ, MG_COMM_STAGE=st), capture_output=True, text=True, timeout=900,
                           cwd=root)
        assert p.returncode == 0, p.stderr[-2000:]
        res[st] = json.loads(p.stdout.strip().splitlines()[-1])
    for k in res["0"]:
        assert res["0"][k] == res["1"][k], k
