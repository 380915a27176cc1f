"""Parity at BASELINE.json's full sizes (C3, C4, C5) in the launch configuration bench.py times
(one handle, all R right-hand sides, the config's levels).  The oracle cannot assemble or
factor these systems in seconds, so (task ③):
  * matvec and G(u) phi: sampled output rows, each computed one by one by the oracle
    (element-by-element, oracle/ebe.py), at 1e-13 relative;
  * solve: the true residual of the GPU solution, evaluated by the oracle's own EbE operator
    (a property that holds at any size), and for C3 / C4 the solution itself against the
    oracle's independent iterative solve (scipy MG-PCG to 1e-13), at 1e-8 relative L2.
"""

import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, ebe, solve  # noqa: E402
from workloads import generate, get_config, rough_vectors  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


@functools.lru_cache(maxsize=None)
def inputs(name):
    cfg = get_config(name)
    return cfg, generate(cfg)


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def sample_nodes(nel, count, seed):
    """Random nodes plus the structural edge cases: domain faces, the first / last planes,
    kernel chunk and tile boundaries along every axis."""
    nn = [n + 1 for n in nel]
    rng = np.random.default_rng(seed)
    pts = [tuple(rng.integers(0, m) for m in nn) for _ in range(count)]
    special = []
    for k, m in enumerate(nn):
        for v in (0, 1, 5, 6, 7, 29, 30, 31, 32, 33, 63, 64, 65, m // 2, m - 2, m - 1):
            if 0 <= v < m:
                p = [rng.integers(0, mm) for mm in nn]
                p[k] = v
                special.append(tuple(p))
    pts += special + [tuple(0 for _ in nn), tuple(m - 1 for m in nn)]
    return np.array([np.ravel_multi_index(p, nn) for p in pts], dtype=np.int64)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_matvec_sampled_rows(name):
    import paper_1909_13585_b200 as mg
    cfg, inp = inputs(name)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    X = rough_vectors(cfg, cfg.nrhs, seed_offset=101)
    Y = torch.empty((cfg.nrhs, X.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_matvec(h, 0, to_dev(X), Y)
    Y = Y.cpu().numpy()
    d = cfg.dim
    nodes = sample_nodes(cfg.nel, 150, seed=7)
    for k in (0, cfg.nrhs - 1):
        ref = ebe.matvec_rows(cfg.nel, inp["E"], inp["fixed"], X[k], nodes)
        got = np.stack([Y[k, d * p:d * p + d] for p in nodes])
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-13
        assert np.abs(got - ref).max() <= 1e-13 * np.abs(ref).max()


def _solve_fullsize(name):
    import paper_1909_13585_b200 as mg
    cfg, inp = inputs(name)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    x = torch.empty((cfg.nrhs, inp["rhs"].shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x, raise_on_error=False)
    return cfg, inp, rep, x.cpu().numpy()


@functools.lru_cache(maxsize=None)
def solved(name):
    return _solve_fullsize(name)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_solve_true_residual_by_oracle_operator(name):
    cfg, inp, rep, X = solved(name)
    assert rep["status"] == "MG_OK", rep
    assert max(rep["true_relres"]) <= cfg.tol
    for k in (0, 1):   # state RHS and the first adjoint RHS
        res = inp["rhs"][k] - ebe.matvec(cfg.nel, inp["E"], inp["fixed"], X[k])
        assert np.linalg.norm(res) / np.linalg.norm(inp["rhs"][k]) <= 2 * cfg.tol


@pytest.mark.parametrize("name,ks", [("C3", (0,)), ("C4", (0, 1))])
def test_fullsize_solution_vs_iterative_oracle(name, ks):
    cfg, inp, rep, X = solved(name)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    U, _ = solve.mgpcg_solve(cfg.nel, K, inp["rhs"][list(ks)], inp["fixed"], cfg.levels, tol=1e-13)
    for i, k in enumerate(ks):
        assert np.linalg.norm(X[k] - U[i]) / np.linalg.norm(U[i]) < 1e-8


def test_fullsize_stress_stiffness_C3():
    """G(u) phi for the 12 phi of C3 with u the GPU state solution (reading r16); two of the
    products checked in full against the oracle's EbE G(u) phi."""
    import paper_1909_13585_b200 as mg
    cfg, inp, rep, X = solved("C3")
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    phi = inp["phi"]
    y = torch.empty((phi.shape[0], phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.stress_stiffness_apply(h, to_dev(inp["Es"]), to_dev(X[0]), to_dev(phi), y)
    y = y.cpu().numpy()
    ref = ebe.stress_stiffness_apply(cfg.nel, inp["Es"], inp["fixed"], X[0], phi[[0, 11]])
    for i, k in enumerate((0, 11)):
        # smooth inputs: normalise by ||G|| ||phi|| scale -> use max-abs relative
        assert np.abs(y[k] - ref[i]).max() <= 1e-12 * np.abs(ref[i]).max()
