"""Parity at BASELINE.json's full sizes (C3, C4, C5) in the launch configuration bench.py times
(one handle, all R right-hand sides, the config's levels).  The oracle cannot assemble or
factor these systems in seconds, so (task ③):
  * matvec and G(u) phi: sampled output rows, each computed one by one by the oracle
    (element-by-element, oracle/ebe.py), at 1e-13 relative;
  * solve: for every right-hand side, the true residual of the GPU solution evaluated by the
    oracle's own EbE operator (a property that holds at any size); for C3 / C4 every solution
    against the oracle's independent iterative solve (scipy MG-PCG to 1e-13), at 1e-8 relative
    L2; for C5 against the same oracle's solution stored at sampled DOFs (plus its norm and f.u)
    by tools/golden_fullsize.py, since the oracle needs ~40 min for C5;
  * G(u) phi on C3, C4, C5: two full products against the oracle's EbE G(u) phi.
"""

import functools
import json
import os

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
    """Every right-hand side: the true residual of the GPU solution under the oracle's own
    element-by-element operator (a property that holds at any size)."""
    cfg, inp, rep, X = solved(name)
    assert rep["status"] == "MG_OK", rep
    assert max(rep["true_relres"]) <= cfg.tol
    for k in range(cfg.nrhs):
        res = inp["rhs"][k] - ebe.matvec(cfg.nel, inp["E"], inp["fixed"], X[k])
        assert np.linalg.norm(res) / np.linalg.norm(inp["rhs"][k]) <= 2 * cfg.tol, k


@functools.lru_cache(maxsize=None)
def oracle_solution(name):
    """All R right-hand sides by the independent iterative oracle (scipy MG-PCG to 1e-13), the
    systems solved in parallel worker processes (one per RHS, forked before any numpy threading)."""
    cfg, inp = inputs(name)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    return _solve_parallel(cfg, K, inp)


def _solve_one(args):
    k = args
    cfg, K, inp = _POOL_STATE
    U, _ = solve.mgpcg_solve(cfg.nel, K, inp["rhs"][k], inp["fixed"], cfg.levels, tol=1e-13)
    return U


_POOL_STATE = None


def _solve_parallel(cfg, K, inp):
    import multiprocessing as mp
    import os
    global _POOL_STATE
    _POOL_STATE = (cfg, K, inp)
    nproc = max(1, min(cfg.nrhs, len(os.sched_getaffinity(0)), 8))
    with mp.get_context("fork").Pool(nproc) as pool:
        U = pool.map(_solve_one, range(cfg.nrhs))
    _POOL_STATE = None
    return np.stack(U)


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_fullsize_solution_vs_iterative_oracle(name):
    """Every right-hand side (state + all adjoint fields) against the oracle's own solution,
    1e-8 relative L2 (BASELINE.json:5)."""
    cfg, inp, rep, X = solved(name)
    U = oracle_solution(name)
    for k in range(cfg.nrhs):
        assert np.linalg.norm(X[k] - U[k]) / np.linalg.norm(U[k]) < 1e-8, k


def _golden(name):
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"fullsize_{name}_solution.json")
    return json.load(open(path))


def test_fullsize_C5_solution_vs_oracle_golden():
    """C5 (12.8M DOFs, 7 RHS) against the oracle's iterative solution (tol 1e-13) stored by
    tools/golden_fullsize.py (calls only oracle/): per RHS the 2-norm and f.u of the whole
    solution, and the solution itself at ~4.8k sampled DOFs (random nodes + faces, planes, tile
    boundaries), all at 1e-8 relative."""
    import hashlib
    cfg, inp, rep, X = solved("C5")
    g = _golden("C5")
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()
    assert g["inputs_sha256"] == dict(E=sha(inp["E"]), fixed=sha(inp["fixed"])), \
        "regenerated C5 moduli / masks differ from the ones the golden file was computed from"
    idx = np.array(g["dofs"], dtype=np.int64)
    # right-hand sides: FFT-filtered, equal to rounding across host CPUs (not bitwise)
    for k in range(cfg.nrhs):
        nb = np.linalg.norm(inp["rhs"][k])
        assert abs(nb - g["rhs_norm2"][k]) <= 1e-13 * nb
        assert np.abs(inp["rhs"][k][idx] - np.array(g["rhs_values"][k])).max() <= 1e-13 * np.abs(inp["rhs"][k]).max()
    assert len(g["rhs"]) == cfg.nrhs
    for e in g["rhs"]:
        k = e["k"]
        assert e["relres"] <= 1e-11   # the stored oracle solution itself (fp64 floor of a true residual)
        ref = np.array(e["values"])
        got = X[k][idx]
        assert np.linalg.norm(got - ref) / np.linalg.norm(ref) < 1e-8, k
        assert abs(np.linalg.norm(X[k]) - e["norm2"]) <= 1e-8 * e["norm2"], k
        assert abs(inp["rhs"][k] @ X[k] - e["work"]) <= 1e-8 * abs(e["work"]), k


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
def test_fullsize_stress_stiffness(name):
    """G(u) phi for all phi of the config with u the GPU state solution (reading r16); two of the
    products checked in full against the oracle's EbE G(u) phi (max-abs relative: smooth inputs,
    SURVEY r17)."""
    import paper_1909_13585_b200 as mg
    cfg, inp, rep, X = solved(name)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    phi = inp["phi"]
    y = torch.empty((phi.shape[0], phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.stress_stiffness_apply(h, to_dev(inp["Es"]), to_dev(X[0]), to_dev(phi), y)
    y = y.cpu().numpy()
    ks = (0, phi.shape[0] - 1)
    ref = ebe.stress_stiffness_apply(cfg.nel, inp["Es"], inp["fixed"], X[0], phi[list(ks)])
    for i, k in enumerate(ks):
        assert np.abs(y[k] - ref[i]).max() <= 1e-12 * np.abs(ref[i]).max(), k
