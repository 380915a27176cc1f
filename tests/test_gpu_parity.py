"""Parity of the CUDA path (through the C ABI) with the CPU oracle, on seeded inputs.

Bars (BASELINE.json:5): matvec and G(u) phi within 1e-13 relative (measured on rough
iid N(0,1) inputs); solutions within 1e-8 relative L2 with both sides
solved to 1e-10 or better.  Sizes span several warp tiles / chunks and ragged tails.
"""

import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, ebe, mg as omg, solve  # noqa: E402
from workloads import generate, get_config, rough_vectors  # noqa: E402

pytestmark = pytest.mark.gpu

DEV = "cuda:0"


@functools.lru_cache(maxsize=None)
def case(name):
    cfg = get_config(name)
    inp = generate(cfg)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
    return cfg, inp, K


@functools.lru_cache(maxsize=None)
def direct(name):
    cfg, inp, K = case(name)
    return solve.direct_solve(K, inp["rhs"], inp["fixed"])


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


def handle(name, **kw):
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    return mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels, **kw)


def rel(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


MATVEC_CASES = ["T2a", "T2b", "T2c", "C1", "C2", "T3a", "T3b", "T3c", "T3d", "T3f", "T3g", "T3h"]


@pytest.mark.parametrize("name", MATVEC_CASES)
def test_matvec_parity_rough(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    h = handle(name)
    X = rough_vectors(cfg, 3)                      # unmasked: exercises the identity rows
    y = torch.empty((3, X.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_matvec(h, 0, to_dev(X), y)
    yo = (K @ X.T).T
    assert rel(y.cpu().numpy(), yo).max() < 1e-13


@pytest.mark.parametrize("name", ["T2a", "T2b", "C1", "C2", "T3a", "T3c"])
def test_stress_stiffness_parity(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    h = handle(name)
    u = rough_vectors(cfg, 1, seed_offset=5)[0]
    phi = rough_vectors(cfg, 2, seed_offset=9)
    y = torch.empty((2, phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.stress_stiffness_apply(h, to_dev(inp["Es"]), to_dev(u), to_dev(phi), y)
    G = assemble.assemble_G(cfg.nel, inp["Es"], u, inp["fixed"])
    yo = (G @ phi.T).T
    assert rel(y.cpu().numpy(), yo).max() < 1e-13


@pytest.mark.parametrize("nphi", [1, 3, 7])
@pytest.mark.parametrize("name", ["T2b", "T3a"])
def test_stress_stiffness_host_buffers_bitwise(name, nphi):
    """G(u) phi with host buffers (pageable, and pinned: the chunked copy-in / compute / copy-out
    pipeline) equals the device-buffer result bit for bit."""
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    h = handle(name)
    u = rough_vectors(cfg, 1, seed_offset=5)[0]
    phi = rough_vectors(cfg, nphi, seed_offset=19)
    yd = torch.empty((nphi, phi.shape[1]), dtype=torch.float64, device=DEV)
    mg.stress_stiffness_apply(h, to_dev(inp["Es"]), to_dev(u), to_dev(phi), yd)
    ref = yd.cpu().numpy()
    yh = np.empty_like(phi)
    mg.stress_stiffness_apply(h, np.ascontiguousarray(inp["Es"]), np.ascontiguousarray(u), np.ascontiguousarray(phi), yh)
    assert np.array_equal(yh, ref)
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
    pEs, pu, pphi = pin(inp["Es"]), pin(u), pin(phi)
    py = torch.empty(phi.shape, dtype=torch.float64).pin_memory()
    mg.stress_stiffness_apply(h, pEs, pu, pphi, py)
    assert np.array_equal(py.numpy(), ref)


SOLVE_CASES = ["T2a", "T2b", "T2c", "C1", "C2", "T3a", "T3b", "T3c", "T3f", "T3g", "T3h"]


@pytest.mark.parametrize("name", SOLVE_CASES)
def test_solve_parity_direct(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    U = direct(name)
    h = handle(name)
    x = torch.empty((cfg.nrhs, U.shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x, raise_on_error=False)
    assert rep["status"] == "MG_OK", rep
    xs = x.cpu().numpy()
    assert rel(xs, U).max() < 1e-8, rep
    assert max(rep["true_relres"]) <= cfg.tol
    assert all(rep["converged"])
    # independent check of the residual with the oracle's own operator
    res = inp["rhs"] - (K @ xs.T).T
    assert (np.linalg.norm(res, axis=1) / np.linalg.norm(inp["rhs"], axis=1)).max() <= 2 * cfg.tol


@pytest.mark.parametrize("name", ["T2b", "T2c", "T3a", "T3c"])
def test_transfers_match_oracle_P(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    h = handle(name)
    rng = np.random.default_rng(1)
    for l in range(cfg.levels - 1):
        nf, nc = H.P[l].shape
        vf = rng.standard_normal((2, nf))
        vc = rng.standard_normal((2, nc))
        c = torch.empty((2, nc), dtype=torch.float64, device=DEV)
        f = torch.empty((2, nf), dtype=torch.float64, device=DEV)
        mg.mg_restrict(h, l, to_dev(vf), c)
        mg.mg_prolong(h, l, to_dev(vc), f)
        assert np.abs(c.cpu().numpy() - (H.P[l].T @ vf.T).T).max() < 1e-14 * np.abs(vf).max() * 8
        assert np.abs(f.cpu().numpy() - (H.P[l] @ vc.T).T).max() < 1e-14 * np.abs(vc).max() * 8


@pytest.mark.parametrize("name", ["T2c", "T3b", "T3d"])
def test_galerkin_levels_match_triple_product(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    h = handle(name)
    rng = np.random.default_rng(2)
    for l in range(1, cfg.levels):
        n = H.A[l].shape[0]
        X = rng.standard_normal((2, n))
        y = torch.empty((2, n), dtype=torch.float64, device=DEV)
        mg.mg_matvec(h, l, to_dev(X), y)
        assert rel(y.cpu().numpy(), (H.A[l] @ X.T).T).max() < 1e-13
        d = torch.empty(n, dtype=torch.float64, device=DEV)
        mg.mg_get_diagonal(h, l, d)
        assert np.abs(d.cpu().numpy() - H.A[l].diagonal()).max() < 1e-13 * np.abs(H.A[l].diagonal()).max()
    d = torch.empty(K.shape[0], dtype=torch.float64, device=DEV)
    mg.mg_get_diagonal(h, 0, d)
    assert np.abs(d.cpu().numpy() - K.diagonal()).max() < 1e-14 * np.abs(K.diagonal()).max()
    nL = H.A[-1].shape[0]
    Ai = torch.empty((nL, nL), dtype=torch.float64, device=DEV)
    mg.mg_get_coarse_inverse(h, Ai)
    ref = np.linalg.inv(H.A[-1].toarray())
    assert np.abs(Ai.cpu().numpy() - ref).max() < 1e-9 * np.abs(ref).max()


def test_coarse_inverse_large_level():
    """Coarsest level as large as C5's (4131 DOFs, padded 4160): the Gauss-Jordan path that folds
    the next diagonal block into the DMMA update kernel, against numpy's inverse."""
    import paper_1909_13585_b200 as mg
    name = "T3e"
    cfg, inp, K = case(name)
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    h = handle(name)
    nL = H.A[-1].shape[0]
    assert nL >= 3072
    Ai = torch.empty((nL, nL), dtype=torch.float64, device=DEV)
    mg.mg_get_coarse_inverse(h, Ai)
    ref = np.linalg.inv(H.A[-1].toarray())
    assert np.abs(Ai.cpu().numpy() - ref).max() < 1e-9 * np.abs(ref).max()


def test_vcycle_many_rhs_matches_oracle():
    """40 right-hand sides (> 32: the dense coarsest apply runs in two RHS chunks)."""
    import paper_1909_13585_b200 as mg
    name = "T3a"
    cfg, inp, K = case(name)
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    V = solve._VCycle(H, 0.6, 1)
    h = handle(name)
    A = rough_vectors(cfg, 40, seed_offset=41, masked=True)
    Z = torch.empty((40, A.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_vcycle(h, to_dev(A), Z)
    Zo = np.stack([V.apply(a) for a in A])
    assert rel(Z.cpu().numpy(), Zo).max() < 1e-9


@pytest.mark.parametrize("name", ["T2b", "T3a"])
def test_vcycle_symmetric_positive(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    h = handle(name)
    A = rough_vectors(cfg, 4, seed_offset=21, masked=True)
    Z = torch.empty((4, A.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_vcycle(h, to_dev(A), Z)
    Zs = Z.cpu().numpy()
    G = A @ Zs.T
    assert np.abs(G - G.T).max() < 1e-12 * np.abs(G).max()
    assert np.all(np.linalg.eigvalsh(0.5 * (G + G.T)) > 0)


@pytest.mark.parametrize("name", ["T2b", "T2c", "C2", "T3a", "T3b"])
def test_vcycle_matches_oracle_vcycle(name):
    """One V(1,1) cycle (damped Jacobi omega = 0.6, Galerkin coarse operators, direct
    coarsest solve) equals the oracle's scipy V-cycle of the same definition."""
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    V = solve._VCycle(H, 0.6, 1)
    h = handle(name)
    A = rough_vectors(cfg, 2, seed_offset=31, masked=True)
    Z = torch.empty((2, A.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_vcycle(h, to_dev(A), Z)
    Zo = np.stack([V.apply(a) for a in A])
    # fp64 rounding of two summation orders, amplified by the coarse solves (cond ~1e5)
    assert rel(Z.cpu().numpy(), Zo).max() < 1e-9


def test_single_rhs_equals_batched_column_bitwise():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2b")
    h = handle("T2b")
    rhs = to_dev(inp["rhs"])
    xb = torch.empty_like(rhs)
    mg.mgcg_solve(h, rhs, 1e-10, xb)
    for k in (0, 3):
        x1 = torch.empty((1, rhs.shape[1]), dtype=torch.float64, device=DEV)
        mg.mgcg_solve(h, rhs[k:k + 1].contiguous(), 1e-10, x1)
        assert torch.equal(x1[0], xb[k])
    xb2 = torch.empty_like(rhs)
    mg.mgcg_solve(h, rhs, 1e-10, xb2)
    assert torch.equal(xb, xb2)            # run-to-run determinism


def test_zero_and_duplicate_rhs():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2a")
    h = handle("T2a")
    rhs = np.stack([np.zeros_like(inp["rhs"][0]), inp["rhs"][1], inp["rhs"][1]])
    x = torch.empty((3, rhs.shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(rhs), 1e-10, x)
    assert rep["iters"][0] == 0 and torch.count_nonzero(x[0]) == 0
    assert torch.equal(x[1], x[2])


@pytest.mark.parametrize("name", ["T3a", "T2b"])
def test_host_buffers_match_device(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    h = handle(name)
    xd = torch.empty((cfg.nrhs, K.shape[0]), dtype=torch.float64, device=DEV)
    mg.mgcg_solve(h, to_dev(inp["rhs"]), 1e-10, xd)
    xh = np.empty((cfg.nrhs, K.shape[0]))
    mg.mgcg_solve(h, np.ascontiguousarray(inp["rhs"]), 1e-10, xh)
    assert np.array_equal(xh, xd.cpu().numpy())


def test_error_statuses():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2a")
    with pytest.raises(mg.MgError) as e:
        mg.mg_setup((30, 16), to_dev(np.ones(480)), to_dev(np.zeros(2 * 31 * 17, np.uint8)), 3)
    assert e.value.name == "MG_ERR_NONDIVISIBLE"
    bad = inp["E"].copy()
    bad[7] = -1.0
    with pytest.raises(mg.MgError) as e:
        mg.mg_setup(cfg.nel, to_dev(bad), to_dev(inp["fixed"]), cfg.levels)
    assert e.value.name == "MG_ERR_MODULUS"
    h = handle("T2a", max_iter=2)
    x = torch.empty((cfg.nrhs, K.shape[0]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(inp["rhs"]), 1e-10, x, raise_on_error=False)
    assert rep["status"] == "MG_ERR_MAXITER" and max(rep["iters"]) == 2


def test_update_modulus_equals_fresh_setup():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2b")
    cfg3, inp3, _ = case("T2b")
    h = handle("T2b")
    E2 = inp["E"][::-1].copy()
    mg.mg_update_modulus(h, to_dev(E2))
    h2 = mg.mg_setup(cfg.nel, to_dev(E2), to_dev(inp["fixed"]), cfg.levels)
    rhs = to_dev(inp["rhs"])
    x1 = torch.empty_like(rhs)
    x2 = torch.empty_like(rhs)
    mg.mgcg_solve(h, rhs, 1e-10, x1)
    mg.mgcg_solve(h2, rhs, 1e-10, x2)
    assert torch.equal(x1, x2)


@pytest.mark.parametrize("name", ["T2c", "T3a"])
def test_profile_kernels_leaves_solver_state_valid(name):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case(name)
    h = handle(name)
    rhs = to_dev(inp["rhs"])
    x1 = torch.empty_like(rhs)
    mg.mgcg_solve(h, rhs, 1e-10, x1)
    ms = mg.mg_profile_kernels(h, cfg.nrhs, reps=2)
    assert all(v > 0 for v in ms.values())
    x2 = torch.empty_like(rhs)
    mg.mgcg_solve(h, rhs, 1e-10, x2)
    assert torch.equal(x1, x2)


@pytest.mark.parametrize("fused", ["0", "1", "2", "3"])
@pytest.mark.parametrize("name", ["T3b", "T3c"])
def test_fused3d_variant_parity(name, fused, monkeypatch):
    """Every MG_FUSED3D setting of the 3D fine V-cycle halves (bit 0: r update + pre-smoother +
    residual in one h8 kernel, the default; bit 1: prolongation + post-smoother) solves to the
    direct solution and applies the oracle's V-cycle."""
    import paper_1909_13585_b200 as mg
    monkeypatch.setenv("MG_FUSED3D", fused)
    cfg, inp, K = case(name)
    U = direct(name)
    h = handle(name)
    x = torch.empty((cfg.nrhs, U.shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x)
    assert rel(x.cpu().numpy(), U).max() < 1e-8, rep
    H = omg.Hierarchy(cfg.nel, K, inp["fixed"], cfg.levels)
    V = solve._VCycle(H, 0.6, 1)
    A = rough_vectors(cfg, 2, seed_offset=31, masked=True)
    Z = torch.empty((2, A.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_vcycle(h, to_dev(A), Z)
    Zo = np.stack([V.apply(a) for a in A])
    assert rel(Z.cpu().numpy(), Zo).max() < 1e-9


@pytest.mark.parametrize("variants", ["9,9,9,9,9", "3,3,3,3,3", "4,4,4,4,4", "5,5,5,5,5", "0,1,2,0,1"])
def test_h8_kernel_variants_matvec_and_solve(variants, monkeypatch):
    """All H8 fine-kernel variants (register prefetch 8/16 rows, 2 CTAs/SM, shared-memory plane
    ring with and without slot retention) give the same operator and solution."""
    import paper_1909_13585_b200 as mg
    monkeypatch.setenv("MG_H8_VARIANTS", variants)
    name = "T3c"
    cfg, inp, K = case(name)
    U = direct(name)
    h = handle(name)
    X = rough_vectors(cfg, 3)
    Y = torch.empty((3, X.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_matvec(h, 0, to_dev(X), Y)
    assert rel(Y.cpu().numpy(), (K @ X.T).T).max() < 1e-13
    x = torch.empty((cfg.nrhs, U.shape[1]), dtype=torch.float64, device=DEV)
    rep = mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x)
    assert rel(x.cpu().numpy(), U).max() < 1e-8, rep
