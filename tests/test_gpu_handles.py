"""Handle-lifetime regressions, all through the C ABI on the GPU:

* one handle reused for block solves and batched solves of changing width (the cached block-PCG
  graph must be re-captured whenever the width or the vectors change);
* several live handles with different element constants (2D / 3D, standard / incompatible-mode
  element, another nu) used interleaved: each keeps its own K0 (the constants are switched per
  call, not per setup);
* mg_update_modulus with an invalid E leaves the handle unchanged (argument errors have no side
  effects, include/mgcg.h).
Parity bars as in test_gpu_parity.py: solutions vs the direct oracle at 1e-8, matvec at 1e-13.
"""

import functools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import assemble, ebe, solve  # noqa: E402
from workloads import generate, get_config, rough_vectors  # noqa: E402

pytestmark = pytest.mark.gpu
DEV = "cuda:0"


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(DEV)


@functools.lru_cache(maxsize=None)
def case(name, nu=0.3, element="std"):
    cfg = get_config(name, nu=nu)
    inp = generate(cfg)
    K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"], nu, element)
    return cfg, inp, K


def rel(a, b):
    return np.linalg.norm(a - b, axis=-1) / np.linalg.norm(b, axis=-1)


def test_block_graph_recaptured_on_width_change():
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2c")
    rng = np.random.default_rng(5)
    F = rng.standard_normal((16, K.shape[0])) * (1 - inp["fixed"])
    U = solve.direct_solve(K, F, inp["fixed"])
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    for kind, k in (("block", 8), ("block", 4), ("pcg", 16), ("block", 4), ("block", 6), ("pcg", 2), ("block", 6)):
        x = torch.zeros((k, K.shape[0]), dtype=torch.float64, device=DEV)
        fn = mg.mgcg_block_solve if kind == "block" else mg.mgcg_solve
        rep = fn(h, to_dev(F[:k]), 1e-10, x)
        assert max(rep["true_relres"]) <= 1e-10, (kind, k, rep)
        assert rel(x.cpu().numpy(), U[:k]).max() < 1e-8, (kind, k)


def _matvec_err(h, cfg, inp, nu, element):
    import paper_1909_13585_b200 as mg
    X = rough_vectors(cfg, 2, seed_offset=31)
    Y = torch.empty((2, X.shape[1]), dtype=torch.float64, device=DEV)
    mg.mg_matvec(h, 0, to_dev(X), Y)
    ref = ebe.matvec(cfg.nel, inp["E"], inp["fixed"], X, nu=nu, element=element)
    return rel(Y.cpu().numpy(), ref).max()


def test_interleaved_handles_keep_their_constants():
    import paper_1909_13585_b200 as mg
    specs = [("T2b", 0.3, "std"), ("T3a", 0.3, "std"), ("T2b", 0.3, "wilson"), ("T3b", 0.25, "std"),
             ("T3a", 0.3, "wilson")]
    hs = []
    for name, nu, el in specs:
        cfg, inp, K = case(name, nu, el)
        hs.append(mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels, nu=nu, element=el))
    for rnd in range(2):   # every handle after all of them were set up, twice, in two orders
        order = range(len(specs)) if rnd == 0 else reversed(range(len(specs)))
        for i in order:
            name, nu, el = specs[i]
            cfg, inp, K = case(name, nu, el)
            assert _matvec_err(hs[i], cfg, inp, nu, el) < 1e-13, specs[i]
            U = solve.direct_solve(K, inp["rhs"], inp["fixed"])
            x = torch.empty((cfg.nrhs, K.shape[0]), dtype=torch.float64, device=DEV)
            mg.mgcg_solve(hs[i], to_dev(inp["rhs"]), cfg.tol, x)
            assert rel(x.cpu().numpy(), U).max() < 1e-8, specs[i]
            if cfg.nphi:
                phi = inp["rhs"][1:1 + min(cfg.nphi, cfg.nrhs - 1)]
                y = torch.empty(phi.shape, dtype=torch.float64, device=DEV)
                mg.stress_stiffness_apply(hs[i], to_dev(inp["Es"]), to_dev(U[0]), to_dev(phi), y)
                ref = ebe.stress_stiffness_apply(cfg.nel, inp["Es"], inp["fixed"], U[0], phi, nu=nu)
                assert np.abs(y.cpu().numpy() - ref).max() <= 1e-12 * np.abs(ref).max(), specs[i]


@pytest.mark.parametrize("bad", [0.0, -1.0, float("nan"), float("inf")])
@pytest.mark.parametrize("host", [False, True])
def test_invalid_update_modulus_leaves_handle_unchanged(bad, host):
    import paper_1909_13585_b200 as mg
    cfg, inp, K = case("T2b")
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    x0 = torch.empty((cfg.nrhs, K.shape[0]), dtype=torch.float64, device=DEV)
    mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x0)
    E2 = inp["E"].copy() * 0.5
    E2[7] = bad
    with pytest.raises(mg.MgError) as ei:
        mg.mg_update_modulus(h, E2 if host else to_dev(E2))
    assert "MG_ERR_MODULUS" in str(ei.value) or "modulus" in str(ei.value).lower()
    x1 = torch.empty_like(x0)
    mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x1)
    assert torch.equal(x0, x1)   # same operators, same graphs: bitwise


@pytest.mark.parametrize("name", ["T2b", "T3c", "T3h"])
def test_update_modulus_then_host_solve(name):
    """mg_update_modulus returns with the new operators only enqueued; a host-buffer mgcg_solve
    uploads its right-hand sides while they are built and then waits for them.  The result equals
    the device-buffer path bit for bit and the direct oracle solve for the new E."""
    import paper_1909_13585_b200 as mg
    cfg, inp, _ = case(name)
    h = mg.mg_setup(cfg.nel, to_dev(inp["E"]), to_dev(inp["fixed"]), cfg.levels)
    E2 = np.ascontiguousarray(inp["E"] * np.linspace(0.5, 2.0, inp["E"].size))
    rhs_h = torch.from_numpy(np.ascontiguousarray(inp["rhs"])).pin_memory()
    x_h = torch.empty(rhs_h.shape, dtype=torch.float64).pin_memory()
    x_d = torch.empty(rhs_h.shape, dtype=torch.float64, device=DEV)
    for _ in range(2):   # the second round reuses the upload buffer and the graphs
        mg.mg_update_modulus(h, torch.from_numpy(E2).pin_memory().numpy())
        mg.mgcg_solve(h, rhs_h.numpy(), cfg.tol, x_h.numpy())
        mg.mg_update_modulus(h, to_dev(E2))
        mg.mgcg_solve(h, to_dev(inp["rhs"]), cfg.tol, x_d)
        assert torch.equal(x_h, x_d.cpu())
    K2 = assemble.assemble_K(cfg.nel, E2, inp["fixed"])
    U = solve.direct_solve(K2, inp["rhs"], inp["fixed"])
    assert rel(x_h.numpy(), U).max() < 1e-8
