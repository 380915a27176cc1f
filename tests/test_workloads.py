"""Input recipe checks (CPU): BASELINE.json configs and SURVEY 8(c) r3-r9."""

import numpy as np
import pytest

from workloads import CONFIGS, generate, get_config, n_dofs, n_nodes
from workloads.generate import cone_filter, heaviside_projection, state_load


def test_config_sizes():
    # 64x32 Q4 has 2,145 nodes and 4,290 DOFs (BASELINE.json:7 miscounts)
    assert n_nodes((64, 32)) == 2145 and n_dofs((64, 32)) == 4290
    assert n_dofs(CONFIGS["C2"].nel) == 231842
    assert n_dofs(CONFIGS["C3"].nel) == 3692162
    assert n_dofs(CONFIGS["C4"].nel) == 698691
    assert n_dofs(CONFIGS["C5"].nel) == 12830211


def test_projection_and_filter():
    x = np.linspace(0, 1, 11)
    p = heaviside_projection(x, 2.0, 0.5)
    assert abs(p[0]) < 1e-15 and abs(p[-1] - 1) < 1e-15 and abs(p[5] - 0.5) < 1e-15
    assert np.all(np.diff(p) > 0)
    for shape in [(9, 7), (5, 4, 6)]:
        u = np.full(shape, 0.37)
        assert np.allclose(cone_filter(u, 2.0), 0.37, atol=1e-15)
        assert np.allclose(cone_filter(u, 4.0, use_fft=True), 0.37, atol=1e-12)
    # single solid element, r = 2: interior weights max(0, 2 - dist), normalised
    z = np.zeros((7, 7)); z[3, 3] = 1
    f = cone_filter(z, 2.0)
    w = np.array([[2 - np.sqrt(2), 1, 2 - np.sqrt(2)], [1, 2, 1], [2 - np.sqrt(2), 1, 2 - np.sqrt(2)]])
    assert abs(f[3, 3] - 2 / w.sum()) < 1e-15


@pytest.mark.parametrize("name", ["C1", "T2b", "T3a", "T3b"])
def test_generated_inputs(name):
    cfg = get_config(name)
    a = generate(cfg)
    b = generate(cfg)
    for k in ("E", "Es", "rhs", "fixed"):
        assert np.array_equal(a[k], b[k])
    n = n_dofs(cfg.nel)
    assert a["rhs"].shape == (cfg.nrhs, n)
    assert np.all(a["E"] >= cfg.Emin) and np.all(a["E"] <= cfg.E0)
    assert np.allclose(a["Es"], a["rho"] ** 3)
    fixed = a["fixed"].astype(bool)
    assert np.all(a["rhs"][:, fixed] == 0)
    assert abs(a["rhs"][0].sum() + 1.0) < 1e-14            # unit total load, negative direction
    for k in range(1, cfg.nrhs):
        assert abs(np.linalg.norm(a["rhs"][k]) - 1) < 1e-14
    if cfg.nphi:
        assert a["phi"].shape == (cfg.nphi, n)


def test_state_load_placement():
    cfg = get_config("C4")
    f = state_load(cfg).reshape(97, 49, 49, 3)
    assert np.count_nonzero(f) == 49 and np.all(f[96, 0, :, 1] < 0)
    cfg = get_config("T3a")
    f = state_load(cfg).reshape(17, 9, 9, 3)
    assert np.count_nonzero(f[16, ..., 0]) == 81 and abs(f[16, 4, 4, 0] + 1 / 64) < 1e-16
