"""Stacked-row tail tile of the 3D fine kernels (h8t.cu TAIL): when the last column tile owns <= 9
node columns, its CTA marches three 7-row groups of 10 lanes instead of one group of 32 lanes.  The
per-element arithmetic and the row exchange are those of an ordinary tile, so the operator
(matvec, V-cycle) is bitwise the same with the tail launch on (MG_H8T_TAIL=1, default) and off; the
CG dot partials are grouped by a different tiling, so a solve agrees to rounding.  The switch is
read once per process: each setting runs in its own interpreter."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, %(root)r)
import paper_1909_13585_b200 as mg
from workloads import generate, get_config
out = {}
for name in %(names)r:
    cfg = get_config(name)
    inp = generate(cfg)
    dev = torch.device("cuda:0")
    h = mg.mg_setup(cfg.nel, torch.from_numpy(inp["E"]).to(dev), torch.from_numpy(inp["fixed"]).to(dev), cfg.levels)
    rhs = torch.from_numpy(np.ascontiguousarray(inp["rhs"])).to(dev)
    g = torch.Generator().manual_seed(7)
    xr = torch.randn(rhs.shape, generator=g, dtype=torch.float64).to(dev)   # rough input
    y = torch.empty_like(rhs)
    mg.mg_matvec(h, 0, xr, y)
    z = torch.empty_like(rhs)
    mg.mg_vcycle(h, xr, z)
    x = torch.empty_like(rhs)
    rep = mg.mgcg_solve(h, rhs, 1e-10, x)
    out[name] = {"y": y.cpu().numpy().tobytes().hex(), "z": z.cpu().numpy().tobytes().hex(),
                 "x": x.cpu().numpy().ravel().tolist(), "iters": list(rep["iters"])}
print(json.dumps(out))
"""


def _run(names, **env):
    e = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "names": names}], env=e,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


def test_tail_geometry():
    """T3f (n2 = 65 = 60 + 5), T3h (n2 = 37 = 30 + 7) and C5 (n2 = 129 = 120 + 9) take the tail
    launch; C4 (n2 = 49 = 30 + 19) and T3g (n2 = 71 = 60 + 11) do not (more than 9 owned columns)."""
    from workloads import get_config

    def tail(name):
        n2 = get_config(name).nel[2] + 1
        ntc = (n2 + 29) // 30
        return ntc >= 2 and n2 - 1 - (30 * (ntc - 1) - 1) <= 9

    assert [tail(n) for n in ("T3f", "T3h", "C5")] == [True, True, True]
    assert [tail(n) for n in ("C4", "T3g", "T3a", "T3c")] == [False] * 4


@pytest.mark.gpu
def test_tail_on_off():
    names = ["T3f", "T3h"]
    on, off = _run(names, MG_H8T_TAIL="1"), _run(names, MG_H8T_TAIL="0")
    for n in names:
        assert on[n]["y"] == off[n]["y"], f"{n}: matvec differs"
        assert on[n]["z"] == off[n]["z"], f"{n}: V-cycle differs"
        xa, xb = np.array(on[n]["x"]), np.array(off[n]["x"])
        assert np.abs(xa - xb).max() <= 1e-9 * np.abs(xb).max(), n
        assert all(abs(a - b) <= 1 for a, b in zip(on[n]["iters"], off[n]["iters"])), n
