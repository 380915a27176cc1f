"""Programmatic dependent launch (PDL) must not change results: the same solves and V-cycles with
MG_PDL=1 (default) and MG_PDL=0 (plain launches) agree bit for bit.  The switch is read once per
process, so each setting runs in its own interpreter."""
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
    x = torch.empty_like(rhs)
    for _ in range(3):   # repeated solves: the graphs are replayed
        mg.mgcg_solve(h, rhs, 1e-10, x)
    out[name] = x.cpu().numpy().tobytes().hex()
print(json.dumps(out))
"""


def _run(names, **env):
    e = dict(os.environ, **env)
    p = subprocess.run([sys.executable, "-c", SCRIPT % {"root": ROOT, "names": names}], env=e,
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert p.returncode == 0, p.stderr[-2000:]
    return json.loads(p.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
def test_pdl_on_off_bitwise():
    """Default (PDL on the 2D iteration and the scalar / dense kernels) vs plain launches, up to
    BASELINE's C3 / C4 sizes."""
    names = ["T2b", "C1", "C2", "C3", "T3a", "C4"]
    on, off = _run(names, MG_PDL="1"), _run(names, MG_PDL="0")
    for n in names:
        assert on[n] == off[n], n


@pytest.mark.gpu
def test_gauss_jordan_pdl_bitwise():
    """The coarsest Gauss-Jordan sequence with programmatic dependent launch (MG_GJ_PDL=1; every
    kernel of it waits on griddepcontrol before touching memory) gives the same inverse, hence
    bitwise the same solves, as plain launches -- small levels (C1, T2b) and the folded
    large-level path (T3e, n >= 3072)."""
    names = ["T2b", "C1", "C2", "T3e"]
    on, off = _run(names, MG_GJ_PDL="1"), _run(names, MG_GJ_PDL="0")
    for n in names:
        assert on[n] == off[n], n


@pytest.mark.gpu
def test_z2_in_post_bitwise():
    """3D fused V-cycle: the prolongation writing only P e with the first post-smoothing sweep forming
    z2 = P e + omega D^-1 r (MG_Z2_IN_POST=1, default) gives bit for bit the solves of the
    prolongation forming z2 itself (=0): the same products, rounded the same way."""
    names = ["T3a", "T3c", "T3f", "C4"]
    on, off = _run(names, MG_Z2_IN_POST="1"), _run(names, MG_Z2_IN_POST="0")
    for n in names:
        assert on[n] == off[n], n


@pytest.mark.gpu
def test_galerkin_warp_bitwise():
    """3D level-1 Galerkin: the warp-per-element kernel for elements with free fine nodes plus the
    general kernel on the listed rest (MG_GAL_WARP=1, default) builds bit for bit the coarse
    operators of the general kernel alone (=0), hence the same solves (slab grids included)."""
    names = ["T3a", "T3d", "T3f", "C4"]
    on, off = _run(names, MG_GAL_WARP="1"), _run(names, MG_GAL_WARP="0")
    for n in names:
        assert on[n] == off[n], n


@pytest.mark.gpu
def test_coarse_xsplit_bitwise():
    """Large 3D coarse levels (C5 level 1): the stencil kernel with the 7 RHS in two groups of
    consecutive CTAs (MG_COARSE_XSPLIT=2, default) accumulates every RHS in the same order as with
    all RHS in one thread (=0): bit for bit the same solves."""
    names = ["C5"]
    on, off = _run(names, MG_COARSE_XSPLIT="2"), _run(names, MG_COARSE_XSPLIT="0")
    for n in names:
        assert on[n] == off[n], n
