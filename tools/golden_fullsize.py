"""Write tests/golden/fullsize_<cfg>_solution.json: the oracle's solution of a full-size config,
sampled (TEST INFRASTRUCTURE; calls only oracle/ and workloads/).

The oracle cannot solve C5 (12.8M DOFs, 7 RHS) inside the GPU test budget (about 40 min single
core here), so this committed script solves it once with the independent iterative oracle
(assembled K, scipy Galerkin MG-PCG to relative residual 1e-13; SURVEY 8(c) "C4, C5") and stores,
per right-hand side: the solution at sampled DOFs, its 2-norm, the work f.u, the iteration count
and the oracle's own relative residual; plus sha256 hashes of the generated inputs so a test can
tell a regenerated-input mismatch apart from a solver mismatch.

  python tools/golden_fullsize.py C5                 (oracle solve, ~25 min)
  python tools/golden_fullsize.py C5 --inputs-only   (refresh the input fingerprint only)
"""

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import assemble, solve  # noqa: E402
from workloads import generate, get_config  # noqa: E402


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def sample_dofs(cfg, count, seed):
    """Random DOFs plus every component of structural edge-case nodes (faces, first / last
    planes, kernel tile boundaries along each axis)."""
    nn = [n + 1 for n in cfg.nel]
    rng = np.random.default_rng(seed)
    pts = [tuple(int(rng.integers(0, m)) for m in nn) for _ in range(count)]
    for k, m in enumerate(nn):
        for v in (0, 1, 2, 5, 6, 7, 29, 30, 31, 32, 33, 63, 64, 65, m // 2, m - 2, m - 1):
            if 0 <= v < m:
                p = [int(rng.integers(0, mm)) for mm in nn]
                p[k] = v
                pts.append(tuple(p))
    pts += [tuple(0 for _ in nn), tuple(m - 1 for m in nn)]
    nodes = sorted(set(int(np.ravel_multi_index(p, nn)) for p in pts))
    return np.array([cfg.dim * p + c for p in nodes for c in range(cfg.dim)], dtype=np.int64)


def input_fingerprint(cfg, inp, idx):
    """E and the masks hash exactly; the adjoint right-hand sides come from FFT filtering, whose last
    bits depend on the host CPU, so they are fingerprinted by their norms and sampled values."""
    return dict(inputs_sha256=dict(E=sha(inp["E"]), fixed=sha(inp["fixed"])),
                rhs_norm2=[float(np.linalg.norm(b)) for b in inp["rhs"]],
                rhs_values=[[float(v) for v in b[idx]] for b in inp["rhs"]])


def refresh_inputs(name):
    """Rewrite only the input fingerprint of an existing golden file (no oracle call)."""
    cfg = get_config(name)
    inp = generate(cfg, with_phi=False)
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}_solution.json")
    g = json.load(open(path))
    g.pop("inputs_sha256", None)
    g.update(input_fingerprint(cfg, inp, np.array(g["dofs"], dtype=np.int64)))
    with open(path, "w") as f:
        json.dump(g, f)
    print("refreshed", path)


def main(name):
    cfg = get_config(name)
    t0 = time.time()
    inp = generate(cfg, with_phi=False)
    print(f"inputs {time.time() - t0:.1f}s", flush=True)
    K = assemble.assemble_K_large(cfg.nel, inp["E"], inp["fixed"])
    print(f"assembled nnz={K.nnz} {time.time() - t0:.1f}s", flush=True)
    U, its = solve.mgpcg_solve(cfg.nel, K, inp["rhs"], inp["fixed"], cfg.levels, tol=1e-13, row_blocks=16)
    print(f"solved its={its} {time.time() - t0:.1f}s", flush=True)
    idx = sample_dofs(cfg, 1500, seed=11)
    rhs_out = []
    for k in range(cfg.nrhs):
        res = inp["rhs"][k] - K @ U[k]
        rhs_out.append(dict(
            k=k, iters=int(its[k]),
            relres=float(np.linalg.norm(res) / np.linalg.norm(inp["rhs"][k])),
            norm2=float(np.linalg.norm(U[k])),
            work=float(inp["rhs"][k] @ U[k]),
            values=[float(v) for v in U[k][idx]],
        ))
    out = dict(
        config=name, nel=list(cfg.nel), nrhs=cfg.nrhs, levels=cfg.levels,
        oracle="oracle.solve.mgpcg_solve (assembled K via assemble_K_large, Galerkin MG-PCG, tol 1e-13)",
        script="tools/golden_fullsize.py",
        dofs=[int(i) for i in idx], rhs=rhs_out, seconds=round(time.time() - t0, 1),
        **input_fingerprint(cfg, inp, idx),
    )
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{name}_solution.json")
    with open(path, "w") as f:
        json.dump(out, f)
    print("wrote", path, f"{time.time() - t0:.1f}s")


if __name__ == "__main__":
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    if "--inputs-only" in sys.argv:
        refresh_inputs(args[0] if args else "C5")
    else:
        main(args[0] if args else "C5")
