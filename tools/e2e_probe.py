"""Wall-clock probe of the C-ABI calls with device vs pinned host buffers (C5 by default):
where does the end-to-end step spend the time that the device-timed step does not?"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_1909_13585_b200 as mg  # noqa: E402
from workloads import generate, get_config  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C5")
inp = generate(cfg)
dev = torch.device("cuda:0")
d = {k: torch.from_numpy(inp[k]).to(dev) for k in ("E", "Es", "fixed", "rhs", "phi")}
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
hE, hEs, hrhs, hphi = pin(inp["E"]), pin(inp["Es"]), pin(inp["rhs"]), pin(inp["phi"])
R, n = inp["rhs"].shape
nphi = cfg.nphi
hx = torch.empty((R, n), dtype=torch.float64).pin_memory().numpy()
hy = torch.empty((nphi, n), dtype=torch.float64).pin_memory().numpy()
x = torch.empty_like(d["rhs"])
y = torch.empty((nphi, n), dtype=torch.float64, device=dev)
h = mg.mg_setup(cfg.nel, d["E"], d["fixed"], cfg.levels)
torch.cuda.synchronize()


def wall(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t))
    return min(ts)


print("update_modulus dev  %.2f ms" % wall(lambda: mg.mg_update_modulus(h, d["E"])))
print("update_modulus host %.2f ms" % wall(lambda: mg.mg_update_modulus(h, hE)))
print("solve dev           %.2f ms" % wall(lambda: mg.mgcg_solve(h, d["rhs"], cfg.tol, x)))
print("solve host          %.2f ms" % wall(lambda: mg.mgcg_solve(h, hrhs, cfg.tol, hx)))
if nphi:
    print("gphi dev            %.2f ms" % wall(lambda: mg.stress_stiffness_apply(h, d["Es"], x[0], d["phi"][:nphi], y)))
    hx0 = np.ascontiguousarray(hx[0])
    print("gphi host           %.2f ms" % wall(lambda: mg.stress_stiffness_apply(h, hEs, hx0, hphi[:nphi], hy)))
t = torch.empty(R * n, dtype=torch.float64, device=dev)
hb = torch.empty(R * n, dtype=torch.float64).pin_memory()
print("H2D %d MB  %.2f ms" % (8 * R * n >> 20, wall(lambda: t.copy_(hb, non_blocking=True))))
print("D2H %d MB  %.2f ms" % (8 * R * n >> 20, wall(lambda: hb.copy_(t, non_blocking=True))))
