"""Time y = G(u) phi on a config through the C ABI (device buffers), CUDA events."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1909_13585_b200 as mg
from workloads import generate, get_config
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = get_config(name); inp = generate(cfg)
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
h = mg.mg_setup(cfg.nel, d(inp["E"]), d(inp["fixed"]), cfg.levels)
phi = d(inp["phi"]); u = d(inp["rhs"][1]); Es = d(inp["Es"])
y = torch.empty_like(phi)
for _ in range(3):
    mg.stress_stiffness_apply(h, Es, u, phi, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    mg.stress_stiffness_apply(h, Es, u, phi, y)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
n, m, k = inp["phi"].shape[1], inp["E"].size, inp["phi"].shape[0]
alg = 8.0 * (n + m + 2 * n * k)
print(f"{name} nphi={k} G(u)phi {ms:.3f} ms, alg {alg/1e9:.3f} GB -> {alg/ms/1e6:.0f} GB/s; launches {mg.mg_kernel_launches(h)}")
