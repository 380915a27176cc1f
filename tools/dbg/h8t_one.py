"""Debug driver: one 3D matvec through the C ABI on a small grid, compared with the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
import paper_1909_13585_b200 as mg
from oracle import assemble
from workloads import generate, get_config, rough_vectors
name = sys.argv[1] if len(sys.argv) > 1 else "T3a"
cfg = get_config(name); inp = generate(cfg)
K = assemble.assemble_K(cfg.nel, inp["E"], inp["fixed"])
d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
h = mg.mg_setup(cfg.nel, d(inp["E"]), d(inp["fixed"]), cfg.levels)
X = rough_vectors(cfg, 3)
y = torch.empty((3, X.shape[1]), dtype=torch.float64, device="cuda")
mg.mg_matvec(h, 0, d(X), y)
torch.cuda.synchronize()
yo = (K @ X.T).T
err = np.linalg.norm(y.cpu().numpy() - yo, axis=1) / np.linalg.norm(yo, axis=1)
print(name, "matvec rel err", err)
