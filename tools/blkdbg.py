import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_1909_13585_b200 as mg
from workloads import generate, get_config
for name in ["T2a", "T2c", "T2b"]:
    cfg = get_config(name); inp = generate(cfg)
    d = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    h = mg.mg_setup(cfg.nel, d(inp["E"]), d(inp["fixed"]), cfg.levels, max_iter=200)
    x = torch.empty((cfg.nrhs, inp["rhs"].shape[1]), dtype=torch.float64, device="cuda")
    rep = mg.mgcg_block_solve(h, d(inp["rhs"]), 1e-10, x, raise_on_error=False)
    print(name, rep["status"], rep["iters"], ["%.2e" % v for v in rep["relres"]], ["%.2e" % v for v in rep["true_relres"]], rep["max_iters"])
    rb = mg.mgcg_solve(h, d(inp["rhs"]), 1e-10, x, raise_on_error=False)
    print("  batched", rb["iters"])
