"""Time one config's solve (device time from the library, median of R runs after a warm-up)."""
import os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2111_00113_b200 as P
from inputs import get_config, rhs_normal
name = sys.argv[1] if len(sys.argv) > 1 else "C3"
R = int(sys.argv[2]) if len(sys.argv) > 2 else 3
cfg = get_config(name)
ctx = P.Context(0)
f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
A = P.StencilOperator(3 if cfg.op == "stencil3d" else 2, cfg.m, cfg.beta)
ts = []
for r in range(R + 1):
    res = ctx.sgmres_solve(A, f, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol,
                           max_cycles=cfg.max_cycles)
    if r:
        ts.append(res.info["t_total_s"])
print(name, os.environ.get("SKS_RESERVE_SMS", "default"), "t_total_ms", [round(t * 1e3, 2) for t in ts],
      "median", round(statistics.median(ts) * 1e3, 2), "cols", res.info["columns_generated"], "rel", res.info["rel_res_true"])
