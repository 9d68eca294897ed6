"""One C2 solve on cuda:0 (first cycle only unless CYCLES is set), for ncu captures of the small-problem kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2111_00113_b200 as P  # noqa: E402
from inputs import get_config, rhs_normal  # noqa: E402
cfg = get_config(os.environ.get("CFG", "C2"))
ctx = P.Context(0)
f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
res = ctx.sgmres_solve(P.StencilOperator(2, cfg.m, cfg.beta), f, d=cfg.d, k=cfg.k, s=cfg.s, seed=cfg.seed,
                       max_cycles=int(os.environ.get("CYCLES", "1")), tol=cfg.tol)
torch.cuda.synchronize()
print(cfg.name, res.info["t_total_s"] * 1e3, "ms", res.info["columns_generated"], "columns")
