"""One C3 sGMRES solve with the SRFT sketch (for ncu captures of the srft_* kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2111_00113_b200 as P  # noqa: E402
from inputs import get_config, rhs_normal  # noqa: E402
cfg = get_config("C3")
ctx = P.Context(0)
f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
r = ctx.sgmres_solve(P.StencilOperator(3, cfg.m, cfg.beta), f, d=cfg.d, k=cfg.k, s=cfg.s, seed=cfg.seed, tol=cfg.tol,
                     max_cycles=1, sketch="srft")
torch.cuda.synchronize()
print(r.info["t_total_s"])
