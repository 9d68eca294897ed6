"""Run ONE sGMRES solve of any stencil/CSR BASELINE config on cuda:0 (for ncu launch lists)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_2111_00113_b200 as P  # noqa: E402
from inputs import get_config, rhs_normal, random_csr_c4  # noqa: E402

cfg = get_config(sys.argv[1] if len(sys.argv) > 1 else "C2")
ctx = P.Context(0)
if cfg.op == "csr":
    rp, ci, v, f = random_csr_c4(cfg.n, seed=cfg.seed)
    A = P.CsrOperator(rp, ci, v, cfg.n)
else:
    A = P.StencilOperator(3 if cfg.op == "stencil3d" else 2, cfg.m, cfg.beta)
    f = rhs_normal(cfg.n, cfg.seed)
ft = torch.from_numpy(f).cuda()
kw = dict(d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol, max_cycles=cfg.max_cycles)
res = ctx.sgmres_solve(A, ft, **kw)
torch.cuda.synchronize()
print(cfg.name, res.info["t_total_s"] * 1e3, "ms", res.info["columns_generated"], "columns")
