#!/bin/bash
# one-barrier cooperative 2D kernel (step_coop1_kernel, SKS_COOP1_MAXN) vs the per-column step launches:
# the whole GPU suite with it enabled for every 2D problem up to 300k points, then C1 / C2 timing
python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
SKS_COOP1_MAXN=300000 timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
for v in "SKS_COOP1_MAXN=0" "SKS_COOP1_MAXN=300000"; do
  env $v timeout 300 python tools/cheb_time.py 2>&1 | grep C2 | sed "s/^/[$v] /"
  env $v timeout 300 python - <<'PY' | sed "s/^/[$v] /"
import sys, statistics
sys.path.insert(0, ".")
import torch, paper_2111_00113_b200 as P
from inputs import get_config, rhs_normal
for name in ("C1", "C2"):
    cfg = get_config(name)
    ctx = P.Context(0)
    f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
    ts = []
    for r in range(4):
        res = ctx.sgmres_solve(P.StencilOperator(2, cfg.m, cfg.beta), f, d=cfg.d, k=cfg.k, s=cfg.s, seed=cfg.seed,
                               max_cycles=cfg.max_cycles, tol=cfg.tol)
        if r: ts.append(res.info["t_total_s"])
    i = res.info
    print("%s %.3f ms basis %.3f ms, %d cycles, %d columns generated, %.2f us/col, rel %.4e" % (
        name, statistics.median(ts) * 1e3, i["t_basis_s"] * 1e3, i["cycles"], i["columns_generated"],
        i["t_basis_s"] * 1e6 / i["columns_generated"], i["rel_res_true"]))
    ctx.close()
PY
done
