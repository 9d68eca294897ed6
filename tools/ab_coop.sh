#!/bin/bash
# cooperative small-problem batches (stencil_coop.cu) vs the per-column kernels (SKS_COOP_MAXN=0): parity + timing
python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 300 python -m pytest tests/test_gpu_determinism.py tests/test_gpu_golden.py -q -m gpu -x -k "C1 or C2 or bitwise" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge.py tests/test_gpu_whiten.py -q -m gpu -x 2>&1 | tail -2
for v in "-" "SKS_COOP_MAXN=0"; do
  EE=$v; [ "$v" = "-" ] && EE=""
  env $EE timeout 300 python tools/cheb_time.py 2>&1 | grep C2 | sed "s/^/[$v] /"
  env $EE timeout 300 python - <<'PY' | sed "s/^/[$v] /"
import sys, statistics
sys.path.insert(0, ".")
import torch, paper_2111_00113_b200 as P
from inputs import get_config, rhs_normal
cfg = get_config("C1")
ctx = P.Context(0)
f = torch.from_numpy(rhs_normal(cfg.n, cfg.seed)).cuda()
ts = []
for r in range(6):
    res = ctx.sgmres_solve(P.StencilOperator(2, cfg.m, cfg.beta), f, d=cfg.d, k=cfg.k, s=cfg.s, seed=cfg.seed, max_cycles=1)
    if r: ts.append(res.info["t_total_s"])
print("C1 %.3f ms" % (statistics.median(ts) * 1e3), res.info["columns_generated"], "%.4e" % res.info["rel_res_true"])
PY
done
