[ -z "$NOBUILD" ] && python -m paper_2111_00113_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_loopback.py tests/test_gpu_determinism.py -q -m gpu -k "csr or C4" 2>&1 | tail -2
for v in ${VARIANTS:-"SKS_CSR_BATCH=8" "-" "SKS_CSR_BATCH=2" "SKS_CSR_V2=1"}; do
  EE=$v; [ "$v" = "-" ] && EE=""
  env $EE python - <<'PY'
import os, sys, statistics
sys.path.insert(0, ".")
import torch, paper_2111_00113_b200 as P
from inputs import get_config, random_csr_c4
cfg = get_config("C4")
rp, ci, v, f = random_csr_c4(cfg.n, seed=cfg.seed)
ctx = P.Context(0)
A = P.CsrOperator(rp, ci, v, cfg.n)
ft = torch.from_numpy(f).cuda()
ts = []
for r in range(5):
    res = ctx.sgmres_solve(A, ft, d=cfg.d, k=cfg.k, s=cfg.s, zeta=cfg.zeta, seed=cfg.seed, tol=cfg.tol, max_cycles=cfg.max_cycles)
    if r: ts.append(res.info["t_total_s"])
print("v2" if os.environ.get("SKS_CSR_V2") else "v1", os.environ.get("SKS_CSR_BATCH", "4"), "L2win", os.environ.get("SKS_CSR_L2", "1"), "C4 %.3f ms" % (statistics.median(ts) * 1e3), "gen", res.info["columns_generated"], "used", res.info["columns"], "res %.3e" % res.info["rel_res_true"])
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv python tools/run_cfg_once.py C4 > /dev/null 2>&1; python tools/launches.py gpurun_out/c4_launches.csv 2>/dev/null | head -12
