#!/bin/bash
# A/B/C timing of environment variants on a bench workload (no oracle leg):
#   tools/ab_multi.sh TAG CONFIG "ENV1" "ENV2" ...     (each ENV is "VAR=a VAR2=b" or "-" for none)
TAG=$1; CFG=$2; shift 2
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -m paper_2111_00113_b200.build > $OUT/build.log 2>&1 || { echo build failed; tail -20 $OUT/build.log; exit 1; }
for rep in 1 2; do
  i=0
  for E in "$@"; do
    i=$((i+1))
    EE=$E; [ "$E" = "-" ] && EE=""
    env $EE timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-oracle > $OUT/v${i}_$rep.json 2> $OUT/v${i}_$rep.err
    python - "$OUT/v${i}_$rep.json" "$E" <<'PY'
import json, sys
try:
    l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    r = l["roofline"]
    print(sys.argv[2], "| solve %.2f ms" % (l["value"] * 1e3), "step %.2f us" % r["avg_launch_us"], "frac %.3f" % r["frac"],
          "cols", l["config"]["columns_generated"], "res %.3e" % l["config"]["rel_res_true"])
except Exception as e:
    print(sys.argv[2], "FAILED", e)
PY
  done
done
