#!/bin/bash
# A/B timing of an environment switch on the C3 bench workload (no oracle leg):
#   tools/ab_env.sh TAG "VAR=a" "VAR=b" [config]
TAG=$1; A=$2; B=$3; CFG=${4:-C3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -m paper_2111_00113_b200.build > $OUT/build.log 2>&1 || { echo build failed; tail -20 $OUT/build.log; exit 1; }
for rep in 1 2; do
  for E in "$A" "$B"; do
    env $E timeout 600 python bench.py --config $CFG --steps 10 --warmup 3 --no-oracle > $OUT/bench_${E//=/_}_$rep.json 2> $OUT/bench_${E//=/_}_$rep.err
    python - "$OUT/bench_${E//=/_}_$rep.json" "$E" <<'PY'
import json, sys
l = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
r = l["roofline"]
print(sys.argv[2], "solve %.2f ms" % (l["value"] * 1e3), "step %.2f us" % r["avg_launch_us"], "frac %.3f" % r["frac"],
      "cols", l["config"]["columns_generated"], "res %.3e" % l["config"]["rel_res_true"])
PY
  done
done
