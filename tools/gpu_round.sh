#!/bin/bash
# One measurement pass on the B200 box (run under gpurun from the repo root):
#   parity tests, smoke, bench (default), ncu launch list of the bench command, and one
#   ncu --set full capture each of the fused step kernel and the sketch kernel.
# usage: tools/gpu_round.sh [tag] [stages]   stages: any of t s b l f (default: all)
TAG=${1:-r01}
ST=${2:-tsblf}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > "$OUT/nvsmi.txt" 2>&1
python -m paper_2111_00113_b200.build > "$OUT/build.log" 2>&1
if [[ $ST == *t* ]]; then
  timeout 1500 python -m pytest tests -q -m gpu -rA > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
fi
if [[ $ST == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
fi
if [[ $ST == *b* ]]; then
  timeout 900 python bench.py > "$OUT/bench.log" 2>&1; echo "bench rc=$?" >> "$OUT/rc.txt"
fi
if [[ $ST == *l* ]]; then
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file "$OUT/launches.csv" \
    python bench.py --steps 1 --warmup 3 --no-oracle > "$OUT/ncu_launches.log" 2>&1; echo "ncu-list rc=$?" >> "$OUT/rc.txt"
  python tools/launches.py "$OUT/launches.csv" > "$OUT/launches_summary.txt" 2>&1
fi
if [[ $ST == *f* ]]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:step3d_zm --launch-skip 60 --launch-count 1 \
    -o "$OUT/step3d" -f python tools/run_c3_once.py C3 1 > "$OUT/ncu_step.log" 2>&1; echo "ncu-step rc=$?" >> "$OUT/rc.txt"
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:sketch_v5 --launch-skip 4 --launch-count 1 \
    -o "$OUT/sketch" -f python tools/run_c3_once.py C3 1 > "$OUT/ncu_sketch.log" 2>&1; echo "ncu-sketch rc=$?" >> "$OUT/rc.txt"
fi
cat "$OUT/rc.txt"
