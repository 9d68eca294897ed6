#!/bin/bash
# Round-2 evidence pass on the B200 box (run under gpurun from the repo root):
#   t: GPU parity suite (incl. the full-size oracle goldens)      s: smoke
#   c: compute-sanitizer racecheck / synccheck / memcheck on tools/sanitize_cases.py
#   n: ncu --set full of the kernels round 1 left uncaptured (step2d_ym C5, step2d_tma C2, csr_* C4,
#      assemble_kernel + panel_kernel C3)
#   o: the CPU oracle on one full C3 cycle, 1 thread and all host cores (tools/time_oracle_cycle.py)
# usage: tools/gpu_r02a.sh TAG [stages]
TAG=${1:-r02a}
ST=${2:-tscno}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
: > "$OUT/rc.txt"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > "$OUT/nvsmi.txt" 2>&1
python -m paper_2111_00113_b200.build > "$OUT/build.log" 2>&1 || { echo "build failed"; tail -30 "$OUT/build.log"; exit 1; }
if [[ $ST == *t* ]]; then
  timeout 1800 python -m pytest tests -q -m gpu -rA > "$OUT/pytest_gpu.log" 2>&1; echo "pytest rc=$?" >> "$OUT/rc.txt"
  tail -3 "$OUT/pytest_gpu.log"
fi
if [[ $ST == *s* ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.log" 2>&1; echo "smoke rc=$?" >> "$OUT/rc.txt"
fi
if [[ $ST == *c* ]]; then
  for tool in racecheck synccheck memcheck; do
    timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py \
      > "$OUT/sanitizer_$tool.log" 2>&1
    echo "sanitizer-$tool rc=$?" >> "$OUT/rc.txt"
  done
fi
if [[ $ST == *n* ]]; then
  NCU="ncu --set full --clock-control none --import-source on"
  timeout 600 $NCU -k regex:step2d_ym --launch-skip 20 --launch-count 1 -o "$OUT/step2d_ym_c5" -f \
    python tools/run_srr_once.py C5 > "$OUT/ncu_ym.log" 2>&1; echo "ncu-ym rc=$?" >> "$OUT/rc.txt"
  timeout 600 $NCU -k regex:step2d_tma --launch-skip 40 --launch-count 1 -o "$OUT/step2d_tma_c2" -f \
    python tools/run_cfg_once.py C2 > "$OUT/ncu_tma.log" 2>&1; echo "ncu-tma rc=$?" >> "$OUT/rc.txt"
  timeout 600 $NCU -k regex:csr_ --launch-skip 4 --launch-count 2 -o "$OUT/csr_c4" -f \
    python tools/run_cfg_once.py C4 > "$OUT/ncu_csr.log" 2>&1; echo "ncu-csr rc=$?" >> "$OUT/rc.txt"
  timeout 600 $NCU -k regex:"assemble|panel_kernel" --launch-skip 2 --launch-count 2 -o "$OUT/assemble_panel_c3" -f \
    python tools/run_cfg_once.py C3 > "$OUT/ncu_asm.log" 2>&1; echo "ncu-asm rc=$?" >> "$OUT/rc.txt"
  for r in "$OUT"/*.ncu-rep; do python tools/ncu_summary.py "$r"; done > "$OUT/ncu_summaries.txt" 2>&1
fi
if [[ $ST == *o* ]]; then
  timeout 2400 python tools/time_oracle_cycle.py --config C3 > "$OUT/oracle_cycle_c3.json" 2> "$OUT/oracle_cycle_c3.log"
  echo "oracle-cycle rc=$?" >> "$OUT/rc.txt"
fi
cat "$OUT/rc.txt"
