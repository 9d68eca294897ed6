# pair kernel: first two TMA stages issued before (ZM_EARLY=1) or after (0) the prologue's partials reduction
for E in ${ES:-1 0}; do
  export SKS_NVCC_EXTRA="${EXTRA_PREFIX:--DZM_EARLY=}$E"
  python -m paper_2111_00113_b200.build > gpurun_out/early$E.build 2>&1 || { echo "early$E build failed"; continue; }
  timeout 900 python -m pytest tests -q -m gpu -x -k "3 or C3 or sgmres or edge" > gpurun_out/early$E.pytest 2>&1; echo "early=$E pytest rc=$? $(tail -1 gpurun_out/early$E.pytest)"
  echo "early=$E $(python tools/solve_time.py C3 3 2>&1 | tail -1)"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/early$E.csv python tools/run_c3_once.py C3 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/early$E.csv 2>/dev/null | grep step3d | head -1
done
