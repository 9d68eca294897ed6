# planes per step of the pair z-march kernel (-DZM_ZS): 3D parity tests, C3 time, step launch time
for z in ${ZSS:-5 3}; do
  export SKS_NVCC_EXTRA="-DZM_ZS=$z"
  python -m paper_2111_00113_b200.build > gpurun_out/zs$z.build 2>&1 || { echo "zs$z build failed"; continue; }
  timeout 600 python -m pytest tests -q -m gpu -x -k "3 or C3" > gpurun_out/zs$z.pytest 2>&1; echo "zs$z pytest rc=$? $(tail -1 gpurun_out/zs$z.pytest)"
  echo "zs$z $(python tools/solve_time.py C3 3 2>&1 | tail -1)"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/zs$z.csv python tools/run_c3_once.py C3 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/zs$z.csv 2>/dev/null | grep step3d | head -1
done
