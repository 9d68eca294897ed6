# step-balanced unit partition of the z-march kernels (SKS_ZM_BALANCE = 1) vs the proportional split (0)
python -m paper_2111_00113_b200.build > gpurun_out/bal.build 2>&1 || exit 1
for B in 1 0; do
  export SKS_ZM_BALANCE=$B
  timeout 900 python -m pytest tests -q -m gpu -x -k "3 or C3 or sgmres or edge" > gpurun_out/bal$B.pytest 2>&1; echo "bal=$B pytest rc=$? $(tail -1 gpurun_out/bal$B.pytest)"
  echo "bal=$B $(python tools/solve_time.py C3 3 2>&1 | tail -1)"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/bal$B.csv python tools/run_c3_once.py C3 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/bal$B.csv 2>/dev/null | grep step3d | head -1
done
