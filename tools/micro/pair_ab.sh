# A/B of the z-march step kernel's columns-per-thread (SKS_ZM_NPY = 1, 2): 3D parity tests,
# C3 solve time, and the step kernel's per-launch time from an ncu launch list.
python -m paper_2111_00113_b200.build > gpurun_out/npy.build 2>&1 || exit 1
for P in ${NPYS:-1 2}; do
  export SKS_ZM_NPY=$P
  timeout 600 python -m pytest tests -q -m gpu -x -k "3 or C3" > gpurun_out/npy$P.pytest 2>&1; echo "npy$P pytest rc=$? $(tail -1 gpurun_out/npy$P.pytest)"
  echo "npy$P $(python tools/solve_time.py C3 3 2>&1 | tail -1)"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/npy$P.csv python tools/run_c3_once.py C3 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/npy$P.csv 2>/dev/null | grep step3d | head -2
done
