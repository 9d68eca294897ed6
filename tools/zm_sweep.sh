#!/bin/bash
# z-march tile / CTAs-per-SM sweep: for each "TX TY CPS", rebuild with -DZM_TX/TY/CPS, run the 3D parity
# tests, time the C3 solve, and list the step kernel's launch time.
while [ $# -ge 3 ]; do
  tx=$1; ty=$2; cps=$3; shift 3
  tag="zm_${tx}x${ty}_c${cps}"
  export SKS_NVCC_EXTRA="-DZM_TX=$tx -DZM_TY=$ty -DZM_CPS=$cps"  # also seen by the tests' build() calls
  python -m paper_2111_00113_b200.build > gpurun_out/$tag.build 2>&1 || { echo "$tag build failed"; continue; }
  timeout 600 python -m pytest tests -q -m gpu -x -k "3 or C3" > gpurun_out/$tag.pytest 2>&1; echo "$tag pytest rc=$? $(tail -1 gpurun_out/$tag.pytest)"
  echo "$tag $(python tools/solve_time.py C3 3 2>&1 | tail -1)"
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$tag.csv python tools/run_c3_once.py C3 1 > /dev/null 2>&1
  python tools/launches.py gpurun_out/$tag.csv 2>/dev/null | grep step3d | head -1
  grep -m1 "step3d_zm_kernel<2, 4, 1, 1>" gpurun_out/$tag.csv | cut -d, -f8,9
done
