#!/bin/bash
# Ritz-vector kernel variants at C5 (ncu launch durations): tools/ab_ritz.sh "-DRV_RB=1" ...
for X in "$@"; do
  SKS_NVCC_EXTRA="$X" python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo "build failed '$X'"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:ritz_vectors python tools/run_srr_once.py C5 1 2>/dev/null | grep -E "duration|dram__" | tr -s ' ' | sed "s/^/[$X] /"
done
python -m paper_2111_00113_b200.build > /dev/null 2>&1
