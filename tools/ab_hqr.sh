#!/bin/bash
# A/B of Francis-QR compile-time options on the C5 small side (usage: tools/ab_hqr.sh "-DOPT_A" "-DOPT_B" ...;
# "" = the default build)
set -u
mkdir -p gpurun_out
for X in "$@"; do
  SKS_NVCC_EXTRA="$X" python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo "build failed for '$X'"; exit 1; }
  echo "== variant '$X'"
  SKS_DEBUG_HQR=1 python tools/run_srr_once.py C5 2 2>&1 | grep -E "hqr:|t_total" | cut -c1-160
done
python -m paper_2111_00113_b200.build > /dev/null 2>&1
