#!/bin/bash
# compile-time CSR SpMV variants on C4 (tools/ab_csr.sh timing per build): tools/ab_csr_build.sh "-DX=0" "" ...
for X in "$@"; do
  SKS_NVCC_EXTRA="$X" python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo "build failed for '$X'"; exit 1; }
  echo "== build '$X'"
  NOBUILD=1 VARIANTS="- -" bash tools/ab_csr.sh 2>&1 | grep -v "^python"
done
python -m paper_2111_00113_b200.build > /dev/null 2>&1
