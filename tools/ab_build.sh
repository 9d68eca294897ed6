#!/bin/bash
# A/B of compile-time variants (SKS_NVCC_EXTRA) on the C3 bench workload and the C2 solve:
#   tools/ab_build.sh "-DOPT=0" "" ...   ("" = the default build); the default build is restored at the end
for X in "$@"; do
  export SKS_NVCC_EXTRA="$X"; python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo "build failed for '$X'"; exit 1; }
  for rep in 1 2; do
    timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-oracle 2>/dev/null | tail -1 | python -c "
import json, sys
l = json.loads(sys.stdin.read()); r = l['roofline']
print('[$X] C3 solve %.2f ms step %.2f us frac %.3f' % (l['value'] * 1e3, r['avg_launch_us'], r['frac']))"
  done
  timeout 300 python tools/cheb_time.py 2>&1 | grep '"C2"' | sed "s/^/[$X] /"
done
python -m paper_2111_00113_b200.build > /dev/null 2>&1
