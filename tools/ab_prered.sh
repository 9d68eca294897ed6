#!/bin/bash
# last-CTA partial pre-reduction (SKS_PRERED) A/B: GPU suite with it on, then C3 bench / C2 / C5 timing
python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
SKS_PRERED=1 timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -2
for rep in 1 2; do
for v in "SKS_PRERED=0" "SKS_PRERED=1"; do
  env $v timeout 600 python bench.py --config C3 --steps 10 --warmup 3 --no-oracle 2>/dev/null | tail -1 | python -c "
import json, sys
l = json.loads(sys.stdin.read()); r = l['roofline']
print('[$v] C3 solve %.2f ms step %.2f us frac %.3f cols %d' % (l['value'] * 1e3, r['avg_launch_us'], r['frac'], l['config']['columns_generated']))"
  env $v timeout 300 python tools/cheb_time.py 2>&1 | grep '"C2"' | sed "s/^/[$v] /"
  env $v python tools/sweep.py C5 2>&1 | cut -c1-120 | sed "s/^/[$v] /"
done
done
