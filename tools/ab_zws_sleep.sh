for v in "0 0" "200 0" "1000 0" "1000 500"; do
  set -- $v
  export SKS_NVCC_EXTRA="-DZWS_SLEEP_B=$1 -DZWS_SLEEP_A=$2"
  python -m paper_2111_00113_b200.build > /dev/null 2>&1 || echo build failed
  SKS_ZM_WS=1 SKS_ZWS_STORE_B=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-oracle > /tmp/b.json 2>/tmp/b.err
  python -c "
import json;l=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);r=l['roofline'];print('sleepB=$1 sleepA=$2', 'solve %.2f'%(l['value']*1e3),'step %.2f'%r['avg_launch_us'])" || tail -3 /tmp/b.err
done
