python -m paper_2111_00113_b200.build > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
SKS_MPK_S=4 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "chebyshev" 2>&1 | tail -2
for v in "-" "SKS_MPK_S=4"; do
  EE=$v; [ "$v" = "-" ] && EE=""
  env $EE timeout 300 python tools/cheb_time.py 2>&1 | grep C2 | grep chebyshev | sed "s/^/[$v] /"
done
