python -m paper_2111_00113_b200.build > /dev/null 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_determinism.py -q -m gpu -x 2>&1 | tail -3
SKS_CHEB_SYNC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k chebyshev 2>&1 | tail -2
for v in 0 1; do SKS_CHEB_SYNC=$v timeout 600 python tools/cheb_time.py 2>&1 | sed "s/^/sync=$v /"; done
