python -m paper_2111_00113_b200.build > /dev/null 2>&1
for v in "SKS_TMA_CPS=1" "SKS_TMA_CPS=2" "SKS_TMA_CPS=4" "SKS_NO_TMA=1"; do
  env $v timeout 300 python tools/cheb_time.py 2>&1 | grep C2 | sed "s/^/[$v] /"
done
