python -m paper_2111_00113_b200.build > /dev/null 2>&1
for cfg in "2 1" "1 2" "1 1"; do
  set -- $cfg
  echo "NST=$1 CPS=$2"
  SKS_TMA_NST=$1 SKS_TMA_CPS=$2 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:step3d --launch-skip 20 --launch-count 30 --csv python tools/run_c3_once.py C3 1 2>/dev/null | grep step3d | awk -F'","' '{print $NF}' | tr -d '"' | awk '{s+=$1; n++} END {print "avg_us", s/n/1000, n}'
done
