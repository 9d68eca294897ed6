#!/bin/bash
# quick GPU check: parity tests (optionally filtered), one C3 solve timed, kernel launch list of one solve
TAG=${1:-q}; FILT=${2:-}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -m paper_2111_00113_b200.build > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
if [ -n "$FILT" ]; then timeout 900 python -m pytest tests -q -m gpu -x -k "$FILT" > $OUT/pytest.log 2>&1; else timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest.log 2>&1; fi
echo "pytest rc=$?" | tee $OUT/rc.txt; tail -3 $OUT/pytest.log
timeout 600 python tools/run_c3_once.py C3 > $OUT/c3.log 2>&1; echo "c3 rc=$?" | tee -a $OUT/rc.txt; tail -2 $OUT/c3.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv python tools/run_c3_once.py C3 > $OUT/ncu.log 2>&1; echo "ncu rc=$?" | tee -a $OUT/rc.txt
python tools/launches.py $OUT/launches.csv 2>&1 | head -20
