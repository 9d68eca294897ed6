#!/bin/bash
# usage: tools/prof_kernel.sh TAG KERNEL_REGEX [launch-skip] [config]  -> gpurun_out/TAG/<name>.ncu-rep
TAG=$1; K=$2; SKIP=${3:-2}; CFG=${4:-C3}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python -m paper_2111_00113_b200.build > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/run_c3_once.py $CFG 1 > $OUT/plain.log 2>&1 || { echo plain run failed; tail $OUT/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip $SKIP --launch-count 1 \
  -o $OUT/$K -f python tools/run_c3_once.py $CFG 1 > $OUT/ncu_$K.log 2>&1; echo "ncu rc=$?"
