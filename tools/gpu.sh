#!/bin/bash
# usage: tools/gpu.sh <timeout> '<remote command>'  -- runs under gpurun from /root/repo, prints the tail
cd /root/repo || exit 1
T=$1; shift
/usr/local/graft/bin/gpurun --timeout "$T" -- "$@" > gpurun_out/last_call.txt 2>&1
tail -3 gpurun_out/last_call.txt
