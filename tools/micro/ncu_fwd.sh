#!/bin/bash
W=${1:-c4}
CMD="python tools/bench_projectors.py $W"
$CMD > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:"k_forward" -s 3 -c 1 -o gpurun_out/prof_fwd_$W -f $CMD > gpurun_out/ncu_fwd_$W.log 2>&1
tail -1 gpurun_out/ncu_fwd_$W.log
