#!/bin/bash
CMD="python tools/bench_projectors.py c3"
$CMD > /dev/null 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_back -s 3 -c 1 -o gpurun_out/prof_back_c3 -f $CMD > gpurun_out/ncu_back.log 2>&1
tail -2 gpurun_out/ncu_back.log
