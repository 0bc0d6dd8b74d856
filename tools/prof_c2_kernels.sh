#!/bin/bash
# ncu --set full of the c2 projector kernels and the Gram-Schmidt kernel
# (after the same command exits 0 without ncu).
mkdir -p gpurun_out
CMD="python tools/bench_projectors.py c2"
$CMD > gpurun_out/plain_proj_c2.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back" -s 4 -c 3 \
    -o gpurun_out/prof_c2_proj -f $CMD > gpurun_out/ncu_c2_proj.log 2>&1
G="python tools/micro/gscheck.py"
$G > /dev/null 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_gs_smem -c 1 \
    -o gpurun_out/prof_gs_smem -f $G > gpurun_out/ncu_gs.log 2>&1
tail -3 gpurun_out/ncu_c2_proj.log gpurun_out/ncu_gs.log
