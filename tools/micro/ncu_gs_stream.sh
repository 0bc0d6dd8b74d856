#!/bin/bash
C="python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C > gpurun_out/plain_c4.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gs_stream|k_cgs2_fused" -s 60 -c 1 -o gpurun_out/prof_gs4 -f $C > gpurun_out/ncu_gs4.log 2>&1
CTK_NO_STREAM_GS=1 $C > gpurun_out/plain_c4b.log 2>&1 && CTK_NO_STREAM_GS=1 timeout 900 ncu --set full --clock-control none -k regex:"k_cgs2_fused" -s 60 -c 1 -o gpurun_out/prof_gs4old -f $C > gpurun_out/ncu_gs4old.log 2>&1
tail -2 gpurun_out/ncu_gs4.log gpurun_out/ncu_gs4old.log
