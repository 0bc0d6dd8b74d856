#!/bin/bash
# Full ncu capture of the c2 Arnoldi-step kernels inside a warm solve.
mkdir -p gpurun_out
C2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C2 > gpurun_out/plain_c2.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_forward|k_back|k_gs_smem" -s 300 -c 6 -o gpurun_out/prof_c2step -f $C2 > gpurun_out/ncu_c2step.log 2>&1
tail -3 gpurun_out/ncu_c2step.log
