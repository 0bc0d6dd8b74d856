#!/bin/bash
# Full ncu capture (with source) of the SMEM Gram-Schmidt step at c1 and c2, mid-solve.
for w in c1 c2; do
  C="python bench.py --workload $w --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
  $C > gpurun_out/plain_gs_$w.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gs_smem" -s 150 -c 1 -o gpurun_out/prof_gs_$w -f $C > gpurun_out/ncu_gs_$w.log 2>&1
done
ls gpurun_out/prof_gs_*
