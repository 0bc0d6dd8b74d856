#!/bin/bash
# Round-2 (final build): --set full captures of K1 / K2 / the pair pre-pass at c5
# (single slice) for profiles/ncu_c5.json (bench.py roofline.traffic / binding).
set -x
mkdir -p gpurun_out/p6
C5="python bench.py --workload c5 --slices-per-gpu 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C5 > gpurun_out/p6/plain_c5.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back|k_pairs" -s 30 -c 3 -o gpurun_out/p6/c5_proj $C5 > gpurun_out/p6/ncu_c5_proj.log 2>&1
ls -la gpurun_out/p6
