#!/bin/bash
# Round-2 (late) evidence after the K2 pair pre-pass: ncu launch list of the
# default bench command (c5 x 8 slices) and --set full captures of K1 / K2 /
# the pair pre-pass at c5 (single slice).
set -x
mkdir -p gpurun_out/p4
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/p4/plain_default.json 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/p4/launches_default.csv $B > gpurun_out/p4/ncu_default.log 2>&1
C5="python bench.py --workload c5 --slices-per-gpu 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C5 > gpurun_out/p4/plain_c5.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back|k_pairs" -s 30 -c 3 -o gpurun_out/p4/c5_proj $C5 > gpurun_out/p4/ncu_c5_proj.log 2>&1
ls -la gpurun_out/p4
