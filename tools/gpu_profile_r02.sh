#!/bin/bash
# Round-2 evidence: ncu launch list of the default bench command (c5 x 8
# slices) and --set full captures of the c5 / c4 kernels (single slice).
set -x
mkdir -p gpurun_out/p2
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/p2/plain_default.json 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1300 --csv --log-file gpurun_out/p2/launches_default.csv $B > gpurun_out/p2/ncu_default.log 2>&1
C5="python bench.py --workload c5 --slices-per-gpu 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C5 > gpurun_out/p2/plain_c5.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -s 10 -c 1 -o gpurun_out/p2/c5_fwd $C5 > gpurun_out/p2/ncu_c5_fwd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_back -s 10 -c 1 -o gpurun_out/p2/c5_back $C5 > gpurun_out/p2/ncu_c5_back.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_stream -s 30 -c 1 -o gpurun_out/p2/c5_gs $C5 > gpurun_out/p2/ncu_c5_gs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_batch -s 3 -c 1 -o gpurun_out/p2/c5_iter $C5 > gpurun_out/p2/ncu_c5_iter.log 2>&1
C4="python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C4 > gpurun_out/p2/plain_c4.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_stream -s 50 -c 1 -o gpurun_out/p2/c4_gs $C4 > gpurun_out/p2/ncu_c4_gs.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_iter_batch -s 6 -c 1 -o gpurun_out/p2/c4_iter $C4 > gpurun_out/p2/ncu_c4_iter.log 2>&1
C2="python bench.py --workload c2 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C2 > gpurun_out/p2/plain_c2.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_smem -s 40 -c 1 -o gpurun_out/p2/c2_gs $C2 > gpurun_out/p2/ncu_c2_gs.log 2>&1
ls -la gpurun_out/p2
