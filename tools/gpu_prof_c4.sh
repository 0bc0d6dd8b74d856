#!/bin/bash
# c4 (AB, 1024^2, L = 2.1M): full ncu captures of the streamed Gram-Schmidt step,
# the projectors and the batched iterate norms (after the plain command exits 0)
C4="python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C4 > gpurun_out/plain_c4.log 2>&1 && timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_gs_stream|k_forward|k_back|k_iter_batch" -s 80 -c 6 -o gpurun_out/prof_c4 -f $C4 > gpurun_out/ncu_c4.log 2>&1
tail -2 gpurun_out/ncu_c4.log
