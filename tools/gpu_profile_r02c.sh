#!/bin/bash
# Round-2 (final build) evidence: full GPU suite, smoke, both bench arms, the
# ncu launch list of the default bench command (c5 x 8 slices) and a --set full
# capture of the streamed Gram-Schmidt step at c4 (k = 50) and c5 (k = 30).
set -x
mkdir -p gpurun_out/p5
python -m pytest tests -m gpu -x -q > gpurun_out/p5/gputest_full.txt 2>&1; tail -3 gpurun_out/p5/gputest_full.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/p5/smoke.txt 2>&1; tail -1 gpurun_out/p5/smoke.txt
python bench.py --impl reference > gpurun_out/p5/bench_ref.json 2> gpurun_out/p5/bench_ref.err
python bench.py > gpurun_out/p5/bench_c5x8.json 2> gpurun_out/p5/bench_c5x8.err; cut -c1-300 gpurun_out/p5/bench_c5x8.json
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$B > gpurun_out/p5/plain_default.json 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1400 --csv --log-file gpurun_out/p5/launches_default.csv $B > gpurun_out/p5/ncu_default.log 2>&1
C4="python bench.py --workload c4 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C4 > gpurun_out/p5/plain_c4.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_stream -s 50 -c 1 -o gpurun_out/p5/c4_gs $C4 > gpurun_out/p5/ncu_c4_gs.log 2>&1
C5="python bench.py --workload c5 --slices-per-gpu 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C5 > gpurun_out/p5/plain_c5.json 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gs_stream -s 30 -c 1 -o gpurun_out/p5/c5_gs $C5 > gpurun_out/p5/ncu_c5_gs.log 2>&1
ls -la gpurun_out/p5
