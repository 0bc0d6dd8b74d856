#!/bin/bash
# Round evidence: tests, bench lines (ours + reference arm), isolated
# projector timings, ncu launch list (c2 bench command) and full captures of
# the hot kernels (each ncu run only after the same command exited 0).
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
python bench.py --workload c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --workload c5 --steps 3 --warmup 3 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python tools/bench_projectors.py > gpurun_out/projectors.jsonl 2>&1
C2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C2 > gpurun_out/plain_c2.log 2>&1 && timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2.csv $C2 > gpurun_out/ncu_c2.log 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches_c2.csv "c2 bench (--steps 1 --warmup 1): warm-up + timed + profiled solves" > gpurun_out/launches_c2_summary.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back|k_gs_smem|k_iter_batch" -s 40 -c 8 -o gpurun_out/prof_c2 -f $C2 > gpurun_out/ncu_c2full.log 2>&1
C3="python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline"
$C3 > gpurun_out/plain_c3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back|k_stage" -s 3 -c 3 -o gpurun_out/prof_c3 -f $C3 > gpurun_out/ncu_c3.log 2>&1
C5="python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C5 > gpurun_out/plain_c5.log 2>&1 && timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_forward|k_back" -s 6 -c 2 -o gpurun_out/prof_c5 -f $C5 > gpurun_out/ncu_c5.log 2>&1
ls -la gpurun_out
