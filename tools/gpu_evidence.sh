#!/bin/bash
# Round evidence: tests, bench lines (ours + reference arm), isolated
# projector timings, ncu launch list (c2 solve) and full captures.
set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
python __graft_entry__.py --smoke 2>&1 | tail -1
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err
python bench.py --workload c1 > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --workload c3 --steps 20 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
python bench.py --workload c4 --steps 2 --warmup 1 > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --workload c5 --steps 2 --warmup 1 > gpurun_out/bench_c5.json 2> gpurun_out/bench_c5.err
python tools/bench_projectors.py > gpurun_out/projectors.jsonl 2>&1
C2="python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e"
$C2 > gpurun_out/plain_c2.log 2>&1 && timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -s 2500 -c 1200 --csv --log-file gpurun_out/launches_c2.csv $C2 > gpurun_out/ncu_c2.log 2>&1
C3="python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline"
$C3 > gpurun_out/plain_c3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward$|k_back$|k_stage" -c 6 -o gpurun_out/prof_c3 $C3 > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_forward$|k_back$|k_cgs2_fused|k_combine" -s 2000 -c 8 -o gpurun_out/prof_c2 $C2 > gpurun_out/ncu_c2full.log 2>&1
ls -la gpurun_out
