#!/bin/bash
# Round-2 first GPU pass: full gpu tests, smoke, default bench.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/r02_gputest.txt
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.txt 2>&1
timeout 600 python bench.py > gpurun_out/r02_bench_c2.json 2> gpurun_out/r02_bench_c2.err
cat gpurun_out/r02_gputest.txt gpurun_out/r02_smoke.txt; tail -c 600 gpurun_out/r02_bench_c2.json
