#!/bin/bash
# Unmodified reference on the GPU box's host cores + the
# c5 stream-A timeline (does the side-stream iterate kernel lengthen it?).
nproc; cat /proc/cpuinfo | grep "model name" | head -1
timeout 1500 python tools/time_reference_cpu.py c1 c2 c3 > gpurun_out/ref_cpu.jsonl 2> gpurun_out/ref_cpu.err
cat gpurun_out/ref_cpu.jsonl | cut -c1-400
CTK_TRACE=1 timeout 300 python bench.py --workload c5 --slices-per-gpu 1 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | grep "ctk trace" | tail -3
CTK_TRACE=1 CTK_ITER_BATCH=0 timeout 300 python bench.py --workload c5 --slices-per-gpu 1 --steps 2 --warmup 2 --no-cpu-baseline --no-e2e 2>&1 | grep "ctk trace" | tail -2
