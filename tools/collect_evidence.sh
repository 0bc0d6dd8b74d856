#!/bin/bash
# Copy a tools/gpu_evidence.sh run (gpurun_out/) into profiles/ (committed):
# bench lines, reference arm, isolated projector timings, ncu launch list and
# full-capture summaries (dram bytes per launch feed bench.py's roofline.traffic).
set -e
R=${1:-r01}
for c in c1 c2 c3 c4 c5; do tail -1 gpurun_out/bench_$c.json > profiles/${R}_bench_$c.json; done
tail -1 gpurun_out/bench_ref_c2.json > profiles/${R}_bench_ref_c2.json
cp gpurun_out/projectors.jsonl profiles/${R}_projectors_isolated.jsonl
cp gpurun_out/launches_c2_summary.txt profiles/${R}_ncu_launches_c2.txt
python tools/ncu_summary.py gpurun_out/prof_c2.ncu-rep profiles/${R}_ncu_c2_kernels.txt profiles/ncu_c2.json \
  "ncu --set full --clock-control none, python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e (c2), launches inside the warm-up solve" > /dev/null
python tools/ncu_summary.py gpurun_out/prof_c3.ncu-rep profiles/${R}_ncu_c3_kernels.txt profiles/ncu_c3.json \
  "ncu --set full --clock-control none, python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline" > /dev/null
python tools/ncu_summary.py gpurun_out/prof_c5.ncu-rep profiles/${R}_ncu_c5_kernels.txt profiles/ncu_c5.json \
  "ncu --set full --clock-control none, python bench.py --workload c5 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e" > /dev/null
ls -la profiles
