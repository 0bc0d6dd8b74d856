#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_gmres.py tests/test_gpu_protocol.py -q -x 2>&1 | tail -15
for w in c1 c2 c4; do timeout 600 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gram_$w.json 2>gpurun_out/gram_$w.err; done
timeout 600 python bench.py --workload c5 --slices-per-gpu 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/gram_c5.json 2>gpurun_out/gram_c5.err
for w in c1 c2 c4 c5; do python -c "
import json,sys
d=json.loads(open('gpurun_out/gram_$w.json').read().strip().splitlines()[-1])
print('$w', round(d['ms_per_step'],3), 'ms', {k:v['mean_ms'] for k,v in d['kernels'].items()})" || tail -5 gpurun_out/gram_$w.err; done
CTK_NO_GRAM_GS=1 timeout 600 python bench.py --workload c4 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/nogram_c4.json 2>&1
python -c "
import json
d=json.loads(open('gpurun_out/nogram_c4.json').read().strip().splitlines()[-1])
print('c4 classic', round(d['ms_per_step'],3), 'ms', {k:v['mean_ms'] for k,v in d['kernels'].items()})"
