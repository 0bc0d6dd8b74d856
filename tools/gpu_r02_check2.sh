#!/bin/bash
timeout 600 python -m pytest tests/test_gpu_krylov.py -q -x 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_protocol.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -6
timeout 600 python -m pytest tests/test_gpu_large_solves.py -q -x -s -k c4 2>&1 | tail -4
for w in c1 c2 c4; do timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/g2_$w.json 2>gpurun_out/g2_$w.err; python -c "
import json
d=json.loads(open('gpurun_out/g2_$w.json').read().strip().splitlines()[-1])
print('$w', round(d['ms_per_step'],3), 'ms', {k:v['mean_ms'] for k,v in d['kernels'].items()})" || tail -3 gpurun_out/g2_$w.err; done
timeout 300 python bench.py --workload c4 --shard angles --steps 3 --warmup 2 > gpurun_out/g2_c4_shard.json 2>gpurun_out/g2_c4_shard.err; tail -c 400 gpurun_out/g2_c4_shard.json; tail -3 gpurun_out/g2_c4_shard.err
timeout 300 python bench.py --workload c3 --shard angles --steps 5 --warmup 3 > gpurun_out/g2_c3_shard.json 2>gpurun_out/g2_c3_shard.err; tail -c 300 gpurun_out/g2_c3_shard.json; tail -3 gpurun_out/g2_c3_shard.err
