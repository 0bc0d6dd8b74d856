#!/bin/bash
# batched-iterate check: krylov + gmres GPU tests, then c2/c1 bench with and without batching
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_gmres.py -q -x 2>&1 | tail -4
for w in c2 c1; do
  for ib in 1 0; do
    CTK_ITER_BATCH=$ib python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ib${ib}_$w.json 2>gpurun_out/ib${ib}_$w.err || tail -3 gpurun_out/ib${ib}_$w.err
    python -c "
import json; d=json.loads(open('gpurun_out/ib${ib}_$w.json').read().strip().splitlines()[-1]); print('batch=$ib $w', '%.4e'%d['value'], d['ms_per_step'], 'e2e %.4e'%d['e2e']['value'], {k:(v['mean_ms'],v['launches']) for k,v in d['kernels'].items()})"
  done
done
