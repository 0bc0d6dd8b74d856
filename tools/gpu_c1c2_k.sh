#!/bin/bash
# krylov/gmres GPU tests + c1/c2 timing x3
timeout 900 python -m pytest tests/test_gpu_krylov.py tests/test_gpu_gmres.py -q -x 2>&1 | tail -1
for w in c2 c1 c2 c1 c2 c1; do
  python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '%.3f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})"
done
