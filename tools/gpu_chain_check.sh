#!/bin/bash
# K1 -> K2 chaining check: GPU solver tests (incl. bitwise chained vs unchained), then c2/c5 bench both ways
timeout 900 python -m pytest tests/test_gpu_gmres.py tests/test_gpu_krylov.py -q -x 2>&1 | tail -2
for w in c2 c2; do for nc in 0 1; do
  CTK_NO_CHAIN=$nc python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w nochain=$nc', '%.3f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})"
done; done
for nc in 0 1; do
  CTK_NO_CHAIN=$nc python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 nochain=$nc', '%.3f'%d['ms_per_step'])"
done
