#!/bin/bash
# streamed Gram-Schmidt ring depth (CTK_TS_NBUF) at c4: in-solve K3 mean and solve time
for nb in 2 3 4; do
  CTK_NVCC_EXTRA="-DCTK_TS_NBUF=$nb" python -m paper_2602_17892_b200.build --force > /dev/null 2>&1
  python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('nbuf=$nb c4', '%.2f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})"
done
python -m paper_2602_17892_b200.build --force > /dev/null 2>&1
