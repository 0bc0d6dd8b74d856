#!/bin/bash
# solve tail check: CTK_TRACE timelines and c1/c2 bench
for w in c1 c2; do CTK_TRACE=1 python tools/one_solve.py $w 3 2>&1 | grep "ctk trace" | tail -1; done
for w in c2 c1 c2 c1; do
  python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w', '%.3f'%d['ms_per_step'])"
done
timeout 600 python -m pytest tests/test_gpu_gmres.py -q -x 2>&1 | tail -1
