#!/bin/bash
# K2 pixels-per-thread (tile height 8 ppt) sweep at c1/c2: isolated B and in-situ solves.
for p in ${PPTS:-1 2}; do
  echo -n "ppt $p: "
  CTK_BACK_PPT=$p python tools/bench_projectors.py c1 c2 | python -c "
import json,sys
print(' '.join('%s B %.4f' % (d['config'], d['B']['ms']) for d in map(json.loads, sys.stdin)), end=' | ')"
  for w in c1 c2; do CTK_BACK_PPT=$p python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w %.3f K2 %.4f' % (d['ms_per_step'], d['kernels']['back']['mean_ms']), end=' | ')"; done; echo
done
