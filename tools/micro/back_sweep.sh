#!/bin/bash
# K2 sweep: PPT-4 resident-CTA bound (build) x split reduction (1 cluster, 2 global):
# isolated B at c1..c5 and the in-situ c2 solve.
for mb in ${MINB4S:-5 6}; do
  CTK_NVCC_EXTRA="-DCTK_BACK_MINB4=$mb" python -c "from paper_2602_17892_b200 import build; build.build(force=True)" || exit 1
  for red in ${REDS:-2 1}; do
    echo -n "minb4 $mb red $red: "
    CTK_BACK_RED=$red CTK_BACK_MAXS=${MAXS:-8} python tools/bench_projectors.py ${CONFS:-c1 c2 c3 c4 c5} | python -c "
import json,sys
print(' '.join('%s %.4f' % (d['config'], d['B']['ms']) for d in map(json.loads, sys.stdin)), end=' | ')"
    CTK_BACK_RED=$red CTK_BACK_MAXS=${MAXS:-8} python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 solve %.3f ms' % d['ms_per_step'], {k: v['mean_ms'] for k, v in d['kernels'].items()})"
  done
done
