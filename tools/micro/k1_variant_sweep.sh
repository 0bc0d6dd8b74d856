#!/bin/bash
# K1 build variants (resident-CTA bound, unroll, dynamic-smem occupancy cap):
# isolated applies c1..c5 at the default splits and the in-situ c2 solve.
for v in ${VARIANTS:-"8 8 0" "8 16 0" "8 4 0" "8 8 28000" "8 8 34000" "8 8 42000"}; do
  set -- $v
  CTK_NVCC_EXTRA="-DCTK_FWD_MINB=$1 -DCTK_FWD_UNROLL=$2 -DCTK_FWD_DYNSMEM=$3" python -c "from paper_2602_17892_b200 import build; build.build(force=True)" || exit 1
  echo -n "minb $1 unroll $2 dyn $3: "
  python tools/bench_projectors.py ${CONFS:-c1 c2 c3 c4 c5} | python -c "
import json,sys
print(' '.join('%s %.4f' % (d['config'], d['A']['ms']) for d in map(json.loads, sys.stdin)), end=' | ')"
  python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 solve %.3f ms' % d['ms_per_step'], 'K1 %.4f' % d['kernels']['forward']['mean_ms'])"
done
