#!/bin/bash
# K1 split x resident-CTA bound sweep: isolated c1/c2/c3 applies and the
# in-situ c2 solve (bench.py) per setting.
for mb in ${MINBS:-12 10}; do
  CTK_NVCC_EXTRA="-DCTK_FWD_MINB=$mb" python -c "from paper_2602_17892_b200 import build; build.build(force=True)" || exit 1
  for s in ${SPLITS:-2 3 4 5 6}; do
    echo -n "minb $mb split $s: "
    CTK_FWD_SPLIT=$s python tools/bench_projectors.py ${CONFS:-c1 c2 c3} | python -c "
import json,sys
print(' '.join('%s A %.4f' % (d['config'], d['A']['ms']) for d in map(json.loads, sys.stdin)), end=' | ')"
    CTK_FWD_SPLIT=$s python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c2 solve %.3f ms' % d['ms_per_step'], 'K1 %.4f' % d['kernels']['forward']['mean_ms'])"
  done
done
