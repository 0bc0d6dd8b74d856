#!/bin/bash
# K1 paired-row (FADD2/FFMA2) vs single-row walk: isolated A at c1..c5, in-situ c2/c5.
for pv in 1 0; do
  CTK_NVCC_EXTRA="-DCTK_FWD_PAIRED=$pv" python -c "from paper_2602_17892_b200 import build; build.build(force=True)" || exit 1
  echo -n "paired $pv: "
  python tools/bench_projectors.py | python -c "
import json,sys
print(' '.join('%s %.4f' % (d['config'], d['A']['ms']) for d in map(json.loads, sys.stdin)), end=' | ')"
  for w in c2 c5; do python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w %.3f K1 %.4f' % (d['ms_per_step'], d['kernels']['forward']['mean_ms']), end=' | ')"; done; echo
done
