#!/bin/bash
# K2 angle split granularity (CTK_BACK_MINANG: min angles per CTA) x CTA target, c1/c2 solves
run() { w=$1; shift
  ms=$(env "$@" python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})")
  echo "$w $* -> $ms"; }
for w in c1 c2; do
  run $w X=0
  run $w CTK_BACK_MINANG=16
  run $w CTK_BACK_MINANG=8
  run $w CTK_BACK_MINANG=16 CTK_BACK_TARGET=2960
  run $w CTK_BACK_MINANG=8 CTK_BACK_TARGET=2960
  run $w X=0
done
python tools/bench_projectors.py 2>&1 | head -2
CTK_BACK_MINANG=16 python tools/bench_projectors.py 2>&1 | head -2
CTK_BACK_MINANG=8 python tools/bench_projectors.py 2>&1 | head -2
