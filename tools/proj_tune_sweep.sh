#!/bin/bash
# c1/c2 solve time vs projector launch shapes (env tuning overrides):
# CTK_FWD_SPLIT (K1 row chunks per ray), CTK_BACK_TARGET (K2 CTA target), CTK_BACK_PPT (K2 rows/thread)
run() {  # $1 = workload, rest = env assignments
  w=$1; shift
  ms=$(env "$@" python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})")
  echo "$w $* -> $ms"
}
run c2 X=0
for s in 1 3 4; do run c2 CTK_FWD_SPLIT=$s; done
for t in 1184 2368 2960 3552; do run c2 CTK_BACK_TARGET=$t; done
run c2 CTK_BACK_PPT=1
run c1 X=0
for s in 2 3 5 6; do run c1 CTK_FWD_SPLIT=$s; done
for t in 1184 2368 2960; do run c1 CTK_BACK_TARGET=$t; done
run c1 CTK_BACK_PPT=2
