#!/bin/bash
# c2 K2 rows-per-thread x CTA target (in-solve and isolated)
run() { w=$1; shift
  ms=$(env "$@" python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})")
  echo "$w $* -> $ms"; }
run c2 X=0
for t in 592 888 1184 1776; do run c2 CTK_BACK_PPT=4 CTK_BACK_TARGET=$t; done
run c2 X=0
