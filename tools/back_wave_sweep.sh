#!/bin/bash
# c2 K2 split count around whole waves (6 CTAs/SM x 148 = 888 slots; 128 tiles)
run() { w=$1; shift
  ms=$(env "$@" python bench.py --workload $w --steps 8 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.3f'%d['ms_per_step'], {k:round(v['mean_ms']*1e3,1) for k,v in d['kernels'].items()})")
  echo "$w $* -> $ms"; }
for t in 640 768 896 1776 768 1776; do run c2 CTK_BACK_TARGET=$t; done
