#!/bin/bash
# SMEM Gram-Schmidt CTA-count sweep at c1 (AB, L = 32,940) and c2 (BA, L = 65,536).
for g in ${GS:-148 96 64 48 32}; do
  for w in c1 c2; do
    echo -n "gs_ctas $g $w: "
    CTK_GS_CTAS=$g python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],3), {k:round(v['mean_ms'],4) for k,v in d['kernels'].items()})"
  done
done
