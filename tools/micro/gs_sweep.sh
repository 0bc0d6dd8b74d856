#!/bin/bash
# Fused CGS2 (c4-size Krylov vectors) CTAs-per-SM sweep: in-situ c4 solve.
for m in ${MULTS:-1 2 4}; do
  echo -n "per_sm $m: "
  CTK_FUSED_PER_SM=$m python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 solve %.2f ms' % d['ms_per_step'], {k: round(v['mean_ms'],4) for k, v in d['kernels'].items()})"
done
