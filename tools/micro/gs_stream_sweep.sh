#!/bin/bash
# Streamed Gram-Schmidt ring depth sweep (build) at c4/c5 (in-situ solves) vs the old paths.
for nbuf in ${NBUFS:-2 3 4}; do
  CTK_NVCC_EXTRA="-DCTK_TS_NBUF=$nbuf" python -c "from paper_2602_17892_b200 import build; build.build(force=True)" || exit 1
  for w in c4 c5; do
    echo -n "nbuf $nbuf $w: "
    python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), {k:round(v['mean_ms'],4) for k,v in d['kernels'].items()})"
  done
done
for w in c4 c5; do echo -n "old paths $w: "; CTK_NO_STREAM_GS=1 python bench.py --workload $w --steps 2 --warmup 3 --no-cpu-baseline --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d['ms_per_step'],2), {k:round(v['mean_ms'],4) for k,v in d['kernels'].items()})"; done
