#!/bin/bash
for t in 0.02 0.0 2.0; do
  CTK_NVCC_EXTRA="-DCTK_ADJ_FAST_MIN=$t" python -m paper_2602_17892_b200.build --force > /dev/null 2>&1 || exit 1
  echo "== fast_min $t"
  python tools/bench_projectors.py --adjoint c4 c5 | python -c "import sys,json; [print(d['config'], d['At']['ms']) for d in map(json.loads, sys.stdin)]"
done
