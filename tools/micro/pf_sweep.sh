#!/bin/bash
# forward L1-prefetch distance sweep (rebuilds libctk per variant)
for pf in none 4 8 16; do
  if [ $pf = none ]; then X=""; else X="-DCTK_FWD_PREFETCH=$pf"; fi
  CTK_NVCC_EXTRA="$X" python -m paper_2602_17892_b200.build --force > /dev/null || exit 1
  echo "== prefetch $pf"
  python tools/micro/deg_probe.py 2>&1 | grep "shift 0.0 "
  python tools/bench_projectors.py c4 c5 | cut -c1-200
  python tools/time_solve.py c2 | tail -1
done
