#!/bin/bash
for ppt in 2 4; do
  CTK_NVCC_EXTRA="-DCTK_BACK_PPT=$ppt" python -m paper_2602_17892_b200.build --force > /dev/null 2>&1 || exit 1
  echo "== ppt $ppt"
  python -m pytest tests/test_gpu_projectors.py -q 2>&1 | tail -1
  python tools/bench_projectors.py c1 c2 c3 c4 c5 | python -c "import sys,json; [print(d['config'], d['B']['ms']) for d in map(json.loads, sys.stdin)]"
  python tools/time_solve.py c1 | tail -1; python tools/time_solve.py c2 | tail -1
done
