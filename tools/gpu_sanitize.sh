#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the hand-synchronised
# paths (tools/sanitize_solves.py) and the peer-exchange kernels' test.
CS=/usr/local/cuda/bin/compute-sanitizer
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_solves.py > gpurun_out/san/$tool.txt 2>&1
  echo "$tool solves rc=$?" >> gpurun_out/san/summary.txt
  tail -3 gpurun_out/san/$tool.txt >> gpurun_out/san/summary.txt
done
timeout 900 $CS --tool memcheck --error-exitcode 9 python -m pytest tests/test_gpu_exchange.py -q -x > gpurun_out/san/memcheck_exchange.txt 2>&1
echo "memcheck exchange rc=$?" >> gpurun_out/san/summary.txt
tail -3 gpurun_out/san/memcheck_exchange.txt >> gpurun_out/san/summary.txt
timeout 900 $CS --tool synccheck --error-exitcode 9 python -m pytest tests/test_gpu_exchange.py -q -x > gpurun_out/san/synccheck_exchange.txt 2>&1
echo "synccheck exchange rc=$?" >> gpurun_out/san/summary.txt
tail -3 gpurun_out/san/synccheck_exchange.txt >> gpurun_out/san/summary.txt
cat gpurun_out/san/summary.txt
