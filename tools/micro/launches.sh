#!/bin/bash
W=${1:-c2}
python tools/one_solve.py $W 2 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv python tools/one_solve.py $W 2 > /dev/null 2>&1
python tools/ncu_launch_summary.py gpurun_out/launches_$W.csv "$W two solves"
