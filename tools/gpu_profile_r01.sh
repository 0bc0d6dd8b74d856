set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --workload c3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2>&1
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b2.json 2>&1
C2="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$C2 > gpurun_out/plain_c2.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 700 --csv --log-file gpurun_out/launches_c2.csv $C2 > gpurun_out/ncu_c2.log 2>&1
C3="python bench.py --workload c3 --steps 1 --warmup 1 --no-cpu-baseline"
$C3 > gpurun_out/plain_c3.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_forward -c 2 -o gpurun_out/prof_fwd_c3 $C3 > gpurun_out/ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_back -c 2 -o gpurun_out/prof_back_c3 $C3 > gpurun_out/ncu_c3b.log 2>&1
ls -la gpurun_out
