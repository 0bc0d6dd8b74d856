#!/bin/bash
# c5 headline: 8 concurrent slices vs 1, and the reference arm.
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r02_bench_c5x8.json 2> gpurun_out/r02_bench_c5x8.err
timeout 600 python bench.py --slices-per-gpu 1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02_bench_c5x1.json 2> gpurun_out/r02_bench_c5x1.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_ref_c5.json 2> gpurun_out/r02_ref_c5.err
for f in gpurun_out/r02_bench_c5x8 gpurun_out/r02_bench_c5x1 gpurun_out/r02_ref_c5; do python - "$f" <<'PY'
import json,sys
f=sys.argv[1]
try:
    d=json.loads(open(f+'.json').read().strip().splitlines()[-1])
except Exception as e:
    print(f, 'FAILED', e); print(open(f+'.err').read()[-2000:]); sys.exit()
keys=['value','ms_per_step','slices_per_s','iters_per_s','rays_executed_per_s','gpu_launches']
print(f, {k:d.get(k) for k in keys}, 'e2e', (d.get('e2e') or {}).get('value'), 'roof', {k:(d.get('roofline') or {}).get(k) for k in ('frac','mean_launch_ms','share_of_step')}, 'clk', d.get('clocks'), 'cpu', (d.get('cpu_baseline') or {}).get('value'))
PY
done
