for w in c2 c1; do
python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/x_$w.json 2>/dev/null
CTK_EXP_SKIP_ITER=1 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/y_$w.json 2>/dev/null
for f in x y; do python -c "
import json; d=json.loads(open('gpurun_out/${f}_$w.json').read().strip().splitlines()[-1]); print('$f $w', d['ms_per_step'], {k:v['mean_ms'] for k,v in d['kernels'].items()})"; done; done
