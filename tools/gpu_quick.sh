#!/bin/bash
# quick GPU check: gpu tests + c3 microbench + c2 solve bench
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --workload c3 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b3.json 2>gpurun_out/b3.err || tail -5 gpurun_out/b3.err
python bench.py --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/b2.json 2>gpurun_out/b2.err || tail -5 gpurun_out/b2.err
for f in gpurun_out/b3.json gpurun_out/b2.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], "value %.3e" % d["value"], "ms/step %.3f" % d["ms_per_step"], "it/s", d.get("iters_per_s"), "roof", d["roofline"]["frac"], {k:(v["mean_ms"], v.get("gbs")) for k,v in d["kernels"].items()})
PY
done
