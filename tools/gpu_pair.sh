#!/bin/bash
for t in 2 1 0; do echo "CTK_FWD_PAIR=$t"; CTK_FWD_PAIR=$t timeout 300 python tools/bench_projectors.py c2 c3 c4 c5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print(d['config'], 'A', d['A']['ms'])"; done
