"""Isolated A / B apply timings at every BASELINE config size (CUDA events,
L2 flushed before each timed apply).  Prints one JSON line per config."""
import json, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, problems
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs']
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
flags = [a for a in sys.argv[1:] if a.startswith('--')]
names = [a for a in sys.argv[1:] if not a.startswith('--')] or ['c1', 'c2', 'c3', 'c4', 'c5']
for name in names:
    spec = problems.CONFIGS[name]
    dg = ct.DeviceGeometry(ct.ImageGrid(spec.N, spec.N, 1.0),
                           ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0), 0)
    raw, nnz = dg.count_segments()
    x = torch.from_numpy(problems.uniform_image(dg.n, 0).astype(np.float32)).cuda()
    u = torch.from_numpy(problems.uniform_sinogram(dg.m, 1).astype(np.float32)).cuda()
    y = torch.empty(dg.m, device='cuda'); xo = torch.empty(dg.n, device='cuda')
    res = {}
    kinds = [('A', lambda: dg.forward(x, out=y)), ('B', lambda: dg.back(u, out=xo))]
    if '--adjoint' in flags:
        kinds.append(('At', lambda: dg.adjoint(u, out=xo)))
    for kind, fn in kinds:
        for _ in range(3): fn()
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); fn(); e1.record(); e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        by = 4 * nnz + 4 * dg.m if kind in ('A', 'At') else 8 * dg.n * dg.n_angles + 4 * dg.n
        res[kind] = {'ms': round(ms, 4), 'GBps': round(by / ms / 1e6, 1), 'frac': round(by / ms / 1e6 / peak, 3),
                     'rays_per_s': round(dg.m / ms * 1e3, -6)}
    print(json.dumps({'config': name, 'nnz': nnz, 'segments': raw, **res}), flush=True)
