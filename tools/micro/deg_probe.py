import sys; sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, problems
for name in ('c1', 'c2', 'c3'):
    spec = problems.CONFIGS[name]
    for shift in (0.0, 1e-3):
        geom = ct.ParallelGeometry(spec.angles() + shift, spec.det_count, 1.0)
        dg = ct.DeviceGeometry(ct.ImageGrid(spec.N, spec.N, 1.0), geom, 0)
        x = torch.rand(dg.n, device='cuda'); y = torch.empty(dg.m, device='cuda')
        for _ in range(5): dg.forward(x, out=y)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): dg.forward(x, out=y)
        e1.record(); torch.cuda.synchronize()
        print(name, 'shift', shift, 'degenerate angles', dg.n_degenerate if hasattr(dg, 'n_degenerate') else '?', '%.1f us' % (e0.elapsed_time(e1) / 50 * 1e3))
