"""Run N device-resident solves of a BASELINE config (for ncu launch lists)."""
import sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
n = int(sys.argv[2]) if len(sys.argv) > 2 else 1
spec = problems.CONFIGS[name]
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
xt = torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda()
b = A.dgeom.forward(xt)
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
for _ in range(n):
    res = gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize()
print(name, len(res.records), res.records[-1].lambda_used)
