"""Wall-clock breakdown of one device-resident solve (setup / native loop / rest)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems, _native
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
spec = problems.CONFIGS[name]
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
xt = torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda()
b = A.dgeom.forward(xt)
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
orig_init = gmres._DeviceSolve.__init__
orig_solve = _native.load().ctk_solve
T = {}
def init(self, *a, **k):
    t = time.perf_counter(); orig_init(self, *a, **k); torch.cuda.synchronize(); T['init'] = time.perf_counter() - t
gmres._DeviceSolve.__init__ = init
for _ in range(3): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize()
for _ in range(3):
    t0 = time.perf_counter()
    res = gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
    torch.cuda.synchronize()
    tot = time.perf_counter() - t0
    last = res.records[-1].elapsed
    print(f"{name}: total {tot*1e3:.2f} ms, init {T['init']*1e3:.2f} ms, last iterate done at {last*1e3:.2f} ms (GPU clock from solve start), records {len(res.records)}")
