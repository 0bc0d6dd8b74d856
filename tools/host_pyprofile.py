"""cProfile of the Python around one device-resident solve (c2 by default):
where the ~0.3 ms of set-up / epilogue outside ctk_solve goes."""
import cProfile, pstats, sys
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
spec = problems.CONFIGS[name]
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
xt = torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda()
b = A.dgeom.forward(xt)
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
for _ in range(5):
    gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(20):
    gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats('tottime').print_stats(25)
