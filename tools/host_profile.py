"""Host-side cost of one public-API solve (numpy b in, numpy x out): wall
times and a cProfile of the Python around libctk's ctk_solve."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
spec = problems.CONFIGS[name]
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
xt = torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda()
b = A.dgeom.forward(xt).cpu().numpy().astype(np.float64)
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
for _ in range(3):
    gmres.run_gmres(A, B, b, cfg)
for _ in range(3):
    t = time.perf_counter(); res = gmres.run_gmres(A, B, b, cfg); w = time.perf_counter() - t
    print(f"{name}: host-buffer solve {w*1e3:.2f} ms; GPU clock at last record {res.records[-1].elapsed*1e3:.2f} ms")
pr = cProfile.Profile()
pr.enable(); gmres.run_gmres(A, B, b, cfg); pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
