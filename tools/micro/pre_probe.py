import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems, _native
spec = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c1']
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
b = A.dgeom.forward(torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda())
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
for _ in range(5): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
import cProfile, pstats
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter(); s = gmres._NativeSolve(A, B, b, cfg, None, None, None, None, True); t1 = time.perf_counter()
    res = s.run(); torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"init {(t1-t0)*1e3:.3f} ms, run {(t2-t1)*1e3:.3f} ms")
pr = cProfile.Profile(); pr.enable()
for _ in range(20): gmres._NativeSolve(A, B, b, cfg, None, None, None, None, True)
pr.disable(); pstats.Stats(pr).sort_stats('tottime').print_stats(12)
