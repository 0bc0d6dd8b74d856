import sys; sys.path.insert(0, '.')
import numpy as np
sys.path.insert(0, 'tests')
import test_gpu_large_solves as T
from paper_2602_17892_b200 import ct, gmres, problems
spec = problems.CONFIGS["c4"]
fx = np.load("tests/golden/c4_solve.npz")
b = T.rebuild_b(spec, fx)
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A, B = ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom)
for path in (0, 1):
    if path: 
        import os; os.environ["CTK_NO_GRAM_GS"] = "1"
    res = gmres.run_gmres(A, B, b, gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=100))
    rec = lambda f: np.array([getattr(r, f) for r in res.records])
    for f in ("lambda_used", "data_residual_norm", "proj_residual_norm", "solution_norm"):
        e = np.abs(rec(f) / fx[f"rec/{f}"] - 1)
        print(path, f, "max", f"{e.max():.2e}", "at", int(e.argmax())+1, "first10", np.array2string(e[:10], precision=1), "last", f"{e[-1]:.2e}")
    x_ref = fx["x_q"].astype(np.float64) * float(fx["x_scale"])
    print(path, "x", np.linalg.norm(res.x - x_ref) / np.linalg.norm(x_ref))
    break
