"""Host-side profile of the device-resident c2 solve (cProfile, main thread)."""
import cProfile, pstats, sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems
spec = problems.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else 'c2']
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
xt = torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda()
b = A.dgeom.forward(xt)
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
for _ in range(3): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize(); print('solve ms', (time.perf_counter() - t) / 5 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(3): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(18)
# time the main thread spends blocked on GPU events vs total
import torch.cuda
orig = torch.cuda.Event.synchronize
acc = {'t': 0.0, 'n': 0}
def timed(self):
    t0 = time.perf_counter(); orig(self); acc['t'] += time.perf_counter() - t0; acc['n'] += 1
torch.cuda.Event.synchronize = timed
t = time.perf_counter()
for _ in range(5): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize(); tot = (time.perf_counter() - t) / 5
print('solve ms %.2f, blocked on events ms %.2f (%d waits/solve)' % (tot * 1e3, acc['t'] / 5 * 1e3, acc['n'] / 5))
# GPU-only: just the Arnoldi chain via the native step, back to back
from paper_2602_17892_b200 import _native
_native.profile_begin()
for _ in range(3): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
torch.cuda.synchronize()
print({k: (n // 3, round(m * 1e3, 1), round(t / 3, 2)) for k, (n, m, t) in _native.profile_end().items()})
