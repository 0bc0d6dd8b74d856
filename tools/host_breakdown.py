"""Wall-clock split of one device-resident solve: Python setup, the ctk_solve
call, and the Python epilogue."""
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
lib = _native.load()
T = {}
class Proxy:
    def __init__(self, lib): self._lib = lib
    def __getattr__(self, n):
        f = getattr(self._lib, n)
        if n != 'ctk_solve': return f
        def g(*a):
            t = time.perf_counter(); r = f(*a); T['solve_call'] = time.perf_counter() - t; T['call_end'] = time.perf_counter(); return r
        return g
orig_load = _native.load
_native.load = lambda: Proxy(orig_load())
for _ in range(5): gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
for _ in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    pre = T['call_end'] - T['solve_call'] - t0
    print(f"{name}: total {(t1-t0)*1e3:.2f} ms = pre {pre*1e3:.2f} + ctk_solve {T['solve_call']*1e3:.2f} + post {(t1-T['call_end'])*1e3:.2f}; last record {res.records[-1].elapsed*1e3:.2f} ms")
