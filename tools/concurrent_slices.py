"""Batched c5 slices: S solves issued one after another vs from S host threads
at once (each thread gets its own stream pair), aggregate slices/s."""
import sys, threading, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems
name = sys.argv[1] if len(sys.argv) > 1 else 'c5'
S = int(sys.argv[2]) if len(sys.argv) > 2 else 2
spec = problems.CONFIGS[name]
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
bs = []
for s in range(S):
    _, x32 = problems.random_ellipse_phantom_device(spec.N, spec.ellipses, s)
    bs.append(A.dgeom.forward(x32))
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
def solve(b):
    gmres.run_gmres(A, B, b, cfg, keep_on_device=True)
    torch.cuda.synchronize()
for b in bs:
    solve(b)                                   # warm-up (main thread)
threads = [threading.Thread(target=solve, args=(b,)) for b in bs]
for t in threads: t.start()
for t in threads: t.join()                     # warm-up (worker threads)
torch.cuda.synchronize()
t0 = time.perf_counter()
for b in bs:
    solve(b)
t_seq = time.perf_counter() - t0
t0 = time.perf_counter()
threads = [threading.Thread(target=solve, args=(b,)) for b in bs]
for t in threads: t.start()
for t in threads: t.join()
t_con = time.perf_counter() - t0
print(f"{name} x{S}: sequential {t_seq*1e3:.1f} ms ({S/t_seq:.3f} slices/s), "
      f"concurrent {t_con*1e3:.1f} ms ({S/t_con:.3f} slices/s), speedup {t_seq/t_con:.3f}")
