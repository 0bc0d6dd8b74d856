"""Where the public-API (host buffer) solve spends its wall time vs the
device-resident solve, under bench.py's conditions (L2 flush + barrier)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200 import ct, gmres, problems
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
spec = problems.CONFIGS[name]
grid = ct.ImageGrid(spec.N, spec.N, 1.0); geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
A = ct.forward_ray_driven(grid, geom); B = ct.back_pixel_driven(grid, geom)
xt = torch.from_numpy(problems.random_ellipse_phantom(spec.N, spec.ellipses, 0).astype(np.float32)).cuda()
b = A.dgeom.forward(xt).cpu().numpy().astype(np.float64)
bd = torch.from_numpy(b.astype(np.float32)).cuda()
cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
stream = torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
def run(kind, do_flush):
    ws = []
    for _ in range(6):
        if do_flush:
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
        torch.cuda.synchronize()
        t = time.perf_counter()
        if kind == 'host':
            gmres.run_gmres(A, B, b, cfg, stream=stream)
        else:
            gmres.run_gmres(A, B, bd, cfg, stream=stream, keep_on_device=True)
            stream.synchronize()
        ws.append(time.perf_counter() - t)
    print(f"{name} {kind:6s} flush={do_flush}: " + " ".join(f"{w*1e3:.2f}" for w in ws))
for kind in ('device', 'host'):
    for fl in (False, True):
        run(kind, fl)
