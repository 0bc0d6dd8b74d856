"""Workload for compute-sanitizer (memcheck / racecheck / synccheck).

Exercises every hand-synchronised path of libctk once:
  * c1 hybrid AB-GMRES + GCV, 50 iterations: K2 split tickets, K2 epilogue
    staging, K1 DSMEM clusters (row split), SMEM Gram-Schmidt (TMA 3-D box),
    batched iterate norms;
  * c2 hybrid BA-GMRES + L-curve, 80 iterations: K1 -> K2 chaining counters,
    SMEM Gram-Schmidt staging for K1;
  * standalone B / K7 adjoint over full and partial angle ranges (shared
    work buffer), c3 A + B;
  * a streamed Gram-Schmidt step (L = 2.1M, 2-D TMA ring).
Prints one line per item; exits non-zero on an exception.
"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2602_17892_b200 import arnoldi, ct, gmres, problems


def ops(name):
    spec = problems.CONFIGS[name]
    grid = ct.ImageGrid(spec.N, spec.N, 1.0)
    geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    return spec, ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom)


def solve(name, iters=None):
    spec, A, B = ops(name)
    xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
    b, _ = problems.add_noise(A.apply(xt), spec.noise, spec.noise_seed)
    cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy,
                             max_iter=iters or spec.max_iter)
    res = gmres.run_gmres(A, B, b, cfg)
    print(f"{name}: {len(res.records)} iterations, stop {res.stop_reason}, "
          f"final data residual {res.records[-1].data_residual_norm:.6g}", flush=True)


def ranges():
    spec, A, B = ops("c1")
    dg = A.dgeom
    D = spec.det_count
    u = torch.from_numpy(problems.uniform_sinogram(dg.m, 3).astype(np.float32)).cuda()
    for a0, a1 in ((0, 180), (0, 90), (3, 19), (0, 180)):
        dg.back(u[a0 * D:a1 * D].contiguous(), a0=a0, a1=a1)
        dg.adjoint(u[a0 * D:a1 * D].contiguous(), a0=a0, a1=a1)
    torch.cuda.synchronize()
    spec, A, B = ops("c3")
    x = torch.from_numpy(problems.uniform_image(A.dgeom.n, 0).astype(np.float32)).cuda()
    A.dgeom.back(A.dgeom.forward(x))
    torch.cuda.synchronize()
    print("ranges + c3 applies ok", flush=True)


def streamed_gs():
    L, k = 2_097_152, 12
    rng = np.random.default_rng(0)
    basis = arnoldi.DeviceBasis(L, k + 2, torch.device("cuda", 0), torch)
    v = torch.from_numpy(rng.standard_normal(L).astype(np.float32)).cuda()
    basis.row(0).copy_(v / v.norm())
    st = torch.cuda.current_stream()
    h = torch.zeros(k + 2, dtype=torch.float64, device="cuda")
    stat = torch.zeros(4, dtype=torch.float64, device="cuda")
    for j in range(k):
        q = torch.from_numpy(rng.standard_normal(L).astype(np.float32)).cuda()
        basis.gs_step(j, q, 2, h, stat, st)
    torch.cuda.synchronize()
    print("streamed GS ok", flush=True)


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "ranges", "gs"]
    if "c1" in which:
        solve("c1")
    if "c2" in which:
        solve("c2")
    if "ranges" in which:
        ranges()
    if "gs" in which:
        streamed_gs()
