"""The angle-sharded native path on the B200 (SURVEY row e).

Only one GPU is available to the test runs, so:
* the native sharded driver (libctk's C++ driver with its own NCCL
  communicator, ``run_gmres(..., comm=)``) runs at world size 1 -- every
  sharded code path (B summed through the communicator, AB's measurement-space
  dots summed between the Gram-Schmidt launches, residual norms summed at the
  end, one stream for all collectives) executes, NCCL included -- and must
  match the single-GPU solve and the reference's records;
* the peer-memory exchange is checked across TWO PROCESSES on the one GPU
  through real CUDA IPC mappings, its three phases separated by host
  barriers so that no kernel ever waits on another process's running kernel
  (every flag a wait needs is already set when it launches);
* the multi-rank sharding logic itself runs on the CPU with world_size-2
  gloo (tests/test_dist_gloo.py).
"""

import os

import numpy as np
import pytest

from paper_2602_17892_b200 import ct, dist, gmres, problems

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def full_ops(spec):
    grid = ct.ImageGrid(spec.N, spec.N, 1.0)
    geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    return grid, geom


def test_native_comm_one_rank(cuda):
    torch = cuda
    spec = problems.CONFIGS["c1"]
    grid, geom = full_ops(spec)
    A, B = dist.sharded_projectors(grid, geom, np.arange(spec.n_angles))
    comm = dist.NativeComm(A.dgeom)
    assert comm.world == 1 and comm.rank == 0
    v = torch.arange(10, dtype=torch.float64, device="cuda")
    comm.allreduce(v)
    torch.cuda.synchronize()
    assert torch.equal(v, torch.arange(10, dtype=torch.float64, device="cuda"))
    u = torch.from_numpy(problems.uniform_sinogram(A.dgeom.m, 4).astype(np.float32)).cuda()
    got = comm.back(u)
    assert torch.equal(got, A.dgeom.back(u))
    comm.close()


@pytest.mark.parametrize("name,method,strategy", [("c1", "ab-hybrid", "gcv"),
                                                  ("c2", "ba-hybrid", "gcv"),
                                                  ("c1", "ab", "none")])
def test_native_sharded_solve_one_rank_matches_single_gpu(cuda, golden, name, method, strategy):
    spec = problems.CONFIGS[name]
    grid, geom = full_ops(spec)
    z = golden(name)
    b, _ = problems.add_noise(z["Ax_true"], spec.noise, spec.noise_seed)
    b = b.astype(np.float32).astype(np.float64)
    K = 40
    cfg = gmres.SolverConfig(method=method, lambda_strategy=strategy, max_iter=K)
    # interleaved shard of one rank = every angle, through the sharded code path
    idx = dist.angle_shards(spec.n_angles, 1)[0]
    A, B = dist.sharded_projectors(grid, geom, idx)
    comm = dist.NativeComm(A.dgeom)
    res = gmres.run_gmres(A, B, dist.local_rows(b, spec.det_count, idx), cfg, comm=comm)
    ref = gmres.run_gmres(ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom),
                          b, cfg)
    comm.close()
    assert len(res.records) == len(ref.records) == K
    f = lambda r, k: np.array([getattr(x, k) for x in r.records])  # noqa: E731
    if strategy != "none":
        assert np.all(np.abs(f(res, "lambda_used") / f(ref, "lambda_used") - 1) <= 0.01)
    for k in ("data_residual_norm", "proj_residual_norm", "solution_norm"):
        np.testing.assert_allclose(f(res, k), f(ref, k), rtol=1e-4, err_msg=k)
    assert rel(res.x, ref.x) <= 1e-4


def _ipc_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as tdist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    spec = problems.CONFIGS["c1"]
    grid, geom = full_ops(spec)
    idx = dist.angle_shards(spec.n_angles, world)[rank]
    A, _ = dist.sharded_projectors(grid, geom, idx)
    dg = A.dgeom
    ex = dist.PeerExchange(dg, rank, world)
    handles = [None] * world
    tdist.all_gather_object(handles, ex.export())
    ex.connect_ipc(handles)                       # real CUDA IPC mappings across processes
    u_full = problems.uniform_sinogram(spec.m, 9)
    u = torch.from_numpy(dist.local_rows(u_full, spec.det_count, idx).astype(np.float32)).cuda()
    for epoch in (1, 2):
        for phase in (1, 2, 4):                   # push | owner reduce | wait: never concurrent
            ex.back(u, phases=phase, epoch=epoch)
            torch.cuda.synchronize()
            tdist.barrier()
    flag = __import__("ctypes").c_int(-1)
    ex._native.check(ex.lib.ctk_xchg_status(ex.handle, __import__("ctypes").byref(flag)))
    np.save(os.path.join(out_dir, f"img{rank}.npy"), ex.img.cpu().numpy())
    np.save(os.path.join(out_dir, f"status{rank}.npy"), np.array([flag.value]))
    tdist.barrier()
    del ex
    tdist.destroy_process_group()


def test_peer_exchange_two_processes_cuda_ipc(cuda, tmp_path):
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_ipc_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    img0, img1 = (np.load(tmp_path / f"img{r}.npy") for r in (0, 1))
    assert np.array_equal(img0, img1)                 # bitwise the same on every rank
    assert all(int(np.load(tmp_path / f"status{r}.npy")[0]) == 0 for r in (0, 1))
    spec = problems.CONFIGS["c1"]
    grid, geom = full_ops(spec)
    dg = ct.DeviceGeometry(grid, geom, 0)
    torch = cuda
    u = torch.from_numpy(problems.uniform_sinogram(spec.m, 9).astype(np.float32)).cuda()
    full = dg.back(u).cpu().numpy()
    assert rel(img0, full) < 1e-6


@pytest.mark.parametrize("nx,ny,h,sp,na,method", [(150, 131, 0.8, 1.1, 77, "ab-hybrid"),
                                                  (131, 300, 1.3, 0.9, 50, "ba-hybrid"),
                                                  (400, 420, 1.0, 1.0, 381, "ab-hybrid")])
def test_native_sharded_solve_on_odd_geometries(cuda, nx, ny, h, sp, na, method):
    """The sharded driver (libctk's NCCL communicator, multi-kernel CGS2 with
    its dots summed between launches, B through the communicator) at world
    size 1 on non-square images with non-unit spacings and an angle count that
    is not a multiple of 4, including streamed-length measurement vectors:
    same records as the single-GPU solve."""
    from oracle import oracle as O
    D = int(np.ceil(np.hypot(nx, ny) * h / sp)) + 3
    grid = ct.ImageGrid(nx, ny, h)
    geom = ct.ParallelGeometry(np.arange(na) * np.pi / na, D, sp)
    og = O.Geometry(nx, ny, h, geom.angles, D, sp)
    rng = np.random.default_rng(nx)
    b = O.forward(og, rng.random(nx * ny).astype(np.float32).astype(np.float64))
    b = (b * (1 + 0.02 * rng.standard_normal(b.size))).astype(np.float32).astype(np.float64)
    K = 14
    cfg = gmres.SolverConfig(method=method, lambda_strategy="gcv", max_iter=K)
    idx = dist.angle_shards(na, 1)[0]
    A, B = dist.sharded_projectors(grid, geom, idx)
    comm = dist.NativeComm(A.dgeom)
    res = gmres.run_gmres(A, B, dist.local_rows(b, D, idx), cfg, comm=comm)
    ref = gmres.run_gmres(ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom),
                          b, cfg)
    comm.close()
    assert len(res.records) == len(ref.records) == K
    f = lambda r, k: np.array([getattr(x, k) for x in r.records])  # noqa: E731
    assert np.all(np.abs(f(res, "lambda_used") / f(ref, "lambda_used") - 1) <= 0.01)
    for k in ("data_residual_norm", "proj_residual_norm", "solution_norm"):
        np.testing.assert_allclose(f(res, k), f(ref, k), rtol=1e-4, err_msg=k)
    assert rel(res.x, ref.x) <= 1e-4
