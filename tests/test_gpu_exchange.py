"""Angle-sharded B with the partial-image sum exchanged over peer memory
(ctk_back_exchange, SURVEY row e).

Only one GPU exists here, so the ranks are emulated in one process on one
device: every rank's buffers live on cuda:0 and connect with raw pointers, and
the three phases run rank by rank in order (all pushes, then all owner
reductions, then all waits) so that no kernel ever spins on work that has not
been issued -- the same kernels a multi-GPU run launches, with the peer
stores landing in the same device's memory.

Bar: every rank's image equals, bitwise, the rank-order fp64 sum of the
per-rank partial images (plain K2 on each rank's angles), and the full B
within the projector bar.
"""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_17892_b200 import ct, dist, problems

pytestmark = pytest.mark.gpu


def run_exchange(torch, N, na, D, nranks, seeds=(1,), mode="interleaved", ny=None, h=1.0, sp=1.0):
    grid = ct.ImageGrid(N, N if ny is None else ny, h)
    angles = np.arange(na) * np.pi / na
    geom = ct.ParallelGeometry(angles, D, sp)
    shards = dist.angle_shards(na, nranks, mode)
    dgs = [ct.DeviceGeometry(grid, ct.ParallelGeometry(angles[idx], D, sp), 0) for idx in shards]
    ex = [dist.PeerExchange(dgs[r], r, nranks) for r in range(nranks)]
    for e in ex:
        e.connect_local(ex)
    full = ct.DeviceGeometry(grid, geom, 0)
    results = []
    for epoch, seed in enumerate(seeds, start=1):
        u = problems.uniform_sinogram(geom.m, seed).reshape(na, D)
        us = [torch.from_numpy(np.ascontiguousarray(u[idx]).ravel().astype(np.float32)).cuda()
              for idx in shards]
        for phase in (1, 2, 4):
            for r in range(nranks):
                ex[r].back(us[r], phases=phase, epoch=epoch)
        torch.cuda.synchronize()
        parts = [dgs[r].back(us[r]).double().cpu().numpy() for r in range(nranks)]
        expect = np.zeros(grid.n)
        for p in parts:
            expect += p
        expect = expect.astype(np.float32)
        ud = torch.from_numpy(u.ravel().astype(np.float32)).cuda()
        whole = full.back(ud).double().cpu().numpy()
        results.append(([e.img.cpu().numpy().copy() for e in ex], expect, whole, u))
    return results, grid, geom


@pytest.mark.parametrize("N,na,D,nranks", [
    (128, 180, 183, 2),      # c1 geometry: angle-split K2 (last-CTA tile reduction)
    (128, 180, 183, 8),      # eight ranks
    (96, 60, 139, 3),        # odd rank count, tiles not a multiple of it
    (300, 40, 425, 2),       # <= 32 angles per rank: unsplit K2 epilogue
    (512, 48, 725, 4),       # 32x32 tiles (4 rows per thread)
])
def test_exchange_equals_rank_ordered_sum(cuda, N, na, D, nranks):
    results, grid, geom = run_exchange(cuda, N, na, D, nranks)
    imgs, expect, whole, _ = results[0]
    for r, img in enumerate(imgs):
        np.testing.assert_array_equal(img, expect, err_msg=f"rank {r}")
    rel = np.linalg.norm(expect - whole) / np.linalg.norm(whole)
    assert rel <= 1e-6, rel


def test_exchange_epochs_and_reference(cuda):
    """Consecutive calls (epochs 1, 2) reuse the flags without a reset; the
    result matches the reference-restated B (oracle) within the bar."""
    results, grid, geom = run_exchange(cuda, 64, 90, 93, 4, seeds=(3, 4), mode="blocks")
    og = O.Geometry(64, 64, 1.0, geom.angles, 93, 1.0)
    for imgs, expect, whole, u in results:
        for img in imgs:
            np.testing.assert_array_equal(img, expect)
        ref = O.back(og, u.ravel().astype(np.float32).astype(np.float64))
        assert np.linalg.norm(imgs[0] - ref) / np.linalg.norm(ref) <= 1e-5


def test_exchange_rejects_bad_setup(cuda):
    grid = ct.ImageGrid(32, 32, 1.0)
    dg = ct.DeviceGeometry(grid, ct.ParallelGeometry(np.arange(8) * np.pi / 8, 45, 1.0), 0)
    with pytest.raises(ValueError):
        dist.PeerExchange(dg, 3, 2)
    with pytest.raises(ValueError):
        dist.PeerExchange(dg, 0, 9)
    ex = dist.PeerExchange(dg, 0, 2)                  # rank 1 never connected
    u = cuda.zeros(dg.m, dtype=cuda.float32, device="cuda")
    with pytest.raises(ValueError):
        ex.back(u)


@pytest.mark.parametrize("nx,ny,h,sp,na,nranks", [(150, 131, 0.8, 1.1, 77, 3), (131, 600, 1.3, 0.9, 50, 4),
                                                  (700, 90, 0.6, 1.0, 96, 8)])
def test_exchange_on_odd_geometries(cuda, nx, ny, h, sp, na, nranks):
    """The peer exchange on non-square images with non-unit spacings (tile
    ownership, edge tiles, windows narrower / wider than a warp), rank counts
    that do not divide the tile count: every rank bitwise the rank-ordered
    sum, and the reference B within the bar."""
    D = int(np.ceil(np.hypot(nx, ny) * h / sp)) + 3
    results, grid, geom = run_exchange(cuda, nx, na, D, nranks, ny=ny, h=h, sp=sp)
    imgs, expect, whole, u = results[0]
    for r, img in enumerate(imgs):
        np.testing.assert_array_equal(img, expect, err_msg=f"rank {r}")
    og = O.Geometry(nx, ny, h, geom.angles, D, sp)
    ref = O.back(og, u.ravel().astype(np.float32).astype(np.float64))
    assert np.linalg.norm(imgs[0] - ref) / np.linalg.norm(ref) <= 1e-5
