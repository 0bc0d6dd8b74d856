"""world_size-2 gloo test of the angle-sharded GMRES driver (CPU).

Each rank owns an interleaved half of the angles and runs
paper_2602_17892_b200.dist.run_gmres_sharded with a host backend whose
projectors are the oracle restricted to the rank's angles; partial images and
dot products go through real torch.distributed all-reduces (gloo).  The
result must equal the single-process reference-algorithm solve.
"""

import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_17892_b200 import dist, gmres, problems

N, NA, D = 24, 16, 35


class HostShardBackend(dist.ShardBackend):
    """Oracle projectors on this rank's angles; gloo all-reduce (test only)."""

    def __init__(self, angle_idx, torch, tdist):
        self.torch, self.tdist = torch, tdist
        angles = np.arange(NA) * np.pi / NA
        self.g = O.Geometry(N, N, 1.0, angles[angle_idx], D, 1.0)
        self.n, self.m_local = self.g.n, self.g.m

    def zeros(self, size):
        return np.zeros(size)

    def from_host(self, arr):
        return np.array(arr, dtype=np.float64)

    def to_host(self, v):
        return np.array(v)

    from_host_f64 = from_host
    to_host_f64 = to_host

    def forward(self, x):
        return O.forward(self.g, x, 1)

    def back_partial(self, u):
        return O.back(self.g, u, 1)

    def allreduce(self, v):
        t = self.torch.from_numpy(v)
        self.tdist.all_reduce(t)

    def norm2(self, v):
        return float(v @ v)

    def scale(self, v, a):
        return v * a

    def add(self, a, b):
        return a + b

    def sub(self, a, b):
        return a - b

    def basis_init(self, L, rows):
        self.W = np.zeros((rows, L))

    def basis_set(self, j, v, scale):
        self.W[j] = v * scale

    def basis_row(self, j):
        return self.W[j]

    def basis_dots(self, k, v, want_norm):
        d = self.W[:k] @ v
        return np.append(d, v @ v) if want_norm else d

    def basis_update(self, k, coef, v):
        return v - np.asarray(coef) @ self.W[:k]

    def basis_combine(self, k, y):
        return np.asarray(y) @ self.W[:k]


def problem():
    angles = np.arange(NA) * np.pi / NA
    g = O.Geometry(N, N, 1.0, angles, D, 1.0)
    x = problems.random_ellipse_phantom(N, 5, 2)
    b, _ = problems.add_noise(O.forward(g, x), 0.02, 3)
    return g, b


def _worker(rank, world, port, method, strategy, out_dir):
    import torch
    import torch.distributed as tdist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    tdist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        idx = dist.angle_shards(NA, world, "interleaved")[rank]
        g, b = problem()
        b_local = b.reshape(NA, D)[idx].ravel()
        be = HostShardBackend(idx, torch, tdist)
        cfg = gmres.SolverConfig(method=method, lambda_strategy=strategy, max_iter=12)
        res = dist.run_gmres_sharded(be, b_local, cfg)
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), x=res.x,
                 lam=[r.lambda_used for r in res.records],
                 dn=[r.data_residual_norm for r in res.records],
                 pn=[r.proj_residual_norm for r in res.records])
    finally:
        tdist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("method,strategy", [("ab-hybrid", "gcv"), ("ba-hybrid", "gcv"),
                                             ("ab", "none")])
def test_sharded_solve_world2_matches_single_process(tmp_path, method, strategy):
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, free_port(), method, strategy, str(tmp_path)), nprocs=2, join=True)
    r0, r1 = (np.load(tmp_path / f"r{r}.npz") for r in (0, 1))
    # every rank holds the same (replicated) answer
    np.testing.assert_array_equal(r0["x"], r1["x"])
    np.testing.assert_array_equal(r0["lam"], r1["lam"])
    g, b = problem()
    ref = O.gmres(lambda v: O.forward(g, v), lambda v: O.back(g, v), b, method, strategy, 12)
    lam = np.array([r["lambda_used"] for r in ref.records])
    dn = np.array([r["data_residual_norm"] for r in ref.records])
    np.testing.assert_allclose(r0["dn"], dn, rtol=1e-9)
    np.testing.assert_allclose(r0["lam"], lam, rtol=1e-9)
    np.testing.assert_allclose(r0["x"], ref.x, rtol=1e-8, atol=1e-10 * np.abs(ref.x).max())


def test_partial_backprojections_sum_to_full_b():
    g, _ = problem()
    u = np.random.default_rng(0).random(g.m)
    full = O.back(g, u)
    parts = dist.angle_shards(NA, 3, "blocks")
    tot = np.zeros(g.n)
    for idx in parts:
        gi = O.Geometry(N, N, 1.0, g.angles[idx], D, 1.0)
        tot += O.back(gi, u.reshape(NA, D)[idx].ravel())
    np.testing.assert_allclose(tot, full, rtol=1e-12, atol=1e-12)
