"""Seeded synthetic inputs for the BASELINE.json configs (c1..c5).

The reference has no random-ellipse phantom (it only ships Shepp-Logan,
ctkrylov/ct.py:99-134), so the recipe below is frozen here:
``default_rng(seed).uniform(lo, hi, size=(E, 6))`` with columns
(cx, cy) in [-N/4, N/4], semi-axes (a, b) in [0.05N, 0.4N], phi in [0, pi),
rho in [0.1, 1.0], evaluated at pixel centres (ctkrylov/ct.py:60-66) with the
rotated membership test of ctkrylov/ct.py:128-133; overlapping densities add.

Geometry for every config is unit pixels and unit-width bins,
``ImageGrid(N, N, 1.0)`` and ``ParallelGeometry(arange(na)*pi/na, D, 1.0)``
(not make_ct_problem, which rescales pixels: ctkrylov/ct.py:325-328).

Values handed to the device are fp32; the fp64 oracle receives
``float64(float32(v))`` so input rounding never counts against parity.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class ConfigSpec:
    name: str
    N: int
    n_angles: int
    det_count: int
    method: str | None = None          # ab-hybrid | ba-hybrid | None (microbench)
    strategy: str | None = None        # gcv | lcurve
    max_iter: int = 0
    noise: float = 0.0
    ellipses: int = 10
    phantom_seed: int = 0
    noise_seed: int = 1
    slices: int = 1

    @property
    def n(self) -> int:
        return self.N * self.N

    @property
    def m(self) -> int:
        return self.n_angles * self.det_count

    def angles(self) -> np.ndarray:
        return np.arange(self.n_angles) * np.pi / self.n_angles


# BASELINE.json "configs".
CONFIGS = {
    "c1": ConfigSpec("c1", 128, 180, 183, "ab-hybrid", "gcv", 50, 0.01, 10),
    "c2": ConfigSpec("c2", 256, 360, 363, "ba-hybrid", "lcurve", 80, 0.02, 10),
    "c3": ConfigSpec("c3", 512, 720, 725),
    "c4": ConfigSpec("c4", 1024, 1440, 1449, "ab-hybrid", "gcv", 100, 0.01, 20),
    "c5": ConfigSpec("c5", 2048, 1800, 2897, "ba-hybrid", "gcv", 60, 0.01, 10, slices=64),
}


def random_ellipse_phantom(N: int, n_ellipses: int, seed: int, pixel_size: float = 1.0) -> np.ndarray:
    """Flattened row-major (N, N) phantom, fp32-representable fp64 values."""
    params = ellipse_params(N, n_ellipses, seed)
    half = 0.5 * N * pixel_size
    xc = -half + (np.arange(N) + 0.5) * pixel_size
    yc = half - (np.arange(N) + 0.5) * pixel_size
    X, Y = np.meshgrid(xc, yc)
    img = np.zeros((N, N))
    for cx, cy, a, b, phi, rho in params:
        c, s = np.cos(phi), np.sin(phi)
        u = ((X - cx) * c + (Y - cy) * s) / a
        v = (-(X - cx) * s + (Y - cy) * c) / b
        img[u * u + v * v <= 1.0] += rho
    return img.ravel().astype(np.float32).astype(np.float64)


def ellipse_params(N: int, n_ellipses: int, seed: int) -> np.ndarray:
    """The recipe's (E, 6) draw: columns cx, cy, a, b, phi, rho."""
    lo = np.array([-0.25 * N, -0.25 * N, 0.05 * N, 0.05 * N, 0.0, 0.1])
    hi = np.array([0.25 * N, 0.25 * N, 0.4 * N, 0.4 * N, np.pi, 1.0])
    return np.random.default_rng(seed).uniform(lo, hi, size=(n_ellipses, 6))


def random_ellipse_phantom_device(N: int, n_ellipses: int, seed: int, pixel_size: float = 1.0,
                                  device: int = 0, stream=None):
    """The same phantom sampled on the GPU (ctk_phantom, row f4): returns
    ``(img64, img32)`` CUDA tensors; ``img64`` is bitwise
    ``random_ellipse_phantom`` before its fp32 rounding, ``img32`` after."""
    from . import ct
    rows = [(rho, a, b, cx, cy, phi) for cx, cy, a, b, phi, rho in ellipse_params(N, n_ellipses, seed)]
    return ct.phantom_device(ct.ImageGrid(N, N, pixel_size), rows, 1.0, device, stream=stream)


def add_noise(b_clean: np.ndarray, level: float, seed: int) -> tuple[np.ndarray, float]:
    """White Gaussian noise scaled to an exact relative level.

    Same contract as ctkrylov/ct.py:267-283: ``||e|| = level * ||b_clean||``
    exactly, deterministic given the seed, level 0 returns a copy.
    """
    if level < 0:
        raise ValueError(f"noise level must be nonnegative, got {level}")
    b_clean = np.asarray(b_clean, dtype=np.float64)
    target = level * float(np.linalg.norm(b_clean))
    if level == 0.0:
        return b_clean.copy(), 0.0
    draw = np.random.default_rng(seed).standard_normal(b_clean.size)
    # (target * g) / ||g||: the reference's evaluation order, so b is bitwise
    # the one the reference would build from the same clean data.
    scaled = (target * draw) / np.linalg.norm(draw)
    return b_clean + scaled, target


def uniform_image(n: int, seed: int = 0) -> np.ndarray:
    """c3 image: default_rng(0).random(n), fp32-representable."""
    return np.random.default_rng(seed).random(n).astype(np.float32).astype(np.float64)


def uniform_sinogram(m: int, seed: int = 1) -> np.ndarray:
    """c3 sinogram: default_rng(1).random(m), fp32-representable."""
    return np.random.default_rng(seed).random(m).astype(np.float32).astype(np.float64)


def slice_seeds(spec: ConfigSpec, s: int) -> tuple[int, int]:
    """(phantom seed, noise seed) of slice s: c5 uses (s, 1000 + s)."""
    if spec.slices > 1:
        return s, 1000 + s
    return spec.phantom_seed, spec.noise_seed
