"""Per-iteration reconstruction metrics and stopping rules (host fp64).

Only evaluated when the caller asks for them (``x_true`` given, or a
stopping rule other than "none"); the configs' timed solves use neither.
Semantics: RRE and SSIM as ctkrylov/metrics.py:13-62; DP / NCP / RNS as
ctkrylov/stopping.py:18-67.
"""

from __future__ import annotations

import numpy as np

DEFAULT_DP_TAU = 1.01
DEFAULT_NCP_THRESHOLD = 0.05
DEFAULT_RNS_EPSILON = 1e-4


def rre(x, x_true) -> float:
    x = np.asarray(x, dtype=np.float64).ravel()
    ref = np.asarray(x_true, dtype=np.float64).ravel()
    if x.shape != ref.shape:
        raise ValueError(f"shape mismatch: {x.shape} vs {ref.shape}")
    d = np.linalg.norm(ref)
    if d == 0.0:
        raise ValueError("RRE is undefined for a zero ground truth")
    return float(np.linalg.norm(x - ref) / d)


def ssim(x, x_true, shape, dynamic_range=None) -> float:
    """Mean SSIM over 8x8 Gaussian (sigma 1.5) windows at stride 1."""
    from scipy.signal import fftconvolve

    ny, nx = shape
    if ny < 8 or nx < 8:
        raise ValueError(f"SSIM needs at least 8x8 images, got {shape}")
    a = np.asarray(x, dtype=np.float64).reshape(shape)
    b = np.asarray(x_true, dtype=np.float64).reshape(shape)
    rng = float(b.max() - b.min()) if dynamic_range is None else float(dynamic_range)
    if rng == 0.0:
        raise ValueError("SSIM is undefined for a constant ground truth")
    k1, k2 = (0.01 * rng) ** 2, (0.03 * rng) ** 2
    t = np.arange(8) - 3.5
    g = np.exp(-(t * t) / (2.0 * 1.5 * 1.5))
    win = np.outer(g, g)
    win /= win.sum()

    def local(img):
        return fftconvolve(img, win[::-1, ::-1], mode="valid")

    ma, mb = local(a), local(b)
    va = local(a * a) - ma * ma
    vb = local(b * b) - mb * mb
    cov = local(a * b) - ma * mb
    num = (2 * ma * mb + k1) * (2 * cov + k2)
    den = (ma * ma + mb * mb + k1) * (va + vb + k2)
    return float(np.mean(num / den))


def dp_should_stop(residual_norm, noise_norm, tau=DEFAULT_DP_TAU) -> bool:
    if tau < 1.0:
        raise ValueError(f"DP safety factor must be >= 1, got {tau}")
    if noise_norm < 0.0:
        raise ValueError(f"noise norm must be nonnegative, got {noise_norm}")
    return residual_norm <= tau * noise_norm


def ncp_distance(residual) -> float:
    r = np.asarray(residual, dtype=np.float64)
    if r.size < 8:
        raise ValueError(f"NCP needs a residual of length >= 8, got {r.size}")
    half = r.size // 2
    power = (np.abs(np.fft.rfft(r)) ** 2)[1: half + 1]
    total = power.sum()
    if total == 0.0:
        return 0.0
    return float(np.max(np.abs(np.cumsum(power) / total - np.arange(1, half + 1) / half)))


def ncp_should_stop(residual, threshold=DEFAULT_NCP_THRESHOLD) -> bool:
    return ncp_distance(residual) <= threshold


def rns_should_stop(history, epsilon=DEFAULT_RNS_EPSILON) -> bool:
    if epsilon <= 0.0:
        raise ValueError(f"RNS tolerance must be positive, got {epsilon}")
    if len(history) < 2:
        return False
    prev, cur = history[-2], history[-1]
    if prev == 0.0:
        return True
    return abs(prev - cur) / prev < epsilon
