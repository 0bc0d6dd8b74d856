"""CPU ORACLE for the hybrid AB-/BA-GMRES projector path -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module, and only
as the checker or the timed CPU baseline.  The product package
(``paper_2602_17892_b200``) never imports it.

What it restates (each item cites the reference it follows; paths are
relative to the reference's ``pkg/src``):

* A, Siddon ray-driven forward projector: ``ctkrylov/ct.py:137-201``, in C
  (``ctk_oracle.c``: per-ray trace, CSR canonicalisation, column-ordered row
  sum), bit-identical to the reference's CSR SpMV.
* B, pixel-driven linear-interpolation backprojector:
  ``ctkrylov/ct.py:204-245``, in C, angle-ordered accumulation.
* Arnoldi with MGS + full reorthogonalisation: ``ctkrylov/arnoldi.py:56-82``.
* Projected LS / Tikhonov solves: ``ctkrylov/arnoldi.py:95-130``.
* L-curve / GCV selection on the 200-point grid: ``ctkrylov/regparam.py:28-158``.
* The (hybrid) AB/BA-GMRES driver with restarts and stopping:
  ``ctkrylov/gmres.py:135-241``.
* Problem generation (row f4): ellipse phantoms at pixel centres
  (``ctkrylov/ct.py:60-66,115-134``) and exact-level noise
  (``ctkrylov/ct.py:267-283``), numpy.

Pinning: ``tests/golden/make_golden.py`` runs the unmodified reference (in
the build container, where ``/root/reference`` exists) and stores its outputs
under ``tests/golden/``; ``tests/test_oracle_golden.py`` checks this module
against them.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libctk_oracle.so")
_lib = None


def build() -> str:
    """Compile ctk_oracle.c with strict IEEE flags (idempotent)."""
    src = os.path.join(_HERE, "ctk_oracle.c")
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE, "CC=gcc"])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i32p = ctypes.POINTER(ctypes.c_int32)
        ci, cd = ctypes.c_int, ctypes.c_double
        L.orc_siddon_ray.argtypes = [ci, ci, cd, cd, cd, cd, i64p, dp]
        L.orc_forward.argtypes = [ci, ci, cd, ci, dp, dp, ci, dp, dp, dp, ci]
        L.orc_row_counts.argtypes = [ci, ci, cd, ci, dp, dp, ci, dp, i64p, i64p, ci]
        L.orc_csr_fill.argtypes = [ci, ci, cd, ci, dp, dp, ci, dp, i64p, i32p, dp, ci]
        L.orc_csr_spmv.argtypes = [ctypes.c_int64, i64p, i32p, dp, dp, dp, ci]
        L.orc_back.argtypes = [ci, ci, cd, ci, dp, dp, ci, cd, dp, dp, ci]
        _lib = L
    return _lib


def _dp(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _i64p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def _i32p(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))


@dataclass
class Geometry:
    """Plain container for the reference's ImageGrid + ParallelGeometry.

    cos/sin tables are scalar ``np.cos(theta)`` values, as the reference's
    ``_siddon_ray`` (ctkrylov/ct.py:145) and ``back_pixel_driven``
    (ctkrylov/ct.py:225) evaluate them; offsets follow
    ``ParallelGeometry.bin_offsets`` (ctkrylov/ct.py:93-96).
    """

    nx: int
    ny: int
    h: float
    angles: np.ndarray
    det_count: int
    det_spacing: float
    cos_tab: np.ndarray = field(init=False)
    sin_tab: np.ndarray = field(init=False)
    offsets: np.ndarray = field(init=False)

    def __post_init__(self):
        self.angles = np.asarray(self.angles, dtype=np.float64)
        self.cos_tab = np.array([np.cos(float(t)) for t in self.angles])
        self.sin_tab = np.array([np.sin(float(t)) for t in self.angles])
        j = np.arange(self.det_count, dtype=np.float64)
        self.offsets = (j - 0.5 * (self.det_count - 1)) * self.det_spacing

    @property
    def n(self):
        return self.nx * self.ny

    @property
    def m(self):
        return len(self.angles) * self.det_count

    @property
    def n_angles(self):
        return len(self.angles)


def forward(g: Geometry, x: np.ndarray, nthreads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    assert x.shape == (g.n,)
    y = np.empty(g.m)
    lib().orc_forward(g.nx, g.ny, g.h, g.n_angles, _dp(g.cos_tab), _dp(g.sin_tab),
                      g.det_count, _dp(g.offsets), _dp(x), _dp(y), nthreads)
    return y


def back(g: Geometry, u: np.ndarray, nthreads: int = 0) -> np.ndarray:
    u = np.ascontiguousarray(u, dtype=np.float64)
    assert u.shape == (g.m,)
    out = np.empty(g.n)
    lib().orc_back(g.nx, g.ny, g.h, g.n_angles, _dp(g.cos_tab), _dp(g.sin_tab),
                   g.det_count, g.det_spacing, _dp(u), _dp(out), nthreads)
    return out


def row_counts(g: Geometry, nthreads: int = 0) -> tuple[np.ndarray, np.ndarray]:
    """Per-ray kept-segment counts (raw) and CSR nnz (duplicates merged)."""
    raw = np.empty(g.m, dtype=np.int64)
    nnz = np.empty(g.m, dtype=np.int64)
    lib().orc_row_counts(g.nx, g.ny, g.h, g.n_angles, _dp(g.cos_tab), _dp(g.sin_tab),
                         g.det_count, _dp(g.offsets), _i64p(raw), _i64p(nnz), nthreads)
    return raw, nnz


def siddon_ray(g: Geometry, theta_index: int, offset: float):
    cap = g.nx + g.ny + 8
    pix = np.empty(cap, dtype=np.int64)
    ln = np.empty(cap)
    k = lib().orc_siddon_ray(g.nx, g.ny, g.h, float(g.cos_tab[theta_index]),
                             float(g.sin_tab[theta_index]), float(offset), _i64p(pix), _dp(ln))
    return pix[:k].copy(), ln[:k].copy()


class CsrForward:
    """A assembled once as CSR, applied by SpMV -- the reference's own
    algorithm for A (ctkrylov/ct.py:182-201), used as the CPU baseline."""

    def __init__(self, g: Geometry, nthreads: int = 0):
        self.g = g
        self.nthreads = nthreads
        _, nnz = row_counts(g, nthreads)
        self.indptr = np.zeros(g.m + 1, dtype=np.int64)
        np.cumsum(nnz, out=self.indptr[1:])
        self.nnz = int(self.indptr[-1])
        self.indices = np.empty(self.nnz, dtype=np.int32)
        self.data = np.empty(self.nnz)
        lib().orc_csr_fill(g.nx, g.ny, g.h, g.n_angles, _dp(g.cos_tab), _dp(g.sin_tab),
                           g.det_count, _dp(g.offsets), _i64p(self.indptr),
                           _i32p(self.indices), _dp(self.data), nthreads)

    def __call__(self, x):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.empty(self.g.m)
        lib().orc_csr_spmv(self.g.m, _i64p(self.indptr), _i32p(self.indices),
                           _dp(self.data), _dp(x), _dp(y), self.nthreads)
        return y


# --------------------------------------------------------------------------
# Host fp64 Krylov machinery, restated (ctkrylov/arnoldi.py, regparam.py,
# gmres.py).  Structure differs from the reference; arithmetic order is kept
# wherever it decides the last bit.
# --------------------------------------------------------------------------

class OracleDegenerate(RuntimeError):
    pass


BREAKDOWN_RTOL = 1e-14  # ctkrylov/arnoldi.py:17


def hessenberg(cols, k):
    """(k+1) x k upper Hessenberg from stored columns (ctkrylov/arnoldi.py:47-53)."""
    H = np.zeros((k + 1, k))
    for j, col in enumerate(cols):
        H[: j + 2, j] = col
    return H


def lambda_selection(H, beta, strategy, fixed=None, count=200):
    """ctkrylov/regparam.py:137-158 (and 28-36, 46-60, 63-134), scalar loops."""
    if strategy == "none":
        return 0.0
    if strategy == "fixed":
        return float(fixed)
    u, s, _ = np.linalg.svd(np.asarray(H, dtype=np.float64), full_matrices=False)
    smax = float(s.max(initial=0.0))
    if smax <= 0.0:
        raise OracleDegenerate("zero singular values")
    lo = max(float(s[s > 0].min()) * 1e-4, 1e-12)
    grid = np.geomspace(lo, smax, count)
    c = beta * u[0, :]
    incompat = max(beta * beta - float(c @ c), 0.0)

    def norms(lam):
        den = s * s + lam * lam
        sol_sq = float(np.sum((s * c / den) ** 2))
        res_sq = float(np.sum(((lam * lam / den) * c) ** 2)) + incompat
        return sol_sq, res_sq

    if strategy == "gcv":
        kp1 = u.shape[0]
        vals = np.empty(count)
        for i, lam in enumerate(grid):
            _, res_sq = norms(lam)
            tr = kp1 - float(np.sum(s * s / (s * s + lam * lam)))
            if tr <= 0.0:
                raise OracleDegenerate("trace")
            vals[i] = res_sq / (tr * tr)
        if not np.all(np.isfinite(vals)):
            raise OracleDegenerate("gcv non-finite")
        return float(grid[count - 1 - int(np.argmin(vals[::-1]))])
    if strategy == "lcurve":
        if not np.any(s > 0):
            raise OracleDegenerate("zero")
        xs, ys = [], []
        for lam in grid:
            sol_sq, res_sq = norms(lam)
            xs.append(0.5 * np.log(max(res_sq, 1e-300)))
            ys.append(0.5 * np.log(max(sol_sq, 1e-300)))
        if count < 5:
            raise OracleDegenerate("few points")
        xa, ya = np.array(xs), np.array(ys)
        dx, dy = np.gradient(xa), np.gradient(ya)
        ddx, ddy = np.gradient(dx), np.gradient(dy)
        den = (dx * dx + dy * dy) ** 1.5
        with np.errstate(divide="ignore", invalid="ignore"):
            kap = (dx * ddy - dy * ddx) / den
        fin = np.isfinite(kap)
        if not np.any(fin):
            raise OracleDegenerate("non-finite curvature")
        kap = np.where(fin, kap, -np.inf)
        if np.max(kap) <= 1e-9:
            raise OracleDegenerate("flat")
        return float(grid[count - 1 - int(np.argmax(kap[::-1]))])
    raise ValueError(strategy)


def projected_tikhonov(H, beta, lam):
    """ctkrylov/arnoldi.py:95-130: (y, ||H y - beta e1||)."""
    kp1, k = H.shape
    if lam == 0.0:
        rhs = np.zeros(kp1)
        rhs[0] = beta
        y = np.linalg.lstsq(H, rhs, rcond=None)[0]
        return y, float(np.linalg.norm(H @ y - rhs))
    stacked = np.vstack([H, lam * np.eye(k)])
    rhs = np.zeros(kp1 + k)
    rhs[0] = beta
    y = np.linalg.lstsq(stacked, rhs, rcond=None)[0]
    e1 = np.zeros(kp1)
    e1[0] = beta
    return y, float(np.linalg.norm(H @ y - e1))


@dataclass
class OracleResult:
    x: np.ndarray
    records: list
    stop_reason: str
    cycles: int


def gmres(A, B, b, method, strategy="none", max_iter=100, lambda_value=None,
          reorthogonalize=True, restart_period=0, x0=None, stopping_rule="none",
          noise_norm=None, dp_tau=1.01, rns_epsilon=1e-4, ncp_threshold=0.05, on_step=None):
    """(Hybrid) AB-/BA-GMRES, ctkrylov/gmres.py:135-241.

    A: R^n -> R^m and B: R^m -> R^n are callables on fp64 vectors.
    Records are dicts with the IterationRecord fields (ctkrylov/gmres.py:95-106).
    on_step(k, H, beta): optional test hook, called with each iteration's
    (k+1) x k Hessenberg before its lambda selection.
    """
    b = np.asarray(b, dtype=np.float64)
    ab = method.startswith("ab")
    hybrid = method.endswith("-hybrid")
    n = len(B(np.zeros(b.size)))
    x = np.zeros(n) if x0 is None else np.asarray(x0, dtype=np.float64).copy()
    M = (lambda v: A(B(v))) if ab else (lambda v: B(A(v)))
    K = max_iter
    p = restart_period if restart_period > 0 else K
    records, history = [], []
    stop, cycles, prev_lam = None, 0, 0.0
    while stop is None and len(records) < K:
        d0 = b - A(x)
        r0 = d0 if ab else B(d0)
        if np.linalg.norm(r0) == 0.0:
            stop = "breakdown"
            if not records:
                records.append(dict(k=0, lambda_used=0.0, residual_norm=0.0,
                                    data_residual_norm=float(np.linalg.norm(d0)),
                                    proj_residual_norm=0.0,
                                    solution_norm=float(np.linalg.norm(x)),
                                    lambda_warning=False))
            break
        cycles += 1
        beta = float(np.linalg.norm(r0))
        basis = [r0 / beta]
        cols = []
        xc = x
        for _ in range(min(p, K - len(records))):
            # --- Arnoldi step, ctkrylov/arnoldi.py:64-82
            k = len(cols)
            q = M(basis[k])
            qn = np.linalg.norm(q)
            h = np.empty(k + 2)
            for i in range(k + 1):
                h[i] = basis[i] @ q
                q = q - h[i] * basis[i]
            if reorthogonalize:
                for i in range(k + 1):
                    cc = basis[i] @ q
                    h[i] += cc
                    q = q - cc * basis[i]
            h[k + 1] = np.linalg.norm(q)
            cols.append(h)
            k += 1
            broke = h[k] <= BREAKDOWN_RTOL * qn
            if not broke:
                basis.append(q / h[k])
            H = hessenberg(cols, k)
            if on_step is not None:
                on_step(k, H, beta)
            warn = False
            if hybrid:
                try:
                    lam = lambda_selection(H, beta, strategy, lambda_value)
                except OracleDegenerate:
                    lam, warn = prev_lam, True
            else:
                lam = 0.0
            prev_lam = lam
            y, pres = projected_tikhonov(H, beta, lam)
            upd = np.column_stack(basis[:k]) @ y
            xk = xc + (B(upd) if ab else upd)
            dres = b - A(xk)
            dn = float(np.linalg.norm(dres))
            records.append(dict(k=len(records) + 1, lambda_used=float(lam),
                                residual_norm=dn if ab else pres, data_residual_norm=dn,
                                proj_residual_norm=pres,
                                solution_norm=float(np.linalg.norm(xk)),
                                lambda_warning=warn))
            history.append(dn)
            x = xk
            if stopping_rule == "dp" and dn <= dp_tau * noise_norm:
                stop = "dp"
            elif stopping_rule == "rns" and len(history) >= 2 and (
                    history[-2] == 0.0 or abs(history[-2] - history[-1]) / history[-2] < rns_epsilon):
                stop = "rns"
            elif stopping_rule == "ncp":
                spec = np.abs(np.fft.rfft(dres)) ** 2
                qh = dres.size // 2
                pw = spec[1:qh + 1]
                tot = pw.sum()
                dist = 0.0 if tot == 0.0 else float(np.max(np.abs(
                    np.cumsum(pw) / tot - np.arange(1, qh + 1) / qh)))
                if dist <= ncp_threshold:
                    stop = "ncp"
            if broke and stop is None:
                stop = "breakdown"
            if stop is not None:
                break
    return OracleResult(x=x, records=records, stop_reason=stop or "maxiter",
                        cycles=max(cycles, 1))


# ---- problem generation (row f4) -------------------------------------------

def phantom(nx: int, ny: int, h: float, rows, scale: float = 1.0) -> np.ndarray:
    """Ellipse phantom at pixel centres (ctkrylov/ct.py:60-66, 115-134):
    rows = (value, a, b, x0, y0, phi_radians); (X, Y) = centre / scale;
    value_e added, in order, where u^2 + v^2 <= 1."""
    xmin = -(0.5 * nx * h)
    ymax = 0.5 * ny * h
    X, Y = np.meshgrid(xmin + (np.arange(nx) + 0.5) * h, ymax - (np.arange(ny) + 0.5) * h)
    X = X / scale
    Y = Y / scale
    img = np.zeros((ny, nx))
    for value, a, b, x0, y0, phi in rows:
        c, s = np.cos(phi), np.sin(phi)
        u = ((X - x0) * c + (Y - y0) * s) / a
        v = (-(X - x0) * s + (Y - y0) * c) / b
        img[u * u + v * v <= 1.0] += value
    return img.ravel()


def shepp_logan_rows():
    """Modified Shepp-Logan (value, a, b, x0, y0, phi_radians) on [-1, 1]^2."""
    tab = ((1.0, 0.69, 0.92, 0.0, 0.0, 0.0), (-0.8, 0.6624, 0.8740, 0.0, -0.0184, 0.0),
           (-0.2, 0.1100, 0.3100, 0.22, 0.0, -18.0), (-0.2, 0.1600, 0.4100, -0.22, 0.0, 18.0),
           (0.1, 0.2100, 0.2500, 0.0, 0.35, 0.0), (0.1, 0.0460, 0.0460, 0.0, 0.1, 0.0),
           (0.1, 0.0460, 0.0460, 0.0, -0.1, 0.0), (0.1, 0.0460, 0.0230, -0.08, -0.605, 0.0),
           (0.1, 0.0230, 0.0230, 0.0, -0.606, 0.0), (0.1, 0.0230, 0.0460, 0.06, -0.605, 0.0))
    return [(v, a, b, x0, y0, np.deg2rad(p)) for v, a, b, x0, y0, p in tab]


def add_noise(b_clean: np.ndarray, level: float, seed: int):
    """(b_clean + e, ||e||) with ||e|| = level ||b_clean|| (ct.py:267-283)."""
    b_clean = np.asarray(b_clean, dtype=np.float64)
    nn = level * float(np.linalg.norm(b_clean))
    if level == 0.0:
        return b_clean.copy(), 0.0
    g = np.random.default_rng(seed).standard_normal(b_clean.size)
    return b_clean + nn * g / np.linalg.norm(g), nn
