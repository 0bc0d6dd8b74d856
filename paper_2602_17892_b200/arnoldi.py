"""Arnoldi process: device-resident basis (K3) + host fp64 projected solves.

Reference: ctkrylov/arnoldi.py.  The reference keeps a Python list of fp64
basis vectors and runs MGS plus a full reorthogonalisation pass
(arnoldi.py:56-82).  Here the basis is one fp32 HBM buffer ``W[K+1][ld]``
and each step's orthogonalisation is libctk's fused CGS2 (ctk_cgs2_step):
h1 = W^T q, q1 = q - W h1, h2 = W^T q1, q2 = q1 - W h2, h = h1 + h2 --
equal to MGS+reorth in exact arithmetic, with fp64 accumulation and
deterministic reductions.  Only the (k+2)-entry Hessenberg column and two
scalars cross to the host per step.

The projected least-squares / Tikhonov problems (arnoldi.py:95-130) stay on
the host in fp64.  They are solved through the thin SVD already computed for
lambda selection: y = V diag(s / (s^2 + lam^2)) U^T (beta e1), the normal-
equation solution of the reference's stacked lstsq, and for lam == 0 the
minimum-norm lstsq solution with numpy's default rcond.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native
from .regparam import svd_of_hessenberg

BREAKDOWN_RTOL = 1e-14   # ctkrylov/arnoldi.py:17


class Breakdown(Exception):
    """Happy breakdown: the Krylov subspace became invariant at step k."""

    def __init__(self, k: int):
        super().__init__(f"Arnoldi breakdown at step {k}: Krylov subspace is invariant")
        self.k = k


@dataclass(frozen=True)
class ProjectedSolution:
    y: np.ndarray
    proj_residual_norm: float
    lambda_used: float
    rank_deficient: bool = False


def hessenberg_from_columns(cols, k: int) -> np.ndarray:
    """(k+1) x k upper Hessenberg from stored columns (arnoldi.py:47-53)."""
    H = np.zeros((k + 1, k))
    for j, col in enumerate(cols[:k]):
        H[: j + 2, j] = col[: j + 2]
    return H


def solve_projected_tikhonov(hess: np.ndarray, beta: float, lam: float,
                             svd=None) -> ProjectedSolution:
    """min ||H y - beta e1||^2 + lam^2 ||y||^2; proj_residual_norm is the
    unregularised residual of that y (arnoldi.py:110-130)."""
    if lam < 0:
        raise ValueError(f"regularization parameter must be nonnegative, got {lam}")
    H = np.asarray(hess, dtype=np.float64)
    kp1, k = H.shape
    s, u, v = svd if svd is not None else svd_of_hessenberg(H)
    c = beta * u[0, :]
    rank_def = False
    if lam == 0.0:
        cutoff = np.finfo(np.float64).eps * max(kp1, k) * (s[0] if s.size else 0.0)
        keep = s > cutoff
        coef = np.zeros_like(s)
        coef[keep] = c[keep] / s[keep]
        rank_def = int(np.count_nonzero(keep)) < k
    else:
        coef = s * c / (s * s + lam * lam)
    y = v @ coef
    e1 = np.zeros(kp1)
    e1[0] = beta
    res = float(np.linalg.norm(H @ y - e1))
    return ProjectedSolution(y=y, proj_residual_norm=res, lambda_used=float(lam),
                             rank_deficient=rank_def)


def solve_projected_ls(hess: np.ndarray, beta: float, svd=None) -> ProjectedSolution:
    return solve_projected_tikhonov(hess, beta, 0.0, svd=svd)


class DeviceBasis:
    """Krylov basis W[rows][ld] (fp32, HBM-resident) plus K3/K4 launchers.

    ``L`` is the vector length (m for AB, n for BA); ``ld`` pads rows to a
    multiple of 4 floats so every row is 16-B aligned for 128-bit loads.
    """

    def __init__(self, L: int, rows: int, device, torch):
        self.torch = torch
        self.L = int(L)
        self.ld = (self.L + 3) // 4 * 4
        self.rows = int(rows)
        self.dev = device
        self.W = torch.zeros((self.rows, self.ld), dtype=torch.float32, device=device)
        self.lib = _native.load()
        self._scratch_words = int(self.lib.ctk_reduce_scratch_bytes(self.rows + 2, self.L)) // 8 + 1
        self._scratch = {}

    def scratch(self, stream) -> int:
        """Reduction scratch owned by one stream (zero-filled once)."""
        key = stream.cuda_stream
        buf = self._scratch.get(key)
        if buf is None:
            buf = self.torch.zeros(self._scratch_words, dtype=self.torch.float64, device=self.dev)
            self._scratch[key] = buf
        return buf.data_ptr()

    def row(self, j: int):
        return self.W[j, : self.L]

    def cgs2_step(self, k: int, q, h_out, stat_out, stream) -> None:
        """Orthogonalise q = M w_k against rows 0..k, write row k+1."""
        if k + 1 >= self.rows:
            raise ValueError(f"basis holds {self.rows} rows; step {k} would write row {k + 1}")
        _native.check(self.lib.ctk_cgs2_step(self.W.data_ptr(), self.ld, k, self.L, q.data_ptr(),
                                             h_out.data_ptr(), stat_out.data_ptr(),
                                             self.scratch(stream), stream.cuda_stream),
                      "ctk_cgs2_step")

    def gs_step(self, k: int, q, passes: int, h_out, stat_out, stream) -> None:
        """Like cgs2_step with 1 (reorthogonalize=False) or 2 Gram-Schmidt passes."""
        if k + 1 >= self.rows:
            raise ValueError(f"basis holds {self.rows} rows; step {k} would write row {k + 1}")
        _native.check(self.lib.ctk_gs_step(self.W.data_ptr(), self.ld, k, self.L, q.data_ptr(),
                                           passes, h_out.data_ptr(), stat_out.data_ptr(),
                                           self.scratch(stream), stream.cuda_stream),
                      "ctk_gs_step")

    def combine(self, k: int, y_dev, dst, x0=None, norm_out=None, stream=None) -> None:
        """dst = (x0 or 0) + W[:k]^T y   (K4, fp64 accumulation)."""
        _native.check(self.lib.ctk_combine(self.W.data_ptr(), self.ld, k, y_dev.data_ptr(),
                                           _native.ptr(x0), dst.data_ptr(), self.L,
                                           _native.ptr(norm_out), self.scratch(stream),
                                           stream.cuda_stream), "ctk_combine")

    def norm2(self, v, out, stream) -> None:
        _native.check(self.lib.ctk_norm2(v.data_ptr(), v.numel(), out.data_ptr(),
                                         self.scratch(stream), stream.cuda_stream), "ctk_norm2")

    def scale_into(self, v, dst, scale_dev, stream) -> None:
        _native.check(self.lib.ctk_scale(v.data_ptr(), dst.data_ptr(), v.numel(),
                                         scale_dev.data_ptr(), stream.cuda_stream), "ctk_scale")

    def dots(self, nvec: int, v, out, want_norm: bool, stream) -> None:
        _native.check(self.lib.ctk_dots(self.W.data_ptr(), self.ld, nvec, v.data_ptr(), self.L,
                                        1 if want_norm else 0, out.data_ptr(),
                                        self.scratch(stream), stream.cuda_stream), "ctk_dots")

    def update(self, nvec: int, coef_dev, v, dst, norm_out=None, stream=None) -> None:
        _native.check(self.lib.ctk_update(self.W.data_ptr(), self.ld, nvec, coef_dev.data_ptr(),
                                          v.data_ptr(), dst.data_ptr(), self.L,
                                          _native.ptr(norm_out), self.scratch(stream),
                                          stream.cuda_stream), "ctk_update")


# ---------------------------------------------------------------------------
# The reference's step-wise Arnoldi API (ctkrylov/arnoldi.py:28-82), the
# second seam of SURVEY row (b), with the basis resident in HBM and each step's
# orthogonalisation on libctk's Gram-Schmidt kernels.  Drivers that call
# arnoldi_step themselves (or monkeypatch it, tests/test_gmres.py:183) keep
# working; the operator is applied on the device when it can be (GPU
# projectors and their compositions), else through its host apply.
# ---------------------------------------------------------------------------

def _torch():
    import torch
    return torch


class ArnoldiState:
    """Growing orthonormal basis and Hessenberg factor for one solver run
    (ctkrylov/arnoldi.py:28-53).  ``basis`` holds w_1 .. w_{k+1} (host fp64
    copies of the HBM rows, built on access); ``hess`` is (k+1) x k;
    ``beta`` = ||r_0||_2."""

    def __init__(self, dbasis: DeviceBasis, beta: float, k: int = 0):
        self._dev = dbasis
        self.beta = float(beta)
        self.k = int(k)
        self._hess_cols: list[np.ndarray] = []
        self._breakdown = False
        torch = dbasis.torch
        self._h = torch.zeros(dbasis.rows + 8, dtype=torch.float64, device=dbasis.dev)
        self._stat = torch.zeros(4, dtype=torch.float64, device=dbasis.dev)

    @classmethod
    def start(cls, r0, device: int = 0, capacity: int = 32) -> "ArnoldiState":
        """r0: host array or CUDA tensor; ValueError on a zero residual."""
        torch = _torch()
        if not torch.cuda.is_available():
            raise _native.CtkError("a CUDA device is required: libctk has no CPU path")
        if isinstance(r0, np.ndarray) or not hasattr(r0, "is_cuda"):
            r = np.asarray(r0, dtype=np.float64)
            beta = float(np.linalg.norm(r))
            v = torch.from_numpy(r.astype(np.float32)).to(torch.device("cuda", device))
        else:
            v = r0.float()
            beta = float(torch.linalg.vector_norm(r0.double()).item())
        if beta == 0.0:
            raise ValueError("Arnoldi cannot start from a zero residual")
        db = DeviceBasis(v.numel(), max(2, capacity), v.device, torch)
        db.row(0).copy_((v.double() / beta).float())
        return cls(db, beta)

    @property
    def basis(self) -> list[np.ndarray]:
        n = self.k if self._breakdown else self.k + 1        # no row appended on breakdown
        W = self._dev.W[:n, : self._dev.L].double().cpu().numpy()
        return [W[i] for i in range(n)]

    @property
    def hess(self) -> np.ndarray:
        """The (k+1) x k upper-Hessenberg matrix assembled from stored columns."""
        return hessenberg_from_columns(self._hess_cols, self.k)

    def _ensure_rows(self, rows: int) -> None:
        db = self._dev
        if rows <= db.rows:
            return
        torch = db.torch
        new = DeviceBasis(db.L, max(rows, 2 * db.rows), db.dev, torch)
        new.W[: db.rows].copy_(db.W)
        self._dev = new
        self._h = torch.zeros(new.rows + 8, dtype=torch.float64, device=db.dev)


def _apply_on_device(M, w):
    """q = M w for a device row w (fp32 CUDA tensor)."""
    if hasattr(M, "apply_device"):
        return M.apply_device(w)
    torch = _torch()
    q = M.apply(w.double().cpu().numpy())              # host operator: the reference contract
    return torch.from_numpy(np.asarray(q, dtype=np.float32)).to(w.device)


def arnoldi_step(state: ArnoldiState, M, reorthogonalize: bool = True) -> None:
    """Advance the factorisation by one step in place (ctkrylov/arnoldi.py:56-82).

    Raises Breakdown(k) when the new direction vanishes relative to
    ||M w_k|| (BREAKDOWN_RTOL); the Hessenberg column is recorded first, as
    in the reference.  Orthogonalisation: CGS2 (or one pass) on the GPU."""
    torch = state._dev.torch
    k = state.k
    state._ensure_rows(k + 2)
    db = state._dev
    w = db.row(k)
    q = _apply_on_device(M, w)
    if q.numel() != db.L:
        from .linop import OperatorShapeError
        raise OperatorShapeError(f"operator returned {q.numel()} entries, basis rows hold {db.L}")
    q = q.contiguous().float().clone()
    stream = torch.cuda.current_stream(db.dev)
    db.gs_step(k, q, 2 if reorthogonalize else 1, state._h, state._stat, stream)
    h = state._h[: k + 2].cpu().numpy().copy()
    qn, broke = state._stat[:2].cpu().numpy()
    state._hess_cols.append(h)
    state.k = k + 1
    if broke != 0.0 or h[k + 1] <= BREAKDOWN_RTOL * qn:
        state._breakdown = True
        raise Breakdown(state.k)
