"""Golub-Kahan solvers -- (hybrid) LSQR and LSMR -- on the GPU.

Device-resident twin of ``ctkrylov.gk`` (gk.py:1-205): the same
``run_lsqr(A, At, b, cfg)`` / ``run_lsmr`` signatures, ``SolverConfig``
validation, records and stop reasons, for the matched pair
``A = forward_ray_driven(...)``, ``At = matched_back(A)`` (K1 + K7).

Per iteration (reference ``_bidiag_step``, gk.py:64-88):

* v = A^T u_k, orthogonalised against V (two Gram-Schmidt passes, K3) and
  normalised -> alpha;  u = A v_k against U -> beta.  Both bases stay in HBM
  (fp32 rows, fp64 accumulation), as the reference keeps both with full
  reorthogonalisation.  Breakdown when alpha or beta <= 1e-14 beta_init.
* the (k+1) x k lower bidiagonal B_k goes to the native fp64 projected solve
  (``ctk_projected_solve``: lambda by GCV/L-curve/fixed exactly as
  ``select_lambda``, LSQR's Tikhonov y).
* LSMR (gk.py:145-150) minimises ||G y - A^T b||^2 + lam^2 ||y||^2 with
  G = [A^T A v_1 .. A^T A v_k]; here G is orthogonalised as it grows
  (G = Q R, K3 again) so the projected problem is the k x k damped problem
  on R and Q^T A^T b (host fp64 lstsq), instead of a dense n x k lstsq.
* x_k = V y, b - A x_k = b - sum y_j (A v_j) and (LSMR) A^T(b - A x_k) =
  A^T b - sum y_j (A^T A v_j) are basis combinations (K4) over rows kept
  during the bidiagonalisation: no extra projector apply per iteration.
"""

from __future__ import annotations

import time

import numpy as np

from . import _native, metrics
from .ct import GpuAdjoint, GpuForward
from .gmres import (ConfigError, IterationRecord, SolveResult, SolverConfig, _check_dims,
                    _blas_single_thread)
from .linop import OperatorShapeError

BREAKDOWN_RTOL = 1e-14                    # ctkrylov/gk.py:72,82


class _GkSolve:
    def __init__(self, A, At, b, cfg: SolverConfig, flavor: str, x_true, image_shape):
        if not isinstance(A, GpuForward) or not isinstance(At, GpuAdjoint) or A.dgeom is not At.dgeom:
            raise TypeError("the device Golub-Kahan solvers need A = forward_ray_driven(...) and "
                            "At = matched_back(A) on one geometry")
        cfg.validate()
        _check_dims(A, At, A.rows)
        if cfg.x0 is not None and np.any(cfg.x0):
            raise ConfigError("Golub-Kahan solvers support only x0 = 0")
        if cfg.restart_period:
            raise ConfigError("Golub-Kahan solvers do not restart")
        self.A, self.At, self.cfg, self.flavor = A, At, cfg, flavor
        dg = self.dg = A.dgeom
        torch = self.torch = dg.torch
        self.lib = _native.load()
        self.x_true = None if x_true is None else np.asarray(x_true, dtype=np.float64)
        self.image_shape = image_shape
        self.hybrid = cfg.method.endswith("-hybrid")
        self.n, self.m = dg.n, dg.m
        K = self.K = cfg.max_iter
        dev = dg.dev
        if torch.is_tensor(b):
            if b.numel() != self.m:
                raise OperatorShapeError(f"data vector has {b.numel()} entries, expected {self.m}")
            self.b = b.to(device=dev, dtype=torch.float32).contiguous()
        else:
            bh = np.asarray(b, dtype=np.float64)
            if bh.shape != (self.m,):
                raise OperatorShapeError(f"data vector has shape {bh.shape}, expected ({self.m},)")
            self.b = torch.from_numpy(bh.astype(np.float32)).to(dev)
        from .arnoldi import DeviceBasis
        self.U = DeviceBasis(self.m, K + 2, dev, torch)
        self.V = DeviceBasis(self.n, K + 2, dev, torch)
        self.AV = DeviceBasis(self.m, K + 1, dev, torch)          # rows A v_j
        if flavor == "lsmr":
            self.G = DeviceBasis(self.n, K + 2, dev, torch)       # orthonormalised A^T A v_j
            self.AtAV = DeviceBasis(self.n, K + 1, dev, torch)    # rows A^T A v_j
            self.R = np.zeros((K + 1, K + 1))
        f32, f64 = torch.float32, torch.float64
        self.tn = torch.empty(self.n, dtype=f32, device=dev)
        self.tm = torch.empty(self.m, dtype=f32, device=dev)
        self.xk = torch.empty(self.n, dtype=f32, device=dev)
        self.r = torch.empty(self.m, dtype=f32, device=dev)
        self.h = torch.zeros(K + 8, dtype=f64, device=dev)
        self.stat = torch.zeros(4, dtype=f64, device=dev)
        self.sc = torch.zeros(4, dtype=f64, device=dev)
        self.stream = torch.cuda.current_stream(dev)

    # -- helpers ----------------------------------------------------------
    def _norm(self, v, basis) -> float:
        basis.norm2(v, self.sc[0:1], self.stream)
        return float(np.sqrt(self.sc[0].item()))

    def _orth_into(self, basis, k, q) -> float:
        """q orthogonalised against rows 0..k-1 of basis, normalised into row
        k; returns its norm before normalisation (alpha / beta)."""
        if k == 0:
            nrm = self._norm(q, basis)
            inv = self.torch.tensor([1.0 / nrm if nrm > 0 else 0.0], dtype=self.torch.float64,
                                    device=self.dg.dev)
            basis.scale_into(q, basis.row(0), inv, self.stream)
            return nrm
        passes = 2 if self.cfg.reorthogonalize else 1
        basis.gs_step(k - 1, q, passes, self.h, self.stat, self.stream)
        return float(self.stat[3].item())

    def _combine(self, basis, k, y, base, dst):
        yd = self.torch.from_numpy(np.ascontiguousarray(y, dtype=np.float64)).to(self.dg.dev)
        basis.combine(k, yd, dst, x0=base, norm_out=self.sc[1:2], stream=self.stream)
        return float(np.sqrt(self.sc[1].item()))

    # -- the solve ----------------------------------------------------------
    def run(self) -> SolveResult:
        with _blas_single_thread():
            return self._run()

    def _run(self) -> SolveResult:
        torch, cfg, dg = self.torch, self.cfg, self.dg
        K = self.K
        t0 = time.perf_counter()
        beta_init = self._norm(self.b, self.U)
        if beta_init == 0.0:
            raise ValueError("cannot bidiagonalize a zero right-hand side")    # gk.py:58
        inv = torch.tensor([1.0 / beta_init], dtype=torch.float64, device=dg.dev)
        self.U.scale_into(self.b, self.U.row(0), inv, self.stream)
        if self.flavor == "lsmr":
            At_b = dg.adjoint(self.b, stream=self.stream)
        alphas: list[float] = []
        betas: list[float] = []
        k = 0
        records: list[IterationRecord] = []
        history: list[float] = []
        snapshots: dict[int, np.ndarray] = {}
        stop = None
        prev_lam = 0.0
        x_host = np.zeros(self.n)
        code = _native.STRATEGY_CODES.get(cfg.lambda_strategy, 0) if self.hybrid else 0
        for _ in range(K):
            # -- one Golub-Kahan step (gk.py:64-88) --
            broke = False
            dg.adjoint(self.U.row(k), out=self.tn, stream=self.stream)
            alpha = self._orth_into(self.V, k, self.tn)
            if alpha <= BREAKDOWN_RTOL * beta_init:
                broke = True
            else:
                alphas.append(alpha)
                dg.forward(self.V.row(k), out=self.AV.row(k), stream=self.stream)
                if self.flavor == "lsmr":
                    dg.adjoint(self.AV.row(k), out=self.AtAV.row(k), stream=self.stream)
                self.tm.copy_(self.AV.row(k))
                beta = self._orth_into(self.U, k + 1, self.tm)
                if self.flavor == "lsmr":
                    self.tn.copy_(self.AtAV.row(k))
                    rho = self._orth_into(self.G, k, self.tn)
                    hk = self.h.cpu().numpy() if k > 0 else np.zeros(1)
                    self.R[:k, k] = hk[:k]
                    self.R[k, k] = rho
                k += 1
                if beta <= BREAKDOWN_RTOL * beta_init:
                    betas.append(0.0)
                    broke = True
                else:
                    betas.append(beta)
            if k == 0:
                stop = "breakdown"
                break
            Bk = np.zeros((k + 1, k))
            for i in range(k):
                Bk[i, i] = alphas[i]
                Bk[i + 1, i] = betas[i]
            out = np.empty(4)
            y = np.empty(k)
            _native.check(self.lib.ctk_projected_solve(
                Bk.ctypes.data, k, float(beta_init), code, float(cfg.lambda_value or 0.0), 200,
                float("nan"), out.ctypes.data, y.ctypes.data), "ctk_projected_solve")
            lam = 0.0
            if self.hybrid:
                lam = prev_lam if out[2] != 0.0 else float(out[0])     # DegenerateCurveError
                if out[2] != 0.0:
                    _native.check(self.lib.ctk_projected_solve(
                        Bk.ctypes.data, k, float(beta_init), 1, lam, 200, float("nan"),
                        out.ctypes.data, y.ctypes.data), "ctk_projected_solve")
            prev_lam = lam
            if self.flavor == "lsqr":
                proj = float(out[1])
            else:
                # min ||G y - A^T b||^2 + lam^2 ||y||^2 with G = Q R
                d = np.empty(k)
                qd = torch.empty(k + 1, dtype=torch.float64, device=dg.dev)
                _native.check(self.lib.ctk_dots(self.G.W.data_ptr(), self.G.ld, k, At_b.data_ptr(),
                                                self.G.L, 0, qd.data_ptr(),
                                                self.G.scratch(self.stream), self.stream.cuda_stream),
                              "ctk_dots")
                d[:] = qd[:k].cpu().numpy()
                R = self.R[:k, :k]
                if lam > 0.0:
                    y = np.linalg.lstsq(np.vstack([R, lam * np.eye(k)]),
                                        np.concatenate([d, np.zeros(k)]), rcond=None)[0]
                else:
                    y = np.linalg.lstsq(R, d, rcond=None)[0]
            sol_norm = self._combine(self.V, k, y, None, self.xk)
            data_norm = self._combine(self.AV, k, -y, self.b, self.r)
            if self.flavor == "lsqr":
                method_norm = data_norm
            else:
                ne = torch.empty(self.n, dtype=torch.float32, device=dg.dev)
                method_norm = self._combine(self.AtAV, k, -y, At_b, ne)
                proj = method_norm
            need_x = self.x_true is not None or (cfg.snapshot_stride and
                                                  (len(records) + 1) % cfg.snapshot_stride == 0)
            if need_x:
                x_host = self.xk.cpu().numpy().astype(np.float64)
            rec = IterationRecord(k=len(records) + 1, lambda_used=float(lam),
                                  residual_norm=float(method_norm), data_residual_norm=float(data_norm),
                                  proj_residual_norm=float(proj), solution_norm=float(sol_norm),
                                  elapsed=time.perf_counter() - t0)
            if self.x_true is not None:
                rec.rre = metrics.rre(x_host, self.x_true)
                if self.image_shape is not None and min(self.image_shape) >= 8:
                    rec.ssim = metrics.ssim(x_host, self.x_true, self.image_shape)
            records.append(rec)
            history.append(float(data_norm))
            if cfg.snapshot_stride and rec.k % cfg.snapshot_stride == 0:
                snapshots[rec.k] = x_host.copy()
            if cfg.stopping_rule == "dp" and metrics.dp_should_stop(
                    data_norm, cfg.noise_norm, cfg.dp_tau):
                stop = "dp"
            elif cfg.stopping_rule == "ncp" and (
                    _ncp_device(torch, self.r, self.stream) <= cfg.ncp_threshold):
                stop = "ncp"
            elif cfg.stopping_rule == "rns" and metrics.rns_should_stop(history, cfg.rns_epsilon):
                stop = "rns"
            if broke and stop is None:
                stop = "breakdown"
            if stop is not None:
                break
        if stop is None:
            stop = "maxiter"
        x = self.xk.cpu().numpy().astype(np.float64) if records else np.zeros(self.n)
        return SolveResult(x=x, records=records, stop_reason=stop, cycles=1, snapshots=snapshots)


def _ncp_device(torch, r, stream) -> float:
    """NCP distance of the residual on the device (ctkrylov/stopping.py:27-46)."""
    m = r.numel()
    with torch.cuda.stream(stream):
        power = torch.fft.rfft(r.to(torch.float64)).abs().square()[1: m // 2 + 1]
        total = power.sum()
        c = torch.cumsum(power, 0) / total
        diag = torch.arange(1, m // 2 + 1, dtype=torch.float64, device=r.device) / (m // 2)
        dist = torch.where(total > 0, (c - diag).abs().max(), torch.zeros_like(total))
    return float(dist.item())


def run_lsqr(A, At, b, cfg: SolverConfig, x_true=None, image_shape=None) -> SolveResult:
    """(Hybrid) LSQR (ctkrylov/gk.py:192-197); At must be matched_back(A)."""
    if cfg.method not in ("lsqr", "lsqr-hybrid"):
        raise ConfigError(f"run_lsqr got method {cfg.method!r}")
    return _GkSolve(A, At, b, cfg, "lsqr", x_true, image_shape).run()


def run_lsmr(A, At, b, cfg: SolverConfig, x_true=None, image_shape=None) -> SolveResult:
    """(Hybrid) LSMR (ctkrylov/gk.py:200-205); At must be matched_back(A)."""
    if cfg.method not in ("lsmr", "lsmr-hybrid"):
        raise ConfigError(f"run_lsmr got method {cfg.method!r}")
    return _GkSolve(A, At, b, cfg, "lsmr", x_true, image_shape).run()
