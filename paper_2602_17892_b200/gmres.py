"""Device-resident (hybrid) AB-/BA-GMRES: the run_gmres twin.

Same signature, configuration, records, stop reasons and restart semantics as
ctkrylov/gmres.py:135-241, but the Krylov basis, iterates and residuals live
in HBM for the whole solve:

* per step: one M-apply (K2 -> K1 for AB, K1 -> K2 for BA), the fused CGS2
  orthogonalisation (K3), and a (k+2)-double Hessenberg column D2H;
* on the host, in fp64: Hessenberg SVD, lambda selection (GCV / L-curve /
  fixed), projected Tikhonov solve -> y (k doubles H2D);
* per iterate: K4 combination x_k = x0 + W y (BA) or x0 + B(W y) (AB),
  the true residual b - A x_k fused into K1, fp64 norms.

The host never waits for the iterate: the next Arnoldi step only needs
w_{k+1}, so it is enqueued (speculatively) before the host solves the
projected problem of step k, and the GPU runs it while the host works
(SURVEY.md §7.3-6).  Residual and solution norms are read back once at the
end unless a stopping rule or x_true needs them every iteration.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import metrics
from .arnoldi import (BREAKDOWN_RTOL, DeviceBasis, hessenberg_from_columns,  # noqa: F401
                      solve_projected_tikhonov)
from .ct import GpuBack, GpuForward
from .linop import LinearOperator, OperatorShapeError
from .regparam import DegenerateCurveError, select_lambda, svd_of_hessenberg

GMRES_METHODS = ("ab", "ba", "ab-hybrid", "ba-hybrid")
GK_METHODS = ("lsqr", "lsmr", "lsqr-hybrid", "lsmr-hybrid")
ALL_METHODS = GMRES_METHODS + GK_METHODS


class ConfigError(ValueError):
    """Inconsistent solver configuration (ctkrylov/gmres.py:29-30)."""


@dataclass(frozen=True)
class SolverConfig:
    """Everything that determines one solver run (ctkrylov/gmres.py:33-92)."""

    method: str = "ab"
    max_iter: int = 100
    lambda_strategy: str = "none"
    lambda_value: float | None = None
    stopping_rule: str = "none"
    dp_tau: float = metrics.DEFAULT_DP_TAU
    noise_norm: float | None = None
    ncp_threshold: float = metrics.DEFAULT_NCP_THRESHOLD
    rns_epsilon: float = metrics.DEFAULT_RNS_EPSILON
    restart_period: int = 0
    reorthogonalize: bool = True
    x0: np.ndarray | None = None
    snapshot_stride: int = 0
    name: str | None = None

    def validate(self) -> None:
        if self.method not in ALL_METHODS:
            raise ConfigError(f"unknown method {self.method!r}; choose from {ALL_METHODS}")
        hybrid = self.method.endswith("-hybrid")
        if hybrid and self.lambda_strategy == "none":
            raise ConfigError(f"{self.method} requires a lambda strategy other than 'none'")
        if not hybrid and self.lambda_strategy != "none":
            raise ConfigError(f"plain method {self.method!r} cannot use lambda strategy "
                              f"{self.lambda_strategy!r}; use the -hybrid variant")
        if self.lambda_strategy == "fixed" and (self.lambda_value is None or self.lambda_value < 0):
            raise ConfigError("fixed lambda strategy requires a nonnegative lambda_value")
        if self.max_iter < 1:
            raise ConfigError(f"max_iter must be positive, got {self.max_iter}")
        if self.restart_period < 0:
            raise ConfigError(f"restart_period must be nonnegative, got {self.restart_period}")
        if self.stopping_rule == "dp":
            if self.noise_norm is None or self.noise_norm < 0:
                raise ConfigError("dp stopping requires a nonnegative noise_norm")
            if self.dp_tau < 1.0:
                raise ConfigError(f"dp safety factor must be >= 1, got {self.dp_tau}")
        if self.stopping_rule not in ("none", "dp", "ncp", "rns"):
            raise ConfigError(f"unknown stopping rule {self.stopping_rule!r}")

    @property
    def label(self) -> str:
        if self.name:
            return self.name
        parts = [self.method]
        if self.lambda_strategy != "none":
            parts.append(self.lambda_strategy)
        if self.restart_period:
            parts.append(f"p{self.restart_period}")
        return "-".join(parts)


@dataclass
class IterationRecord:
    k: int
    lambda_used: float
    residual_norm: float
    data_residual_norm: float
    proj_residual_norm: float
    solution_norm: float
    rre: float | None = None
    ssim: float | None = None
    elapsed: float = 0.0
    lambda_warning: bool = False


@dataclass
class SolveResult:
    x: np.ndarray
    records: list[IterationRecord]
    stop_reason: str
    cycles: int = 1
    snapshots: dict[int, np.ndarray] = field(default_factory=dict)

    @property
    def data_residuals(self) -> np.ndarray:
        return np.array([r.data_residual_norm for r in self.records])

    @property
    def rres(self) -> np.ndarray:
        return np.array([r.rre for r in self.records], dtype=np.float64)


def _check_dims(A: LinearOperator, B: LinearOperator, m: int) -> None:
    if A.cols != B.rows or B.cols != A.rows:
        raise OperatorShapeError(
            f"forward {A.rows}x{A.cols} and back {B.rows}x{B.cols} are not a projector pair")
    if m != A.rows:
        raise OperatorShapeError(f"data vector has shape ({m},), expected ({A.rows},)")


class KernelTimer:
    """CUDA-event brackets around projector launches (bench roofline)."""

    def __init__(self, torch):
        self.torch = torch
        self.events: dict[str, list] = {}

    def bracket(self, name, stream):
        torch = self.torch
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        self.events.setdefault(name, []).append((e0, e1))
        return e1

    def summary(self) -> dict[str, tuple[int, float]]:
        """name -> (launches, mean ms); call after synchronising."""
        out = {}
        for name, evs in self.events.items():
            ms = [a.elapsed_time(b) for a, b in evs]
            out[name] = (len(ms), float(np.mean(ms)) if ms else 0.0)
        return out


class _DeviceSolve:
    def __init__(self, A, B, b, cfg, x_true, image_shape, stream, timer, keep_on_device=False):
        if not isinstance(A, GpuForward) or not isinstance(B, GpuBack) or A.dgeom is not B.dgeom:
            raise TypeError("the device-resident run_gmres needs the GPU projector pair from "
                            "paper_2602_17892_b200.ct (forward_ray_driven / back_pixel_driven "
                            "on one geometry)")
        self.A, self.B, self.cfg = A, B, cfg
        dg = self.dg = A.dgeom
        torch = self.torch = dg.torch
        self.stream = stream if stream is not None else torch.cuda.current_stream(dg.dev)
        self.timer = timer
        self.keep_on_device = keep_on_device
        self.h2d = 0                     # bytes copied host->device / device->host by the solve
        self.d2h = 0
        self.x_true = None if x_true is None else np.asarray(x_true, dtype=np.float64)
        self.image_shape = image_shape
        self.ab = cfg.method.startswith("ab")
        self.hybrid = cfg.method.endswith("-hybrid")
        self.n, self.m = dg.n, dg.m
        L = self.m if self.ab else self.n
        self.K = cfg.max_iter
        self.p = cfg.restart_period if cfg.restart_period > 0 else self.K
        rows = min(self.p, self.K) + 1
        f32, f64, dev = torch.float32, torch.float64, dg.dev
        with torch.cuda.stream(self.stream):
            if torch.is_tensor(b):
                if b.numel() != self.m:
                    raise OperatorShapeError(f"data vector has {b.numel()} entries, expected {self.m}")
                self.b = b.to(device=dev, dtype=f32).contiguous()
            else:
                bh = np.asarray(b, dtype=np.float64)
                if bh.shape != (self.m,):
                    raise OperatorShapeError(f"data vector has shape {bh.shape}, expected ({self.m},)")
                self.b = torch.from_numpy(bh.astype(np.float32)).pin_memory().to(dev, non_blocking=True)
                self.h2d += 4 * self.m
            self.basis = DeviceBasis(L, rows, dev, torch)
            x0 = cfg.x0
            if x0 is None:
                self.x_cur = torch.zeros(self.n, dtype=f32, device=dev)
            else:
                x0 = np.asarray(x0, dtype=np.float64)
                if x0.shape != (self.n,):
                    raise ConfigError(f"x0 has shape {x0.shape}, expected ({self.n},)")
                self.x_cur = torch.from_numpy(x0.astype(np.float32)).to(dev)
                self.h2d += 4 * self.n
            self.xk = torch.empty(self.n, dtype=f32, device=dev)
            self.q = torch.empty(L, dtype=f32, device=dev)
            self.tmp = torch.empty(self.n if self.ab else self.m, dtype=f32, device=dev)
            self.z = torch.empty(self.m, dtype=f32, device=dev) if self.ab else None
            self.r = torch.empty(self.m, dtype=f32, device=dev)
            self.hcols = rows + 1 + 4                      # h[0..rows] + 4 stats
            self.hs = torch.zeros((rows, self.hcols), dtype=f64, device=dev)
            self.h_host = torch.zeros((rows, self.hcols), dtype=f64).pin_memory()
            self.y_dev = torch.zeros((self.K, rows), dtype=f64, device=dev)
            self.y_pin = torch.zeros((self.K, rows), dtype=f64).pin_memory()
            self.norms = torch.zeros((self.K + 1, 2), dtype=f64, device=dev)   # res^2, sol^2
            self.scal = torch.zeros(4, dtype=f64, device=dev)
            self.scal_host = torch.zeros(4, dtype=f64).pin_memory()
        self.ev_h = [None] * rows

    # -- projector launches (optionally event-bracketed) ------------------
    def _fwd(self, x, out, b=None):
        if self.timer is None:
            return self.dg.forward(x, out=out, b=b, stream=self.stream)
        e1 = self.timer.bracket("forward", self.stream)
        self.dg.forward(x, out=out, b=b, stream=self.stream)
        e1.record(self.stream)

    def _back(self, u, out, x0=None):
        if self.timer is None:
            return self.dg.back(u, out=out, x0=x0, stream=self.stream)
        e1 = self.timer.bracket("back", self.stream)
        self.dg.back(u, out=out, x0=x0, stream=self.stream)
        e1.record(self.stream)

    def _arnoldi(self, j):
        """Enqueue step j: q = M w_j, CGS2 -> h column + w_{j+1}; D2H h."""
        torch = self.torch
        w = self.basis.row(j)
        if self.ab:
            self._back(w, self.tmp)
            self._fwd(self.tmp, self.q)
        else:
            self._fwd(w, self.tmp)
            self._back(self.tmp, self.q)
        hrow = self.hs[j]
        stat = hrow[self.hcols - 4:]
        self.basis.cgs2_step(j, self.q, hrow, stat, self.stream)
        with torch.cuda.stream(self.stream):
            self.h_host[j].copy_(hrow, non_blocking=True)
        self.d2h += 8 * self.hcols
        ev = torch.cuda.Event()
        ev.record(self.stream)
        self.ev_h[j] = ev

    def _iterate(self, it, k, y):
        """Enqueue x_k = x0 + (B) W y, r = b - A x_k, norms into slot it."""
        torch = self.torch
        with torch.cuda.stream(self.stream):
            self.y_pin[it, :k] = torch.from_numpy(y)
            self.y_dev[it, :k].copy_(self.y_pin[it, :k], non_blocking=True)
        self.h2d += 8 * k
        ydev = self.y_dev[it]
        nrm = self.norms[it]
        if self.ab:
            self.basis.combine(k, ydev, self.z, stream=self.stream)
            self._back(self.z, self.xk, x0=self.x_cur)
            self.basis.norm2(self.xk, nrm[1:2], self.stream)
        else:
            self.basis.combine(k, ydev, self.xk, x0=self.x_cur, norm_out=nrm[1:2],
                               stream=self.stream)
        self._fwd(self.xk, self.r, b=self.b)
        self.basis.norm2(self.r, nrm[0:1], self.stream)
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(self.stream)
        return ev

    def _host_vec(self, t):
        self.d2h += 4 * t.numel()
        with self.torch.cuda.stream(self.stream):
            return t.to("cpu", non_blocking=False).numpy().astype(np.float64)

    def run(self) -> SolveResult:
        torch, cfg = self.torch, self.cfg
        K, p = self.K, self.p
        records: list[IterationRecord] = []
        pending: list[tuple] = []          # (record, slot, event)
        history: list[float] = []
        snapshots: dict[int, np.ndarray] = {}
        stop = None
        cycles = 0
        prev_lam = 0.0
        need_sync = cfg.stopping_rule != "none" or self.x_true is not None
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_start.record(self.stream)
        t_start = time.perf_counter()
        first_cycle = True
        while stop is None and len(records) < K:
            if not first_cycle:
                with torch.cuda.stream(self.stream):
                    self.x_cur.copy_(self.xk)
            first_cycle = False
            # ---- cycle start: r0 = b - A x (AB) or B(b - A x) (BA), beta = ||r0||
            w0 = self.basis.row(0)
            if self.ab:
                self._fwd(self.x_cur, w0, b=self.b)
                self.basis.norm2(w0, self.scal[0:1], self.stream)
            else:
                self._fwd(self.x_cur, self.r, b=self.b)
                self.basis.norm2(self.r, self.scal[1:2], self.stream)
                self._back(self.r, w0)
                self.basis.norm2(w0, self.scal[0:1], self.stream)
            with torch.cuda.stream(self.stream):
                self.scal_host.copy_(self.scal, non_blocking=True)
            self.d2h += 32
            self.stream.synchronize()
            beta = float(np.sqrt(self.scal_host[0].item()))
            d0n = beta if self.ab else float(np.sqrt(self.scal_host[1].item()))
            if beta == 0.0:
                stop = "breakdown"
                if not records:
                    x_host = self._host_vec(self.x_cur)
                    records.append(self._make_record(0, 0.0, 0.0, d0n, 0.0,
                                                     float(np.linalg.norm(x_host)), x_host,
                                                     time.perf_counter() - t_start))
                break
            cycles += 1
            with torch.cuda.stream(self.stream):
                self.scal[2] = 1.0 / beta
            self.basis.scale_into(w0, w0, self.scal[2:3], self.stream)

            steps = min(p, K - len(records))
            cols: list[np.ndarray] = []
            self._arnoldi(0)
            last_ev = None
            for j in range(steps):
                self.ev_h[j].synchronize()
                hrow = self.h_host[j].numpy()
                cols.append(hrow[: j + 2].copy())
                broke = hrow[self.hcols - 3] != 0.0
                k = j + 1
                if not broke and j + 1 < steps:
                    self._arnoldi(j + 1)          # speculative: overlaps the host work below
                H = hessenberg_from_columns(cols, k)
                svd = svd_of_hessenberg(H)
                warn = False
                if self.hybrid:
                    try:
                        lam = select_lambda(H, beta, cfg.lambda_strategy, cfg.lambda_value, svd=svd)
                    except DegenerateCurveError:
                        lam, warn = prev_lam, True
                else:
                    lam = 0.0
                prev_lam = lam
                sol = solve_projected_tikhonov(H, beta, lam, svd=svd)
                slot = len(records)
                ev = self._iterate(slot, k, sol.y)
                last_ev = ev
                rec = IterationRecord(k=slot + 1, lambda_used=float(lam), residual_norm=0.0,
                                      data_residual_norm=0.0,
                                      proj_residual_norm=sol.proj_residual_norm,
                                      solution_norm=0.0, lambda_warning=warn)
                records.append(rec)
                if cfg.snapshot_stride and rec.k % cfg.snapshot_stride == 0:
                    snapshots[rec.k] = self._host_vec(self.xk)
                if need_sync:
                    ev.synchronize()
                    self._finish(rec, slot, ev_start, ev)
                    history.append(rec.data_residual_norm)
                    if self.x_true is not None:
                        xh = self._host_vec(self.xk)
                        self._metrics(rec, xh)
                    if cfg.stopping_rule == "dp" and metrics.dp_should_stop(
                            rec.data_residual_norm, cfg.noise_norm, cfg.dp_tau):
                        stop = "dp"
                    elif cfg.stopping_rule == "ncp" and metrics.ncp_should_stop(
                            self._host_vec(self.r), cfg.ncp_threshold):
                        stop = "ncp"
                    elif cfg.stopping_rule == "rns" and metrics.rns_should_stop(
                            history, cfg.rns_epsilon):
                        stop = "rns"
                else:
                    pending.append((rec, slot, ev))
                if broke and stop is None:
                    stop = "breakdown"
                if stop is not None:
                    break
            if last_ev is not None:
                last_ev.synchronize()
        self.stream.synchronize()
        if pending:
            norms = self.norms.cpu().numpy()
            self.d2h += self.norms.numel() * 8
            for rec, slot, ev in pending:
                self._finish(rec, slot, ev_start, ev, norms)
        x_final = self.xk if records and records[-1].k > 0 else self.x_cur
        x_out = x_final.clone() if self.keep_on_device else self._host_vec(x_final)
        res = SolveResult(x=x_out, records=records, stop_reason=stop or "maxiter",
                          cycles=max(cycles, 1), snapshots=snapshots)
        res.transfer = {"h2d_bytes": self.h2d, "d2h_bytes": self.d2h}
        return res

    def _finish(self, rec, slot, ev_start, ev, norms=None):
        if norms is None:
            norms = self.norms[slot].cpu().numpy()[None, :]
            row = norms[0]
        else:
            row = norms[slot]
        rec.data_residual_norm = float(np.sqrt(row[0]))
        rec.solution_norm = float(np.sqrt(row[1]))
        rec.residual_norm = rec.data_residual_norm if self.ab else rec.proj_residual_norm
        rec.elapsed = ev_start.elapsed_time(ev) / 1000.0

    def _metrics(self, rec, x_host):
        rec.rre = metrics.rre(x_host, self.x_true)
        if self.image_shape is not None and min(self.image_shape) >= 8:
            rec.ssim = metrics.ssim(x_host, self.x_true, self.image_shape)

    def _make_record(self, k, lam, method_norm, data_norm, proj_norm, sol_norm, x_host, elapsed):
        rec = IterationRecord(k=k, lambda_used=float(lam), residual_norm=float(method_norm),
                              data_residual_norm=float(data_norm),
                              proj_residual_norm=float(proj_norm),
                              solution_norm=float(sol_norm), elapsed=elapsed)
        if self.x_true is not None:
            self._metrics(rec, x_host)
        return rec


def run_gmres(A: LinearOperator, B: LinearOperator, b, cfg: SolverConfig,
              x_true: np.ndarray | None = None, image_shape: tuple[int, int] | None = None,
              *, stream=None, kernel_timer: KernelTimer | None = None,
              keep_on_device: bool = False) -> SolveResult:
    """(Hybrid) AB-/BA-GMRES with optional restarting, on the GPU.

    ``b`` may be a host array (the reference's contract) or a CUDA tensor
    (device-resident input).  Returns a SolveResult with a host ``x`` (a CUDA
    tensor when ``keep_on_device``); ``result.transfer`` counts the bytes the
    solve moved across PCIe.
    """
    cfg.validate()
    if cfg.method not in GMRES_METHODS:
        raise ConfigError(f"run_gmres got non-GMRES method {cfg.method!r}")
    shape = tuple(b.shape)
    if len(shape) != 1:
        raise OperatorShapeError(f"data vector has shape {shape}, expected ({A.rows},)")
    _check_dims(A, B, int(shape[0]))
    return _DeviceSolve(A, B, b, cfg, x_true, image_shape, stream, kernel_timer,
                        keep_on_device).run()


def run_ab_gmres(A, B, b, cfg: SolverConfig, **kwargs) -> SolveResult:
    if not cfg.method.startswith("ab"):
        cfg = replace(cfg, method="ab-hybrid" if cfg.lambda_strategy != "none" else "ab")
    return run_gmres(A, B, b, cfg, **kwargs)


def run_ba_gmres(A, B, b, cfg: SolverConfig, **kwargs) -> SolveResult:
    if not cfg.method.startswith("ba"):
        cfg = replace(cfg, method="ba-hybrid" if cfg.lambda_strategy != "none" else "ba")
    return run_gmres(A, B, b, cfg, **kwargs)
