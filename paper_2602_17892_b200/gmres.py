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

import ctypes
import os
import threading
import time
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native, metrics
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


_POOL = None
_STREAMS: dict = {}


def _pool():
    """Host worker threads for the per-iteration projected problems (LAPACK
    releases the GIL, so independent iterations' SVDs run in parallel)."""
    global _POOL
    if _POOL is None:
        import os
        from concurrent.futures import ThreadPoolExecutor
        _POOL = ThreadPoolExecutor(max_workers=max(2, min(8, (os.cpu_count() or 2) - 1)),
                                   thread_name_prefix="ctk-lambda")
    return _POOL


_PINNED_LOCAL = threading.local()
_PINNED_KEEP = 16                              # buffers kept per thread (LRU)


def _pinned(torch, name, shape, dtype, zero=True):
    """Page-locked host buffer reused across solves (per thread, name, shape,
    dtype).  A fresh pin_memory() per solve goes through torch's caching host
    allocator, which falls back to cudaHostAlloc (milliseconds) whenever the
    previous solve's block is still fenced by an event.  Solves are
    synchronous, so a buffer is free again when its solve returns.  The cache
    is thread-local (freed with its thread) and keeps the _PINNED_KEEP most
    recently used buffers; release_pinned() drops the calling thread's."""
    from collections import OrderedDict
    cache = getattr(_PINNED_LOCAL, "cache", None)
    if cache is None:
        cache = _PINNED_LOCAL.cache = OrderedDict()
    key = (name, tuple(shape), dtype)
    t = cache.get(key)
    if t is None:
        t = torch.empty(shape, dtype=dtype).pin_memory()
        cache[key] = t
        while len(cache) > _PINNED_KEEP:
            cache.popitem(last=False)
    else:
        cache.move_to_end(key)
    if zero:
        t.zero_()
    return t


def release_pinned() -> None:
    """Free the calling thread's cached page-locked buffers."""
    _PINNED_LOCAL.cache = None


_WORKSPACES: dict = {}
_WORKSPACE_KEEP = 8                            # shapes x threads kept alive
_CACHE_LOCK = threading.Lock()


def _solve_workspace(torch, dg, ab, L, rows, K):
    """Device buffers of one solve shape, reused by later solves of the same
    shape on this thread (allocation + zero-fill of ~10 tensors costs more
    host time than a c1 Arnoldi step).  Every buffer is written before it is
    read inside a solve (the reduction scratch resets its own tickets);
    x_cur is re-zeroed per solve.  Keeps the 4 most recent shapes."""
    key = (threading.get_ident(), id(dg), bool(ab), int(L), int(rows), int(K))
    with _CACHE_LOCK:
        ws = _WORKSPACES.pop(key, None)
    if ws is None:
        f32, f64, dev = torch.float32, torch.float64, dg.dev
        n, m = dg.n, dg.m
        ldm, ldn = (m + 3) // 4 * 4, (n + 3) // 4 * 4
        hcols = rows + 1 + 4
        ws = {
            "basis": DeviceBasis(L, rows, dev, torch),
            "x_cur": torch.zeros(n, dtype=f32, device=dev),
            "q": torch.empty(L, dtype=f32, device=dev),
            "tmp": torch.empty(n if ab else m, dtype=f32, device=dev),
            "hs": torch.zeros((rows, hcols), dtype=f64, device=dev),
            "scal": torch.zeros(4, dtype=f64, device=dev),
            "xk": torch.empty(n, dtype=f32, device=dev),
            "z": torch.empty(m, dtype=f32, device=dev) if ab else None,
            "aux1": torch.zeros((rows, ldn if ab else ldm), dtype=f32, device=dev),
            "aux2": torch.zeros((rows, ldm), dtype=f32, device=dev) if ab else None,
            "d0": torch.zeros(ldm, dtype=f32, device=dev),
            "r": torch.empty(m, dtype=f32, device=dev),
            "y_dev": torch.zeros((K, rows), dtype=f64, device=dev),
            "norms": torch.zeros((K + 1, 2), dtype=f64, device=dev),
        }
    with _CACHE_LOCK:
        _WORKSPACES[key] = ws                  # most recent last
        while len(_WORKSPACES) > _WORKSPACE_KEEP:
            _WORKSPACES.pop(next(iter(_WORKSPACES)))
    return ws


def _side_stream(torch, dev, kind, priority):
    """Cached solver streams: the Arnoldi stream at the highest priority (it is
    the critical path), the iterate stream at the lowest.  Per host thread, so
    independent solves issued from different threads (batched slices) run
    concurrently instead of serialising on one stream pair."""
    key = (dev.index, kind, threading.get_ident())
    with _CACHE_LOCK:
        s = _STREAMS.get(key)
        if s is None:
            s = torch.cuda.Stream(dev, priority=priority)
            _STREAMS[key] = s
    return s


def _projected_task(lib, H, beta, code, value, fallback=float("nan")):
    """Native fp64 projected problem of one iteration (SVD, lambda selection,
    Tikhonov solve; ctk_host.cpp).  ctypes drops the GIL for the call, so
    several iterations solve concurrently on the worker threads.
    Returns (out = [lambda, ||H y - beta e1||, degenerate, rank_def], y)."""
    k = H.shape[1]
    out = np.empty(4)
    y = np.empty(k)
    _native.check(lib.ctk_projected_solve(H.ctypes.data, k, float(beta), code,
                                          float(value or 0.0), 200, float(fallback),
                                          out.ctypes.data, y.ctypes.data), "ctk_projected_solve")
    return out, y


_TP_CONTROLLER = []


def _blas_single_thread():
    """Single-threaded BLAS for the driver's worker threads (their projected
    solves are tiny; a threaded BLAS would oversubscribe the host).  The
    threadpoolctl controller scans the loaded libraries once (~5 ms), then
    each limit costs ~20 us."""
    import contextlib
    if not _TP_CONTROLLER:
        try:
            from threadpoolctl import ThreadpoolController
            _TP_CONTROLLER.append(ThreadpoolController())
        except Exception:   # pragma: no cover
            _TP_CONTROLLER.append(None)
    ctl = _TP_CONTROLLER[0]
    return ctl.limit(limits=1, user_api="blas") if ctl is not None else contextlib.nullcontext()


class _DeviceSolve:
    """One run_gmres call.

    Streams: ``sa`` runs the Arnoldi process ahead (LOOKAHEAD steps in
    flight; each step needs only w_k, never lambda); ``sb`` runs the iterate
    updates x_k = x0 + (B) W y_k and true residuals as the host hands over
    each y_k.  Host worker threads solve the projected problems of different
    iterations concurrently; results are consumed strictly in iteration order
    (the degenerate-curve fallback needs the previous lambda).
    """

    LOOKAHEAD = int(os.environ.get("CTK_LOOKAHEAD", "6"))   # tuning override

    def __init__(self, A, B, b, cfg, x_true, image_shape, stream, timer, keep_on_device=False):
        if not isinstance(A, GpuForward) or not isinstance(B, GpuBack) or A.dgeom is not B.dgeom:
            raise TypeError("the device-resident run_gmres needs the GPU projector pair from "
                            "paper_2602_17892_b200.ct (forward_ray_driven / back_pixel_driven "
                            "on one geometry)")
        self.A, self.B, self.cfg = A, B, cfg
        dg = self.dg = A.dgeom
        torch = self.torch = dg.torch
        self.caller = stream if stream is not None else torch.cuda.current_stream(dg.dev)
        self.sa = _side_stream(torch, dg.dev, "arnoldi", -100)
        self.sb = _side_stream(torch, dg.dev, "combine", 100)
        self.sa.wait_stream(self.caller)
        self.lib = _native.load()
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
        with torch.cuda.stream(self.sa):
            if torch.is_tensor(b):
                if b.numel() != self.m:
                    raise OperatorShapeError(f"data vector has {b.numel()} entries, expected {self.m}")
                self.b = b.to(device=dev, dtype=f32).contiguous()
            else:
                bh = np.asarray(b, dtype=np.float64)
                if bh.shape != (self.m,):
                    raise OperatorShapeError(f"data vector has shape {bh.shape}, expected ({self.m},)")
                bp = _pinned(torch, "b", (self.m,), torch.float32, zero=False)
                bp.numpy()[:] = bh                          # fp64 -> fp32 into page-locked memory
                self.b = torch.empty(self.m, dtype=f32, device=dev)
                self.b.copy_(bp, non_blocking=True)
                self.h2d += 4 * self.m
            ws = _solve_workspace(torch, dg, self.ab, L, rows, self.K)
            self.basis = ws["basis"]
            x0 = cfg.x0
            if x0 is None:
                self.x_cur = ws["x_cur"]
                self.x_cur.zero_()
            else:
                x0 = np.asarray(x0, dtype=np.float64)
                if x0.shape != (self.n,):
                    raise ConfigError(f"x0 has shape {x0.shape}, expected ({self.n},)")
                self.x_cur = torch.from_numpy(x0.astype(np.float32)).to(dev)
                self.h2d += 4 * self.n
            # stream sa (Arnoldi) buffers
            self.q, self.tmp, self.hs, self.scal = ws["q"], ws["tmp"], ws["hs"], ws["scal"]
            self.hcols = rows + 1 + 4                      # h[0..rows] + 4 stats
            self.h_host = _pinned(torch, "h", (rows, self.hcols), f64)
            self.scal_host = _pinned(torch, "scal", (4,), f64)
            # stream sb (iterate) buffers; rows kept by each Arnoldi step so
            # iterates follow by linearity (ctk_iterate): BA keeps A w_j, AB
            # keeps B w_j and A B w_j
            self.xk, self.z, self.r = ws["xk"], ws["z"], ws["r"]
            self.aux1, self.aux2, self.d0 = ws["aux1"], ws["aux2"], ws["d0"]
            self.y_dev, self.norms = ws["y_dev"], ws["norms"]
            self.y_pin = _pinned(torch, "y", (self.K, rows), f64)
        self.ev_h = [None] * rows
        # the side stream must not touch buffers before their zero-fill lands
        self.sb.wait_stream(self.sa)

    # -- projector launches (optionally event-bracketed) ------------------
    def _fwd(self, x, out, stream, b=None):
        if self.timer is None:
            return self.dg.forward(x, out=out, b=b, stream=stream)
        e1 = self.timer.bracket("forward", stream)
        self.dg.forward(x, out=out, b=b, stream=stream)
        e1.record(stream)

    def _back(self, u, out, stream, x0=None):
        if self.timer is None:
            return self.dg.back(u, out=out, x0=x0, stream=stream)
        e1 = self.timer.bracket("back", stream)
        self.dg.back(u, out=out, x0=x0, stream=stream)
        e1.record(stream)

    def _aux(self):
        """(aux1, ld1, aux2, ld2) pointers for the native step / iterate calls."""
        a2 = self.aux2
        return (self.aux1.data_ptr(), self.aux1.shape[1],
                None if a2 is None else a2.data_ptr(), 0 if a2 is None else a2.shape[1])

    def _work(self, stream):
        """(stage, back) workspaces of one stream for the native calls."""
        dg = self.dg
        stage = dg._workspace("stage", dg.stage_floats, stream)
        wf = int(self.lib.ctk_back_work_floats(dg.handle, 0, dg.n_angles))
        back = dg._workspace("back", wf, stream) if wf > 0 else None
        return stage.data_ptr(), _native.ptr(back)

    def _arnoldi(self, j):
        """Enqueue step j on sa: q = M w_j, CGS2 -> h column + w_{j+1}; D2H h."""
        torch, sa = self.torch, self.sa
        stage, back = self._work(sa)
        hrow = self.hs[j]
        _native.check(self.lib.ctk_arnoldi_step(
            self.dg.handle, int(self.ab), 2 if self.cfg.reorthogonalize else 1,
            self.basis.W.data_ptr(), self.basis.ld, j,
            self.q.data_ptr(), self.tmp.data_ptr(), *self._aux(), stage, back, hrow.data_ptr(),
            self.hcols,
            self.h_host[j].data_ptr(), self.basis.scratch(sa), sa.cuda_stream), "ctk_arnoldi_step")
        self.d2h += 8 * self.hcols
        ev = torch.cuda.Event()
        ev.record(sa)
        self.ev_h[j] = ev

    def _iterate(self, it, k, y, after):
        """Enqueue on sb: x_k = x0 + (B) W y, r = b - A x_k, norms -> slot it."""
        torch, sb = self.torch, self.sb
        sb.wait_event(after)
        self.y_pin[it, :k] = torch.from_numpy(y)
        self.h2d += 8 * k
        stage, back = self._work(sb)
        _native.check(self.lib.ctk_iterate(
            self.dg.handle, int(self.ab), self.basis.W.data_ptr(), self.basis.ld, k,
            self.y_pin[it].data_ptr(), self.y_dev[it].data_ptr(), self.x_cur.data_ptr(),
            self.xk.data_ptr(), _native.ptr(self.z), self.b.data_ptr(), self.r.data_ptr(),
            self.norms[it].data_ptr(), *self._aux(), self.d0.data_ptr(), stage, back,
            self.basis.scratch(sb), sb.cuda_stream), "ctk_iterate")
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(sb)
        return ev

    def _ncp_distance(self, r, stream) -> float:
        """NCP distance of the residual on the device (cuFFT via torch.fft,
        fp64): the KS distance of its normalised cumulative periodogram from
        the white-noise diagonal, ctkrylov/stopping.py:27-46.  Only the scalar
        crosses PCIe (the reference ships the m-length residual to numpy)."""
        torch = self.torch
        m = r.numel()
        if m < 8:
            raise ValueError(f"NCP needs a residual of length >= 8, got {m}")
        with torch.cuda.stream(stream):
            power = torch.fft.rfft(r.to(torch.float64)).abs().square()
            q = m // 2
            power = power[1: q + 1]
            total = power.sum()
            c = torch.cumsum(power, 0) / total
            diag = torch.arange(1, q + 1, dtype=torch.float64, device=r.device) / q
            dist = torch.where(total > 0, (c - diag).abs().max(), torch.zeros_like(total))
            out = dist.to("cpu", non_blocking=True)
        stream.synchronize()
        self.d2h += 8
        return float(out)

    def _host_vec(self, t, stream):
        """fp64 numpy copy of a device fp32 vector: one D2H into a reused
        page-locked buffer (no pageable staging), widened on the host."""
        self.d2h += 4 * t.numel()
        pin = _pinned(self.torch, "xout", (t.numel(),), self.torch.float32, zero=False)
        with self.torch.cuda.stream(stream):
            pin.copy_(t, non_blocking=True)
        stream.synchronize()
        return pin.numpy().astype(np.float64)

    def _cycle_start(self):
        """r0 = b - A x (AB) or B(b - A x) (BA) into W row 0; returns (beta, ||d0||)."""
        torch, sa = self.torch, self.sa
        w0 = self.basis.row(0)
        if self.ab:
            self._fwd(self.x_cur, w0, sa, b=self.b)
            self.basis.norm2(w0, self.scal[0:1], sa)
        else:
            self._fwd(self.x_cur, self.tmp, sa, b=self.b)
            self.basis.norm2(self.tmp, self.scal[1:2], sa)
            self._back(self.tmp, w0, sa)
            self.basis.norm2(w0, self.scal[0:1], sa)
        with torch.cuda.stream(sa):
            self.d0[: self.m].copy_(w0 if self.ab else self.tmp)     # d0 = b - A x0
            self.scal_host.copy_(self.scal, non_blocking=True)
        self.d2h += 32
        sa.synchronize()
        beta = float(np.sqrt(self.scal_host[0].item()))
        d0n = beta if self.ab else float(np.sqrt(self.scal_host[1].item()))
        return beta, d0n

    def run(self) -> SolveResult:
        with _blas_single_thread():
            return self._run()

    def _run(self) -> SolveResult:
        torch, cfg = self.torch, self.cfg
        sa, sb = self.sa, self.sb
        K, p = self.K, self.p
        pool = _pool()
        records: list[IterationRecord] = []
        pending: list[tuple] = []          # (record, slot, event) awaiting norms
        history: list[float] = []
        snapshots: dict[int, np.ndarray] = {}
        stop = None
        cycles = 0
        state = {"prev_lam": 0.0}
        need_sync = cfg.stopping_rule != "none" or self.x_true is not None
        ev_start = torch.cuda.Event(enable_timing=True)
        ev_start.record(sa)
        sb.wait_event(ev_start)
        t_start = time.perf_counter()
        last_ev = None
        first_cycle = True
        while stop is None and len(records) < K:
            if not first_cycle:
                sa.wait_stream(sb)
                with torch.cuda.stream(sa):
                    self.x_cur.copy_(self.xk)
            first_cycle = False
            beta, d0n = self._cycle_start()
            if beta == 0.0:
                stop = "breakdown"
                if not records:
                    x_host = self._host_vec(self.x_cur, sa)
                    records.append(self._make_record(0, 0.0, 0.0, d0n, 0.0,
                                                     float(np.linalg.norm(x_host)), x_host,
                                                     time.perf_counter() - t_start))
                break
            cycles += 1
            with torch.cuda.stream(sa):
                self.scal[2] = 1.0 / beta
            self.basis.scale_into(self.basis.row(0), self.basis.row(0), self.scal[2:3], sa)
            sb.wait_stream(sa)                     # x_cur / W0 ready for the iterate stream

            steps = min(p, K - len(records))
            code = _native.STRATEGY_CODES[cfg.lambda_strategy] if self.hybrid else 0
            Hfull = np.zeros((steps + 1, steps))     # grows one column per step
            queued = 0                             # Arnoldi steps enqueued on sa
            futures: dict[int, tuple] = {}
            done_k = 0                             # iterates handed to sb
            last_k = steps
            broke_at = None

            def enqueue_to(n):
                nonlocal queued
                while queued < min(n, steps):
                    self._arnoldi(queued)
                    queued += 1

            def consume(k):
                """Iterate k (1-based in this cycle), strictly in order."""
                nonlocal stop, last_ev
                H, fut = futures.pop(k)
                out, y = fut.result()
                warn = False
                if not self.hybrid:
                    lam = 0.0
                elif out[2] != 0.0:        # DegenerateCurveError: previous lambda (gmres.py:196-200)
                    lam, warn = state["prev_lam"], True
                    out, y = _projected_task(self.lib, H, beta, 1, lam)
                else:
                    lam = float(out[0])
                state["prev_lam"] = lam
                proj_res = float(out[1])
                slot = len(records)
                ev = self._iterate(slot, k, y, self.ev_h[k - 1])
                last_ev = ev
                rec = IterationRecord(k=slot + 1, lambda_used=float(lam), residual_norm=0.0,
                                      data_residual_norm=0.0,
                                      proj_residual_norm=proj_res,
                                      solution_norm=0.0, lambda_warning=warn)
                records.append(rec)
                if cfg.snapshot_stride and rec.k % cfg.snapshot_stride == 0:
                    snapshots[rec.k] = self._host_vec(self.xk, sb)
                if need_sync:
                    ev.synchronize()
                    self._finish(rec, slot, ev_start, ev)
                    history.append(rec.data_residual_norm)
                    if self.x_true is not None:
                        self._metrics(rec, self._host_vec(self.xk, sb))
                    if cfg.stopping_rule == "dp" and metrics.dp_should_stop(
                            rec.data_residual_norm, cfg.noise_norm, cfg.dp_tau):
                        stop = "dp"
                    elif cfg.stopping_rule == "ncp" and (
                            self._ncp_distance(self.r, sb) <= cfg.ncp_threshold):
                        stop = "ncp"
                    elif cfg.stopping_rule == "rns" and metrics.rns_should_stop(
                            history, cfg.rns_epsilon):
                        stop = "rns"
                else:
                    pending.append((rec, slot, ev))
                if broke_at is not None and k == broke_at and stop is None:
                    stop = "breakdown"

            enqueue_to(self.LOOKAHEAD)
            for j in range(steps):
                self.ev_h[j].synchronize()
                hrow = self.h_host[j].numpy()
                k = j + 1
                Hfull[: j + 2, j] = hrow[: j + 2]
                broke = hrow[self.hcols - 3] != 0.0
                H = Hfull[: k + 1, :k].copy()
                futures[k] = (H, pool.submit(_projected_task, self.lib, H, beta, code,
                                             cfg.lambda_value))
                if broke:
                    broke_at = last_k = k
                else:
                    enqueue_to(k + self.LOOKAHEAD)
                # hand finished projected solves to the iterate stream, in order
                while stop is None and done_k + 1 in futures and (
                        need_sync or futures[done_k + 1][1].done()):
                    done_k += 1
                    consume(done_k)
                if stop is not None or broke:
                    break
            while stop is None and done_k < last_k and done_k + 1 in futures:
                done_k += 1
                consume(done_k)
            if stop is None and broke_at is not None:
                stop = "breakdown"
        sa.synchronize()
        sb.synchronize()
        self.caller.wait_stream(sa)
        self.caller.wait_stream(sb)
        if pending:
            norms = self.norms.cpu().numpy()
            self.d2h += self.norms.numel() * 8
            for rec, slot, ev in pending:
                self._finish(rec, slot, ev_start, ev, norms)
        x_final = self.xk if records and records[-1].k > 0 else self.x_cur
        x_out = x_final.clone() if self.keep_on_device else self._host_vec(x_final, sb)
        res = SolveResult(x=x_out, records=records, stop_reason=stop or "maxiter",
                          cycles=max(cycles, 1), snapshots=snapshots)
        res.transfer = {"h2d_bytes": self.h2d, "d2h_bytes": self.d2h}
        return res

    def _finish(self, rec, slot, ev_start, ev, norms=None):
        if norms is None:
            row = self.norms[slot].cpu().numpy()
            self.d2h += 16
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


class _NativeSolve(_DeviceSolve):
    """run_gmres entirely in libctk's C++ driver (ctk_solve): no Python work
    per iteration.  Used when no per-iteration host data is requested
    (x_true metrics, snapshots, ncp stopping)."""

    def run(self) -> SolveResult:
        torch, cfg = self.torch, self.cfg
        dg, K = self.dg, self.K
        rows = self.basis.rows
        n1 = K + 1
        out_arrays = {
            "k": np.zeros(n1, dtype=np.int32), "warn": np.zeros(n1, dtype=np.int32),
            "lambda_": np.zeros(n1), "residual": np.zeros(n1), "data_residual": np.zeros(n1),
            "proj_residual": np.zeros(n1), "solution_norm": np.zeros(n1), "elapsed": np.zeros(n1)}
        norms_host = _pinned(torch, "norms", ((K + 1) * 2,), torch.float64)
        cfgc = _native.SolveCfg(
            ab=int(self.ab), hybrid=int(self.hybrid),
            strategy=_native.STRATEGY_CODES.get(cfg.lambda_strategy, 0),
            max_iter=K, restart_period=cfg.restart_period,
            stopping=_native.STOP_CODES[cfg.stopping_rule], lookahead=self.LOOKAHEAD,
            lambda_value=float(cfg.lambda_value or 0.0), dp_tau=float(cfg.dp_tau),
            noise_norm=float(cfg.noise_norm or 0.0), rns_epsilon=float(cfg.rns_epsilon),
            reorthogonalize=int(bool(cfg.reorthogonalize)))
        sa, sb = self.sa, self.sb
        stage_a, back_a = self._work(sa)
        stage_b, back_b = self._work(sb)
        P = _native.ptr
        bufs = _native.SolveBufs(
            W=self.basis.W.data_ptr(), ld=self.basis.ld, rows=rows,
            q=self.q.data_ptr(), tmp=self.tmp.data_ptr(), z=P(self.z), r=self.r.data_ptr(),
            xk=self.xk.data_ptr(), x_cur=self.x_cur.data_ptr(), b=self.b.data_ptr(),
            aux1=self.aux1.data_ptr(), ld1=self.aux1.shape[1],
            aux2=P(self.aux2), ld2=0 if self.aux2 is None else self.aux2.shape[1],
            d0=self.d0.data_ptr(),
            hs=self.hs.data_ptr(), h_host=self.h_host.data_ptr(), hcols=self.hcols,
            y_dev=self.y_dev.data_ptr(), y_host=self.y_pin.data_ptr(),
            norms=self.norms.data_ptr(), norms_host=norms_host.data_ptr(),
            scal=self.scal.data_ptr(), scal_host=self.scal_host.data_ptr(),
            stage_a=stage_a, back_a=back_a, stage_b=stage_b, back_b=back_b,
            scratch_a=self.basis.scratch(sa), scratch_b=self.basis.scratch(sb),
            stream_a=sa.cuda_stream, stream_b=sb.cuda_stream,
            comm=None if getattr(self, "comm", None) is None else self.comm.handle.value)
        # optional per-iteration records computed on the device (row f1)
        out_arrays["rre"] = np.full(n1, np.nan)
        out_arrays["ssim"] = np.full(n1, np.nan)
        keep = []                                  # keep buffers alive across the call
        if self.x_true is not None:
            xt = torch.from_numpy(self.x_true.astype(np.float32)).to(dg.dev)
            met = torch.zeros((K + 1) * 2, dtype=torch.float64, device=dg.dev)
            met_h = _pinned(torch, "metrics", ((K + 1) * 2,), torch.float64)
            scr = torch.zeros(int(self.lib.ctk_metrics_scratch_bytes()) // 8 + 1,
                              dtype=torch.float64, device=dg.dev)
            keep += [xt, met, met_h, scr]
            shape = self.image_shape
            use_ssim = shape is not None and min(shape) >= 8
            dyn = float(self.x_true.max() - self.x_true.min()) if use_ssim else 0.0
            bufs.x_true, bufs.metrics, bufs.metrics_host = xt.data_ptr(), met.data_ptr(), met_h.data_ptr()
            bufs.scratch_m = scr.data_ptr()
            bufs.img_ny, bufs.img_nx = (int(shape[0]), int(shape[1])) if use_ssim else (0, 0)
            bufs.dyn_range = dyn
        snaps = []
        if cfg.snapshot_stride:
            nsn = K // cfg.snapshot_stride
            snaps = [torch.empty(self.n, dtype=torch.float32).pin_memory() for _ in range(nsn)]
            arr = (ctypes.c_void_p * max(nsn, 1))(*[t.data_ptr() for t in snaps])
            keep.append(arr)
            bufs.snapshot_stride, bufs.snaps, bufs.n_snaps = cfg.snapshot_stride, ctypes.addressof(arr), nsn
        outc = _native.SolveOut(**{k: v.ctypes.data for k, v in out_arrays.items()})
        with _blas_single_thread():
            _native.check(self.lib.ctk_solve(dg.handle, ctypes.byref(cfgc), ctypes.byref(bufs),
                                             ctypes.byref(outc)), "ctk_solve")
        self.caller.wait_stream(sa)
        self.caller.wait_stream(sb)
        nrec = outc.n_records
        self.d2h += 8 * self.hcols * nrec + 16 * (K + 1) + 32
        self.h2d += sum(8 * int(k) for k in out_arrays["k"][:nrec])
        cols = [out_arrays[f][:nrec].tolist() for f in
                ("k", "lambda_", "residual", "data_residual", "proj_residual", "solution_norm")]
        el = out_arrays["elapsed"][:nrec].tolist()
        wn = out_arrays["warn"][:nrec].tolist()
        records = [IterationRecord(kk, lam, rn, dn, pn, sn, None, None, e, bool(w))
                   for kk, lam, rn, dn, pn, sn, e, w in zip(*cols, el, wn)]
        if self.x_true is not None:
            xn = float(np.linalg.norm(self.x_true))
            shape = self.image_shape
            cnt = (shape[0] - 7) * (shape[1] - 7) if shape is not None and min(shape) >= 8 else 0
            for i, rec in enumerate(records):
                if rec.k == 0:
                    continue
                rec.rre = float(np.sqrt(out_arrays["rre"][i]) / xn) if xn > 0 else None
                if cnt and bufs.dyn_range > 0:
                    rec.ssim = float(out_arrays["ssim"][i] / cnt)
        snapshots = {}
        for i, t in enumerate(snaps):
            kk = (i + 1) * cfg.snapshot_stride
            if kk <= nrec:
                snapshots[kk] = t.numpy().astype(np.float64)
        self.d2h += 4 * self.n * len(snapshots)
        x_final = self.x_cur if outc.x_is_x0 else self.xk
        x_out = x_final.clone() if self.keep_on_device else self._host_vec(x_final, sb)
        res = SolveResult(x=x_out, records=records,
                          stop_reason=_native.STOP_NAMES.get(outc.stop_reason, "maxiter"),
                          cycles=outc.cycles, snapshots=snapshots)
        res.transfer = {"h2d_bytes": self.h2d, "d2h_bytes": self.d2h}
        return res


def run_gmres(A: LinearOperator, B: LinearOperator, b, cfg: SolverConfig,
              x_true: np.ndarray | None = None, image_shape: tuple[int, int] | None = None,
              *, stream=None, keep_on_device: bool = False, comm=None) -> SolveResult:
    """(Hybrid) AB-/BA-GMRES with optional restarting, on the GPU.

    ``b`` may be a host array (the reference's contract) or a CUDA tensor
    (device-resident input).  Returns a SolveResult with a host ``x`` (a CUDA
    tensor when ``keep_on_device``); ``result.transfer`` counts the bytes the
    solve moved across PCIe.

    ``comm`` (a :class:`paper_2602_17892_b200.dist.NativeComm`): angle-sharded
    solve on the native driver -- A, B are this rank's angle subset, ``b`` its
    sinogram rows; the iterate is replicated on every rank.
    """
    cfg.validate()
    if cfg.method not in GMRES_METHODS:
        raise ConfigError(f"run_gmres got non-GMRES method {cfg.method!r}")
    shape = tuple(b.shape)
    if len(shape) != 1:
        raise OperatorShapeError(f"data vector has shape {shape}, expected ({A.rows},)")
    _check_dims(A, B, int(shape[0]))
    native = cfg.stopping_rule != "ncp" and os.environ.get("CTK_PY_DRIVER", "0") != "1"
    if comm is not None and not native:
        raise ConfigError("the angle-sharded solve runs on the native driver "
                          "(no ncp stopping, CTK_PY_DRIVER unset)")
    cls = _NativeSolve if native else _DeviceSolve
    solver = cls(A, B, b, cfg, x_true, image_shape, stream, None, keep_on_device)
    solver.comm = comm
    return solver.run()


def run_ab_gmres(A, B, b, cfg: SolverConfig, **kwargs) -> SolveResult:
    if not cfg.method.startswith("ab"):
        cfg = replace(cfg, method="ab-hybrid" if cfg.lambda_strategy != "none" else "ab")
    return run_gmres(A, B, b, cfg, **kwargs)


def run_ba_gmres(A, B, b, cfg: SolverConfig, **kwargs) -> SolveResult:
    if not cfg.method.startswith("ba"):
        cfg = replace(cfg, method="ba-hybrid" if cfg.lambda_strategy != "none" else "ba")
    return run_gmres(A, B, b, cfg, **kwargs)
