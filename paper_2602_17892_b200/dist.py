"""Multi-GPU hybrid GMRES: angle sharding over NCCL.

One process per GPU (torchrun), ``torch.distributed`` with NCCL over
NVLink/NVSwitch.  Work is split by projection angle:

* A is angle-sharded with a replicated image: each rank projects its own
  sinogram rows, no communication.
* B produces a partial image per rank (the rank's angles only), summed over
  ranks by :class:`PeerExchange` -- K2 pushes finished tiles to their owner
  over NVLink peer memory, the owner reduces in rank order and delivers --
  or, where the ranks cannot map each other's memory, one NCCL all-reduce
  (sum, fp32, n values).
* AB-GMRES: Krylov vectors live in measurement space and are sharded with
  the angles; every dot product / norm is a local partial plus one batched
  fp64 all-reduce per CGS2 sweep (h1 with ||q||^2, h2, ||q2||^2).
* BA-GMRES: Krylov vectors live in image space and are replicated; the only
  collective is B's partial-image all-reduce.
* The (k+1) x k Hessenberg, lambda selection and Tikhonov solve stay on the
  host in fp64 and are computed redundantly on every rank from bitwise
  identical all-reduced inputs, so no broadcast is needed.
* Independent slices (the c5 batch) need none of this: each rank runs the
  single-GPU driver on its own slices (bench.py's weak-scaling mode).

Two drivers share this decomposition: :class:`NativeComm` +
``gmres.run_gmres(..., comm=)`` run it in libctk's C++ driver (collectives
issued from C++, stream-ordered on the Arnoldi stream, iterates by
linearity: one A and one B apply per Arnoldi step, as on one GPU) -- the
production path and ``bench.py --shard angles``; :func:`run_gmres_sharded`
is the same algorithm in Python over a small backend interface, which the
CPU test suite runs on a world_size-2 gloo group.

The driver below is written against a small backend interface so that the
same sharding logic runs on the GPU (:class:`CudaShardBackend`: libctk
kernels + NCCL) and, in the CPU test suite, on a world_size-2 gloo group
with a host backend supplied by the tests.
"""

from __future__ import annotations

import time

import numpy as np

from .gmres import (GMRES_METHODS, ConfigError, IterationRecord, SolveResult, SolverConfig)
from . import metrics
from .arnoldi import solve_projected_tikhonov, hessenberg_from_columns
from .regparam import DegenerateCurveError, select_lambda, svd_of_hessenberg


def angle_shards(n_angles: int, world: int, mode: str = "interleaved") -> list[np.ndarray]:
    """Angle indices owned by each rank.

    "interleaved" (a = r mod world) balances the per-angle cost, which varies
    with |cos| + |sin| (segments per ray); "blocks" gives contiguous ranges.
    Every rank owns at least one angle.
    """
    if world < 1 or n_angles < world:
        raise ValueError(f"cannot shard {n_angles} angles over {world} ranks")
    idx = np.arange(n_angles)
    if mode == "interleaved":
        return [idx[r::world] for r in range(world)]
    if mode == "blocks":
        return [a for a in np.array_split(idx, world)]
    raise ValueError(f"unknown shard mode {mode!r}")


class ShardBackend:
    """Interface of the sharded driver.

    Vectors are backend arrays; the Krylov basis is owned by the backend
    (``basis_*``), rows 0..k addressed by index.  Small fp64 messages go
    through ``from_host_f64`` / ``allreduce`` / ``to_host_f64``.
    """

    n: int          # image size (replicated)
    m_local: int    # this rank's sinogram rows * det_count

    def zeros(self, size): raise NotImplementedError
    def from_host(self, arr): raise NotImplementedError
    def to_host(self, v): raise NotImplementedError
    def from_host_f64(self, arr): raise NotImplementedError
    def to_host_f64(self, v): raise NotImplementedError
    def forward(self, x): raise NotImplementedError               # image -> local sinogram
    def back_partial(self, u): raise NotImplementedError          # local sinogram -> partial image
    def allreduce(self, v): raise NotImplementedError             # in-place sum over ranks

    def back_sum(self, u):                                        # sum over ranks of B_r u_r
        img = self.back_partial(u)
        self.allreduce(img)
        return img

    def norm2(self, v): raise NotImplementedError                 # fp64 scalar (local part)
    def scale(self, v, a): raise NotImplementedError
    def add(self, a, b): raise NotImplementedError
    def sub(self, a, b): raise NotImplementedError
    # Krylov basis
    def basis_init(self, L, rows): raise NotImplementedError
    def basis_set(self, j, v, scale): raise NotImplementedError   # row j = v * scale
    def basis_row(self, j): raise NotImplementedError
    def basis_dots(self, k, v, want_norm): raise NotImplementedError   # host fp64, k (+1)
    def basis_update(self, k, coef, v): raise NotImplementedError      # v - sum coef_j W_j
    def basis_combine(self, k, y): raise NotImplementedError           # sum y_j W_j


def _allreduce_host(be, values) -> np.ndarray:
    """All-reduce a small fp64 host vector through the backend (one message)."""
    v = be.from_host_f64(np.asarray(values, dtype=np.float64))
    be.allreduce(v)
    return be.to_host_f64(v)


def run_gmres_sharded(be: ShardBackend, b_local, cfg: SolverConfig, x0=None) -> SolveResult:
    """(Hybrid) AB-/BA-GMRES over an angle-sharded projector pair.

    Same configuration, records and stop reasons as the single-GPU driver
    (ctkrylov/gmres.py:135-241).  ``b_local`` is this rank's slice of the data
    (its angles' rows).  Returns the replicated iterate on every rank.
    """
    cfg.validate()
    if cfg.method not in GMRES_METHODS:
        raise ConfigError(f"run_gmres got non-GMRES method {cfg.method!r}")
    ab = cfg.method.startswith("ab")
    hybrid = cfg.method.endswith("-hybrid")
    b = be.from_host(b_local) if isinstance(b_local, np.ndarray) else b_local
    x = be.zeros(be.n) if x0 is None else be.from_host(np.asarray(x0, dtype=np.float64))
    K = cfg.max_iter
    p = cfg.restart_period if cfg.restart_period > 0 else K

    def back_full(u):
        return be.back_sum(u)                 # N1: partial images summed over ranks

    def gdots(k, v, want_norm):               # global dots: local partial + one all-reduce
        loc = be.basis_dots(k, v, want_norm)
        return _allreduce_host(be, loc) if ab else loc

    def gnorm2(v):
        loc = be.norm2(v)
        return float(_allreduce_host(be, [loc])[0]) if ab else loc

    rows = min(p, K) + 1
    be.basis_init(be.m_local if ab else be.n, rows)
    records: list[IterationRecord] = []
    history: list[float] = []
    stop = None
    cycles = 0
    prev_lam = 0.0
    t0 = time.perf_counter()
    while stop is None and len(records) < K:
        d0 = be.sub(b, be.forward(x))                          # local rows of b - A x
        r0 = d0 if ab else back_full(d0)
        beta = float(np.sqrt(gnorm2(r0)))
        if beta == 0.0:
            stop = "breakdown"
            if not records:
                dn = float(np.sqrt(_allreduce_host(be, [be.norm2(d0)])[0]))
                records.append(IterationRecord(0, 0.0, 0.0, dn, 0.0,
                                               float(np.sqrt(be.norm2(x))),
                                               elapsed=time.perf_counter() - t0))
            break
        cycles += 1
        be.basis_set(0, r0, 1.0 / beta)
        cols: list[np.ndarray] = []
        xc = x
        for _ in range(min(p, K - len(records))):
            k = len(cols)
            w = be.basis_row(k)
            q = be.forward(back_full(w)) if ab else back_full(be.forward(w))
            # CGS2 with batched all-reduces: [h1, ||q||^2], h2, ||q2||^2
            h1n = gdots(k + 1, q, True)
            h1, qn = h1n[:-1], float(np.sqrt(h1n[-1]))
            q = be.basis_update(k + 1, h1, q)
            h2 = gdots(k + 1, q, False)
            q = be.basis_update(k + 1, h2, q)
            hk = float(np.sqrt(gnorm2(q)))
            col = np.empty(k + 2)
            col[: k + 1] = h1 + h2
            col[k + 1] = hk
            cols.append(col)
            k += 1
            broke = hk <= 1e-14 * qn
            if not broke:
                be.basis_set(k, q, 1.0 / hk)
            H = hessenberg_from_columns(cols, k)
            svd = svd_of_hessenberg(H)
            warn = False
            if hybrid:
                try:
                    lam = select_lambda(H, beta, cfg.lambda_strategy, cfg.lambda_value, svd=svd)
                except DegenerateCurveError:
                    lam, warn = prev_lam, True
            else:
                lam = 0.0
            prev_lam = lam
            sol = solve_projected_tikhonov(H, beta, lam, svd=svd)
            z = be.basis_combine(k, sol.y)
            xk = be.add(xc, back_full(z) if ab else z)
            r = be.sub(b, be.forward(xk))
            dn = float(np.sqrt(_allreduce_host(be, [be.norm2(r)])[0]))
            rec = IterationRecord(k=len(records) + 1, lambda_used=float(lam),
                                  residual_norm=dn if ab else sol.proj_residual_norm,
                                  data_residual_norm=dn,
                                  proj_residual_norm=sol.proj_residual_norm,
                                  solution_norm=float(np.sqrt(be.norm2(xk))),
                                  elapsed=time.perf_counter() - t0, lambda_warning=warn)
            records.append(rec)
            history.append(dn)
            x = xk
            if cfg.stopping_rule == "dp" and metrics.dp_should_stop(dn, cfg.noise_norm, cfg.dp_tau):
                stop = "dp"
            elif cfg.stopping_rule == "rns" and metrics.rns_should_stop(history, cfg.rns_epsilon):
                stop = "rns"
            elif cfg.stopping_rule == "ncp":
                raise ConfigError("ncp stopping needs the gathered residual; use the single-GPU driver")
            if broke and stop is None:
                stop = "breakdown"
            if stop is not None:
                break
    return SolveResult(x=be.to_host(x), records=records, stop_reason=stop or "maxiter",
                       cycles=max(cycles, 1))


class _DeviceArray:
    """__cuda_array_interface__ over a libctk-owned fp32 buffer (zero copy)."""

    def __init__(self, ptr: int, n: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f4", "data": (ptr, False),
                                         "version": 3, "strides": None}


class PeerExchange:
    """Angle-sharded B summed over peer memory (``ctk_back_exchange``).

    Each rank's K2 pushes its finished partial tiles into the tile owner's
    receive buffer (NVLink peer stores), the owner sums them in rank order and
    delivers the tile to every rank -- the N1 all-reduce fused into the
    back-projection (see csrc/ctk_exchange.cu).  ``img`` is the exchange's
    result buffer (overwritten by the next call).  Connect with
    :meth:`connect_ipc` across processes (handles gathered over
    torch.distributed) or :meth:`connect_local` in one process.
    """

    def __init__(self, dgeom, rank: int, nranks: int):
        import ctypes
        from . import _native
        self._native, self._ct = _native, ctypes
        self.lib = _native.load()
        self.dg = dgeom
        h = ctypes.c_void_p()
        _native.check(self.lib.ctk_xchg_create(dgeom.handle, rank, nranks, ctypes.byref(h)),
                      "ctk_xchg_create")
        self.handle = h
        self.rank, self.nranks = rank, nranks
        r, x, f = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(self.lib.ctk_xchg_local(h, ctypes.byref(r), ctypes.byref(x), ctypes.byref(f)))
        self.local_ptrs = (r.value, x.value, f.value)
        torch = dgeom.torch
        self.img = torch.as_tensor(_DeviceArray(x.value, dgeom.n), device=dgeom.dev)
        self.epoch = 0
        wf = int(self.lib.ctk_back_work_floats(dgeom.handle, 0, dgeom.n_angles))
        self.work = torch.zeros(max(wf, 4), dtype=torch.float32, device=dgeom.dev)

    def export(self) -> bytes:
        buf = self._ct.create_string_buffer(int(self.lib.ctk_xchg_handle_bytes()))
        self._native.check(self.lib.ctk_xchg_export(self.handle, buf), "ctk_xchg_export")
        return buf.raw

    def connect_ipc(self, handles: list) -> None:
        blob = b"".join(handles)
        self._native.check(self.lib.ctk_xchg_connect_ipc(self.handle, blob), "ctk_xchg_connect_ipc")

    def connect_local(self, peers: list) -> None:
        ct = self._ct
        arr = [(ct.c_void_p * self.nranks)(*[p.local_ptrs[i] for p in peers]) for i in range(3)]
        self._native.check(self.lib.ctk_xchg_connect_ptrs(self.handle, *arr), "ctk_xchg_connect_ptrs")

    def back(self, u, phases: int = 7, epoch: int | None = None, stream=None):
        """img = sum over ranks of B_rank u_rank (this rank's phases)."""
        if epoch is None:
            self.epoch += 1
            epoch = self.epoch
        self.dg._check(u, self.dg.m, "u")
        stream = self.dg._stream(stream)
        self._native.check(self.lib.ctk_back_exchange(self.dg.handle, self.handle, u.data_ptr(),
                                                      epoch, phases, self.work.data_ptr(),
                                                      stream.cuda_stream), "ctk_back_exchange")
        return self.img

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.ctk_xchg_destroy(h)
            except Exception:
                pass
            self.handle = None


def nccl_library() -> str | None:
    """Path of the libnccl.so.2 torch uses (libctk loads the same instance)."""
    import os
    try:
        import nvidia.nccl
        for base in getattr(nvidia.nccl, "__path__", []):
            p = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(p):
                return p
    except Exception:
        pass
    return None


def open_peer_exchange(dgeom, group=None):
    """PeerExchange over CUDA IPC among the ranks of `group`, or None when any
    rank cannot create or map the buffers (every rank agrees)."""
    import torch
    import torch.distributed as tdist
    world = tdist.get_world_size(group)
    rank = tdist.get_rank(group)
    if not 1 < world <= 8:
        return None
    ok, ex, mine = True, None, b""
    try:
        ex = PeerExchange(dgeom, rank, world)
        mine = ex.export()
    except Exception:
        ok = False
    handles = [None] * world
    tdist.all_gather_object(handles, mine if ok else None, group=group)
    if ok and all(h is not None for h in handles):
        try:
            ex.connect_ipc(handles)
        except Exception:
            ok = False
    else:
        ok = False
    flag = torch.tensor([1 if ok else 0], device=dgeom.dev)
    tdist.all_reduce(flag, op=tdist.ReduceOp.MIN, group=group)
    return ex if int(flag.item()) == 1 else None


class NativeComm:
    """libctk's communicator for the angle-sharded native solve (ctk_comm_*):
    its own NCCL communicator (the id shipped over torch.distributed), plus
    the peer-memory exchange for B's partial images when every rank maps the
    others' buffers.  Without an initialised process group it is a one-rank
    communicator (the sharded code path on one GPU).  Pass it to
    ``gmres.run_gmres(A_local, B_local, b_local, cfg, comm=...)``."""

    def __init__(self, dgeom, group=None, peer_exchange: bool | None = None,
                 nccl_lib: str | None = None):
        import ctypes
        import os

        from . import _native
        self._native, self._ct = _native, ctypes
        self.lib = _native.load()
        self.dg = dgeom
        try:
            import torch.distributed as tdist
            dist_on = tdist.is_available() and tdist.is_initialized()
        except Exception:
            dist_on = False
        self.rank = tdist.get_rank(group) if dist_on else 0
        self.world = tdist.get_world_size(group) if dist_on else 1
        lib_path = (nccl_lib or nccl_library() or "").encode() or None
        nbytes = int(self.lib.ctk_comm_id_bytes())
        idb = None
        if self.rank == 0:
            buf = ctypes.create_string_buffer(nbytes)
            _native.check(self.lib.ctk_comm_unique_id(lib_path, buf), "ctk_comm_unique_id")
            idb = buf.raw
        if self.world > 1:
            obj = [idb]
            tdist.broadcast_object_list(obj, src=tdist.get_global_rank(group, 0) if group else 0,
                                        group=group)
            idb = obj[0]
        h = ctypes.c_void_p()
        _native.check(self.lib.ctk_comm_create(lib_path, idb, self.world, self.rank,
                                               dgeom.dev.index, ctypes.byref(h)), "ctk_comm_create")
        self.handle = h
        self.xchg = None
        if peer_exchange is None:
            peer_exchange = os.environ.get("CTK_PEER_EXCHANGE", "1") != "0"
        if peer_exchange and self.world > 1:
            self.xchg = open_peer_exchange(dgeom, group)
            if self.xchg is not None:
                _native.check(self.lib.ctk_comm_attach_exchange(h, self.xchg.handle),
                              "ctk_comm_attach_exchange")
        wf = int(self.lib.ctk_back_work_floats(dgeom.handle, 0, dgeom.n_angles))
        self.work = dgeom.torch.zeros(max(wf, 4), dtype=dgeom.torch.float32, device=dgeom.dev)

    def back(self, u, out=None, stream=None):
        """out (every rank) = sum over ranks of B_rank u_rank."""
        dg = self.dg
        dg._check(u, dg.m, "u")
        if out is None:
            out = dg.torch.empty(dg.n, dtype=dg.torch.float32, device=dg.dev)
        stream = dg._stream(stream)
        self._native.check(self.lib.ctk_comm_back(self.handle, dg.handle, u.data_ptr(),
                                                  out.data_ptr(), self.work.data_ptr(),
                                                  stream.cuda_stream), "ctk_comm_back")
        return out

    def allreduce(self, t, stream=None):
        """In-place sum of a CUDA fp32 / fp64 tensor over ranks (stream-ordered)."""
        torch = self.dg.torch
        dtype = {torch.float32: 0, torch.float64: 1}[t.dtype]
        stream = self.dg._stream(stream)
        self._native.check(self.lib.ctk_comm_allreduce(self.handle, t.data_ptr(), t.numel(), dtype,
                                                       stream.cuda_stream), "ctk_comm_allreduce")
        return t

    def close(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self.lib.ctk_comm_destroy(h)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def sharded_projectors(grid, geometry, angle_idx, device: int = 0):
    """(A, B) over this rank's angles: the drop-in operators of the sharded
    solve (rows of A / columns of B are the rank's sinogram rows)."""
    from .ct import ParallelGeometry, back_pixel_driven, forward_ray_driven
    local = ParallelGeometry(np.asarray(geometry.angles)[np.asarray(angle_idx)],
                             geometry.det_count, geometry.det_spacing)
    A = forward_ray_driven(grid, local, device=device)
    B = back_pixel_driven(grid, local, device=device)
    return A, B


def local_rows(v, det_count: int, angle_idx):
    """This rank's sinogram rows (angle-major) of a full-geometry vector."""
    idx = np.asarray(angle_idx)
    if isinstance(v, np.ndarray):
        return np.ascontiguousarray(v.reshape(-1, det_count)[idx].ravel())
    import torch
    return v.view(-1, det_count)[torch.as_tensor(idx, device=v.device)].reshape(-1).contiguous()


class CudaShardBackend(ShardBackend):
    """libctk projectors on this rank's angles; partial images summed over
    NVLink peer memory (:class:`PeerExchange`) when every rank can map the
    others' buffers, else NCCL all-reduce.  Small fp64 messages go through
    NCCL.

    Vectors are CUDA tensors (fp32 for images/sinograms, fp64 for the small
    reduction messages).  The process group defaults to the world group.
    """

    def __init__(self, grid, geometry, angle_idx, device: int = 0, group=None,
                 peer_exchange: bool | None = None):
        import os

        import torch
        import torch.distributed as tdist

        from .ct import DeviceGeometry, ParallelGeometry

        self.torch, self.dist, self.group = torch, tdist, group
        self.dev = torch.device("cuda", device)
        local = ParallelGeometry(np.asarray(geometry.angles)[np.asarray(angle_idx)],
                                 geometry.det_count, geometry.det_spacing)
        self.dg = DeviceGeometry(grid, local, device)
        self.n = self.dg.n
        self.m_local = self.dg.m
        self.xchg = None
        world = tdist.get_world_size(group) if tdist.is_initialized() else 1
        if peer_exchange is None:
            peer_exchange = os.environ.get("CTK_PEER_EXCHANGE", "1") != "0"
        if peer_exchange and 1 < world <= 8:
            self.xchg = self._open_exchange(world)

    def _open_exchange(self, world):
        """All ranks agree: every rank creates its buffers, handles are
        all-gathered, every rank maps its peers; any failure -> NCCL path."""
        return open_peer_exchange(self.dg, self.group)

    def back_sum(self, u):
        if self.xchg is None:
            return super().back_sum(u)
        return self.xchg.back(u).clone()

    def zeros(self, size):
        return self.torch.zeros(size, dtype=self.torch.float32, device=self.dev)

    def from_host(self, arr):
        return self.torch.from_numpy(np.asarray(arr, dtype=np.float32)).to(self.dev)

    def to_host(self, v):
        return v.cpu().numpy().astype(np.float64)

    def from_host_f64(self, arr):
        return self.torch.from_numpy(arr).to(self.dev)

    def to_host_f64(self, v):
        return v.cpu().numpy()

    def forward(self, x):
        return self.dg.forward(x)

    def back_partial(self, u):
        return self.dg.back(u)

    def allreduce(self, v):
        self.dist.all_reduce(v, op=self.dist.ReduceOp.SUM, group=self.group)

    def norm2(self, v):
        return float(self.torch.dot(v.double(), v.double()).item())

    def scale(self, v, a):
        return (v.double() * a).float()

    def add(self, a, b):
        return a + b

    def sub(self, a, b):
        return a - b

    # Krylov basis on libctk's K3/K4 kernels (fp64 accumulation, deterministic)
    def basis_init(self, L, rows):
        from .arnoldi import DeviceBasis
        self.basis = DeviceBasis(L, rows, self.dev, self.torch)
        self.stream = self.torch.cuda.current_stream(self.dev)
        self._out = self.torch.zeros(rows + 2, dtype=self.torch.float64, device=self.dev)

    def basis_set(self, j, v, scale):
        self.basis.row(j).copy_(v)
        self.basis.row(j).mul_(scale)

    def basis_row(self, j):
        return self.basis.row(j)

    def basis_dots(self, k, v, want_norm):
        self.basis.dots(k, v, self._out, want_norm, self.stream)
        return self._out[: k + (1 if want_norm else 0)].cpu().numpy().copy()

    def basis_update(self, k, coef, v):
        c = self.torch.from_numpy(np.asarray(coef, dtype=np.float64)).to(self.dev)
        out = self.torch.empty_like(v)
        self.basis.update(k, c, v, out, stream=self.stream)
        return out

    def basis_combine(self, k, y):
        yd = self.torch.from_numpy(np.asarray(y, dtype=np.float64)).to(self.dev)
        out = self.torch.empty(self.basis.L, dtype=self.torch.float32, device=self.dev)
        self.basis.combine(k, yd, out, stream=self.stream)
        return out
