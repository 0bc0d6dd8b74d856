"""ctypes binding of libctk.so (the C ABI declared in include/ctk.h).

The library is the product's only compute path: there is no CPU fallback.
Loading fails loudly when libctk.so is missing or unbuildable, and every
compute entry point checks that a CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os

from . import build as _build

CTK_OK = 0
CTK_ERR_ARG = -1
CTK_ERR_SHAPE = -2
CTK_ERR_GEOMETRY = -3
CTK_ERR_CUDA = -4

# Every symbol include/ctk.h declares, with its ctypes signature.
_c = ctypes
_vp, _dp, _fp = _c.c_void_p, _c.c_void_p, _c.c_void_p
SIGNATURES = {
    "ctk_version": (_c.c_int, []),
    "ctk_last_error": (_c.c_char_p, []),
    "ctk_device_count": (_c.c_int, [_c.POINTER(_c.c_int)]),
    "ctk_launch_counter": (_c.c_int64, []),
    "ctk_geom_create": (_c.c_int, [_c.c_int, _c.c_int, _c.c_double, _c.c_int,
                                   _c.POINTER(_c.c_double), _c.POINTER(_c.c_double), _c.c_int,
                                   _c.POINTER(_c.c_double), _c.c_double, _c.c_int,
                                   _c.POINTER(_c.c_void_p)]),
    "ctk_geom_destroy": (_c.c_int, [_vp]),
    "ctk_geom_info": (_c.c_int, [_vp, _c.POINTER(_c.c_int64), _c.POINTER(_c.c_int64),
                                 _c.POINTER(_c.c_int64), _c.POINTER(_c.c_int)]),
    "ctk_forward": (_c.c_int, [_vp, _fp, _fp, _c.c_int, _c.c_int, _fp, _fp, _vp]),
    "ctk_forward_exact": (_c.c_int, [_vp, _fp, _fp, _c.c_int, _c.c_int, _vp]),
    "ctk_count_segments": (_c.c_int, [_vp, _c.c_int, _c.c_int, _vp, _vp]),
    "ctk_back_work_floats": (_c.c_int64, [_vp, _c.c_int, _c.c_int]),
    "ctk_back_work_layout": (_c.c_int, [_vp, _vp]),
    "ctk_adjoint": (_c.c_int, [_vp, _fp, _fp, _c.c_int, _c.c_int, _fp, _fp, _vp]),
    "ctk_adjoint_work_floats": (_c.c_int64, [_vp, _c.c_int, _c.c_int]),
    "ctk_back": (_c.c_int, [_vp, _fp, _fp, _c.c_int, _c.c_int, _fp, _fp, _vp]),
    "ctk_reduce_scratch_bytes": (_c.c_size_t, [_c.c_int, _c.c_int64]),
    "ctk_dots": (_c.c_int, [_fp, _c.c_int64, _c.c_int, _fp, _c.c_int64, _c.c_int, _dp, _vp, _vp]),
    "ctk_update": (_c.c_int, [_fp, _c.c_int64, _c.c_int, _dp, _fp, _fp, _c.c_int64, _dp, _vp,
                              _vp]),
    "ctk_norm2": (_c.c_int, [_fp, _c.c_int64, _dp, _vp, _vp]),
    "ctk_scale": (_c.c_int, [_fp, _fp, _c.c_int64, _dp, _vp]),
    "ctk_cgs2_step": (_c.c_int, [_fp, _c.c_int64, _c.c_int, _c.c_int64, _fp, _dp, _dp, _vp,
                                 _vp]),
    "ctk_combine": (_c.c_int, [_fp, _c.c_int64, _c.c_int, _dp, _fp, _fp, _c.c_int64, _dp, _vp,
                               _vp]),
    "ctk_gs_step": (_c.c_int, [_fp, _c.c_int64, _c.c_int, _c.c_int64, _fp, _c.c_int, _dp, _dp,
                               _vp, _vp]),
    "ctk_arnoldi_step": (_c.c_int, [_vp, _c.c_int, _c.c_int, _fp, _c.c_int64, _c.c_int, _fp, _fp,
                                    _fp, _c.c_int64, _fp, _c.c_int64, _fp, _fp,
                                    _dp, _c.c_int, _dp, _vp, _vp]),
    "ctk_iterate": (_c.c_int, [_vp, _c.c_int, _fp, _c.c_int64, _c.c_int, _dp, _dp, _fp, _fp, _fp,
                               _fp, _fp, _dp, _fp, _c.c_int64, _fp, _c.c_int64, _fp,
                               _fp, _fp, _vp, _vp]),
    "ctk_iterate_batch": (_c.c_int, [_fp, _c.c_int64, _fp, _fp, _c.c_int64, _fp, _c.c_int64,
                                     _fp, _fp, _c.c_int64, _c.c_int, _c.c_int, _dp, _c.c_int, _dp,
                                     _vp, _c.c_int, _vp]),
    "ctk_set_lapack": (_c.c_int, [_vp, _vp]),
    "ctk_set_lapack_extra": (_c.c_int, [_vp]),
    "ctk_set_svd_path": (_c.c_int, [_c.c_int]),
    "ctk_projected_solve": (_c.c_int, [_dp, _c.c_int, _c.c_double, _c.c_int, _c.c_double,
                                       _c.c_int, _c.c_double, _dp, _dp]),
    "ctk_solve": (_c.c_int, [_vp, _vp, _vp, _vp]),
    "ctk_metrics_scratch_bytes": (_c.c_size_t, []),
    "ctk_metrics": (_c.c_int, [_fp, _fp, _c.c_int, _c.c_int, _c.c_double, _dp, _vp, _vp]),
    "ctk_phantom": (_c.c_int, [_c.c_int, _c.c_int, _c.c_double, _c.c_double, _c.c_double,
                               _c.c_double, _c.POINTER(_c.c_double), _c.c_int, _dp, _fp, _vp]),
    "ctk_noise_scratch_bytes": (_c.c_size_t, []),
    "ctk_add_noise": (_c.c_int, [_fp, _dp, _dp, _c.c_int64, _c.c_double, _dp, _fp, _dp, _vp, _vp]),
    "ctk_xchg_create": (_c.c_int, [_vp, _c.c_int, _c.c_int, _c.POINTER(_c.c_void_p)]),
    "ctk_xchg_destroy": (_c.c_int, [_vp]),
    "ctk_xchg_local": (_c.c_int, [_vp, _c.POINTER(_c.c_void_p), _c.POINTER(_c.c_void_p),
                                  _c.POINTER(_c.c_void_p)]),
    "ctk_xchg_handle_bytes": (_c.c_size_t, []),
    "ctk_xchg_export": (_c.c_int, [_vp, _c.c_char_p]),
    "ctk_xchg_connect_ipc": (_c.c_int, [_vp, _c.c_char_p]),
    "ctk_xchg_connect_ptrs": (_c.c_int, [_vp, _c.POINTER(_c.c_void_p), _c.POINTER(_c.c_void_p),
                                         _c.POINTER(_c.c_void_p)]),
    "ctk_back_exchange": (_c.c_int, [_vp, _vp, _fp, _c.c_uint, _c.c_int, _fp, _vp]),
    "ctk_xchg_status": (_c.c_int, [_vp, _c.POINTER(_c.c_int)]),
    "ctk_comm_id_bytes": (_c.c_size_t, []),
    "ctk_comm_unique_id": (_c.c_int, [_c.c_char_p, _vp]),
    "ctk_comm_create": (_c.c_int, [_c.c_char_p, _vp, _c.c_int, _c.c_int, _c.c_int,
                                   _c.POINTER(_c.c_void_p)]),
    "ctk_comm_destroy": (_c.c_int, [_vp]),
    "ctk_comm_attach_exchange": (_c.c_int, [_vp, _vp]),
    "ctk_comm_rank": (_c.c_int, [_vp, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "ctk_comm_allreduce": (_c.c_int, [_vp, _vp, _c.c_int64, _c.c_int, _vp]),
    "ctk_comm_back": (_c.c_int, [_vp, _vp, _fp, _fp, _fp, _vp]),
    "ctk_profile_begin": (_c.c_int, []),
    "ctk_profile_end": (_c.c_int, [_c.c_int, _c.POINTER(_c.c_int64), _c.POINTER(_c.c_double),
                                   _c.POINTER(_c.c_double)]),
}

PROFILE_KINDS = ("forward", "back", "cgs2", "combine")


class SolveCfg(ctypes.Structure):
    _fields_ = [("ab", ctypes.c_int), ("hybrid", ctypes.c_int), ("strategy", ctypes.c_int),
                ("max_iter", ctypes.c_int), ("restart_period", ctypes.c_int),
                ("stopping", ctypes.c_int), ("lookahead", ctypes.c_int),
                ("lambda_value", ctypes.c_double), ("dp_tau", ctypes.c_double),
                ("noise_norm", ctypes.c_double), ("rns_epsilon", ctypes.c_double),
                ("reorthogonalize", ctypes.c_int)]


class SolveBufs(ctypes.Structure):
    _fields_ = [("W", _vp), ("ld", ctypes.c_int64), ("rows", ctypes.c_int),
                ("q", _vp), ("tmp", _vp), ("z", _vp), ("r", _vp), ("xk", _vp), ("x_cur", _vp),
                ("b", _vp), ("aux1", _vp), ("ld1", ctypes.c_int64), ("aux2", _vp),
                ("ld2", ctypes.c_int64), ("d0", _vp),
                ("hs", _vp), ("h_host", _vp), ("hcols", ctypes.c_int),
                ("y_dev", _vp), ("y_host", _vp), ("norms", _vp), ("norms_host", _vp),
                ("scal", _vp), ("scal_host", _vp),
                ("stage_a", _vp), ("back_a", _vp), ("stage_b", _vp), ("back_b", _vp),
                ("scratch_a", _vp), ("scratch_b", _vp), ("stream_a", _vp), ("stream_b", _vp),
                ("x_true", _vp), ("img_nx", ctypes.c_int), ("img_ny", ctypes.c_int),
                ("dyn_range", ctypes.c_double), ("metrics", _vp), ("metrics_host", _vp),
                ("scratch_m", _vp), ("snapshot_stride", ctypes.c_int), ("snaps", _vp),
                ("n_snaps", ctypes.c_int), ("comm", _vp)]


class SolveOut(ctypes.Structure):
    _fields_ = [("n_records", ctypes.c_int), ("stop_reason", ctypes.c_int),
                ("cycles", ctypes.c_int), ("x_is_x0", ctypes.c_int),
                ("k", _vp), ("warn", _vp), ("lambda_", _vp), ("residual", _vp),
                ("data_residual", _vp), ("proj_residual", _vp), ("solution_norm", _vp),
                ("elapsed", _vp), ("rre", _vp), ("ssim", _vp)]


STOP_CODES = {"none": 0, "dp": 3, "rns": 4}
STOP_NAMES = {1: "maxiter", 2: "breakdown", 3: "dp", 4: "rns"}

_lib = None


class CtkError(RuntimeError):
    """A libctk call failed (CUDA runtime error or invalid call)."""


def lib_path() -> str:
    return _build.LIB


def load(build_if_missing: bool = True):
    """Load libctk.so (building it in-tree with nvcc if absent or stale)."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if build_if_missing and not _build.up_to_date():
        try:
            _build.build()
        except Exception as exc:  # no toolchain on this host and no prebuilt lib
            if not os.path.exists(path):
                raise CtkError(f"libctk.so is missing and could not be built: {exc}") from exc
    if not os.path.exists(path):
        raise CtkError(f"libctk.so not found at {path}; run `python -m paper_2602_17892_b200.build`")
    L = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _register_lapack(L)
    _lib = L
    return L


def _register_lapack(L) -> None:
    """Hand libctk the LAPACK dgesdd that scipy exports (cython_lapack)."""
    try:
        from scipy.linalg import cython_blas, cython_lapack
        api = ctypes.pythonapi
        api.PyCapsule_GetName.restype = ctypes.c_char_p
        api.PyCapsule_GetName.argtypes = [ctypes.py_object]
        api.PyCapsule_GetPointer.restype = ctypes.c_void_p
        api.PyCapsule_GetPointer.argtypes = [ctypes.py_object, ctypes.c_char_p]

        def fnptr(cap):
            return ctypes.c_void_p(api.PyCapsule_GetPointer(cap, api.PyCapsule_GetName(cap)))

        L.ctk_set_lapack(fnptr(cython_lapack.__pyx_capi__["dgesdd"]),
                         fnptr(cython_blas.__pyx_capi__["ddot"]))
        L.ctk_set_lapack_extra(fnptr(cython_lapack.__pyx_capi__["dbdsqr"]))
    except Exception:   # the projected solve then reports "not registered"
        pass


STRATEGY_CODES = {"none": 0, "fixed": 1, "lcurve": 2, "gcv": 3}


def check(rc: int, what: str = "") -> None:
    """Map a CTK_ERR_* status to the reference's exception types."""
    if rc == CTK_OK:
        return
    msg = (load().ctk_last_error() or b"").decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if rc == CTK_ERR_SHAPE:
        from .linop import OperatorShapeError
        raise OperatorShapeError(msg)
    if rc == CTK_ERR_GEOMETRY:
        from .ct import GeometryError
        raise GeometryError(msg)
    if rc == CTK_ERR_ARG:
        raise ValueError(msg)
    raise CtkError(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    check(load().ctk_device_count(ctypes.byref(n)))
    return n.value


def launch_counter() -> int:
    """Kernels libctk has launched in this process (evidence for bench.py)."""
    return int(load().ctk_launch_counter())


def profile_begin() -> None:
    check(load().ctk_profile_begin(), "ctk_profile_begin")


def profile_end() -> dict:
    """{kind: (launches, mean_ms, total_ms)} for the calls since profile_begin()."""
    n = len(PROFILE_KINDS)
    counts = (ctypes.c_int64 * n)()
    mean = (ctypes.c_double * n)()
    total = (ctypes.c_double * n)()
    check(load().ctk_profile_end(n, counts, mean, total), "ctk_profile_end")
    return {k: (int(counts[i]), float(mean[i]), float(total[i]))
            for i, k in enumerate(PROFILE_KINDS) if counts[i]}


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()
