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
}

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
    _lib = L
    return L


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


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    if t is None:
        return None
    return t.data_ptr()
