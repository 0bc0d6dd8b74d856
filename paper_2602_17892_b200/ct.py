"""2-D parallel-beam CT operators on the B200: drop-ins for ctkrylov.ct.

``forward_ray_driven(grid, geometry)`` and ``back_pixel_driven(grid,
geometry)`` keep the reference's signatures (ctkrylov/ct.py:182, 204) and
return :class:`~paper_2602_17892_b200.linop.LinearOperator` subclasses whose
``apply`` honours the reference contract (float64 numpy in and out), while
the work runs in libctk's sm_100a kernels (K1/K1d forward, K2 back).  The
same objects expose device-tensor entry points (``apply_device``) used by the
device-resident GMRES driver, which never leaves HBM between iterations.

Conventions are the reference's (ctkrylov/ct.py:10-18): image row-major
(ny, nx) with row 0 at the top; sinogram angle-major, sample a*D + j.  B is
the reference's unmatched pixel-driven backprojector -- never A's adjoint.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .linop import LinearOperator, OperatorShapeError


class GeometryError(ValueError):
    """Invalid grid / geometry configuration (ctkrylov/ct.py:33-34)."""


@dataclass(frozen=True)
class ImageGrid:
    """Centred square-pixel grid (ctkrylov/ct.py:37-66)."""

    nx: int
    ny: int
    pixel_size: float = 1.0

    def __post_init__(self):
        if self.nx <= 0 or self.ny <= 0 or self.pixel_size <= 0:
            raise GeometryError(f"invalid grid: nx={self.nx}, ny={self.ny}, h={self.pixel_size}")

    @property
    def n(self) -> int:
        return self.nx * self.ny

    @property
    def extent(self) -> tuple[float, float, float, float]:
        half_x = 0.5 * self.nx * self.pixel_size
        half_y = 0.5 * self.ny * self.pixel_size
        return (-half_x, half_x, -half_y, half_y)

    def pixel_centers(self) -> tuple[np.ndarray, np.ndarray]:
        xmin, _, _, ymax = self.extent
        h = self.pixel_size
        return np.meshgrid(xmin + (np.arange(self.nx) + 0.5) * h,
                           ymax - (np.arange(self.ny) + 0.5) * h)


@dataclass(frozen=True)
class ParallelGeometry:
    """View angles plus a centred linear detector (ctkrylov/ct.py:69-96)."""

    angles: np.ndarray
    det_count: int
    det_spacing: float

    def __post_init__(self):
        ang = np.asarray(self.angles, dtype=np.float64)
        object.__setattr__(self, "angles", ang)
        if ang.ndim != 1 or ang.size == 0:
            raise GeometryError("angles must be a non-empty 1-D array")
        if np.any(np.diff(ang) <= 0) or ang[0] < 0 or ang[-1] >= np.pi:
            raise GeometryError("angles must be strictly increasing within [0, pi)")
        if self.det_count <= 0 or self.det_spacing <= 0:
            raise GeometryError(
                f"invalid detector: count={self.det_count}, spacing={self.det_spacing}")

    @property
    def m(self) -> int:
        return len(self.angles) * self.det_count

    def bin_offsets(self) -> np.ndarray:
        j = np.arange(self.det_count, dtype=np.float64)
        return (j - 0.5 * (self.det_count - 1)) * self.det_spacing


def trig_tables(geometry: ParallelGeometry) -> tuple[np.ndarray, np.ndarray]:
    """Scalar np.cos/np.sin per angle, bitwise what the reference evaluates
    (ctkrylov/ct.py:145 in _siddon_ray, 225 in back_pixel_driven)."""
    cos_tab = np.array([np.cos(float(t)) for t in geometry.angles], dtype=np.float64)
    sin_tab = np.array([np.sin(float(t)) for t in geometry.angles], dtype=np.float64)
    return cos_tab, sin_tab


def _torch():
    import torch
    return torch


def _require_cuda(device: int):
    torch = _torch()
    if not torch.cuda.is_available():
        raise _native.CtkError("a CUDA device is required: libctk has no CPU path")
    if device >= torch.cuda.device_count():
        raise _native.CtkError(f"CUDA device {device} not present")
    return torch


def _dptr(arr: np.ndarray):
    return arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


class DeviceGeometry:
    """A libctk geometry handle on one GPU plus its stream-local workspaces.

    The handle is immutable once built (thread-/stream-safe, like the
    reference's pure apply).  Work buffers (K1's zero-bordered staging copies,
    K2's split partial images) are cached per CUDA stream.
    """

    def __init__(self, grid: ImageGrid, geometry: ParallelGeometry, device: int = 0):
        torch = _require_cuda(device)
        self.torch = torch
        self.grid = grid
        self.geometry = geometry
        self.device = int(device)
        self.dev = torch.device("cuda", self.device)
        self.cos_tab, self.sin_tab = trig_tables(geometry)
        self.offsets = np.ascontiguousarray(geometry.bin_offsets())
        lib = _native.load()
        handle = ctypes.c_void_p()
        _native.check(lib.ctk_geom_create(
            grid.nx, grid.ny, float(grid.pixel_size), len(geometry.angles),
            _dptr(self.cos_tab), _dptr(self.sin_tab), geometry.det_count, _dptr(self.offsets),
            float(geometry.det_spacing), self.device, ctypes.byref(handle)), "ctk_geom_create")
        self._lib = lib
        self.handle = handle
        n, m, st = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        ndeg = ctypes.c_int()
        _native.check(lib.ctk_geom_info(handle, ctypes.byref(n), ctypes.byref(m),
                                        ctypes.byref(st), ctypes.byref(ndeg)))
        self.n, self.m = n.value, m.value
        self.stage_floats = st.value
        self.n_degenerate = ndeg.value
        self.n_angles = len(geometry.angles)
        self.det_count = geometry.det_count
        self._work = {}

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self._lib.ctk_geom_destroy(h)
            except Exception:
                pass
            self.handle = None

    # -- workspace ---------------------------------------------------------
    def _stream(self, stream):
        if stream is None:
            stream = self.torch.cuda.current_stream(self.dev)
        return stream

    def _workspace(self, kind: str, floats: int, stream):
        key = (kind, stream.cuda_stream)
        buf = self._work.get(key)
        if buf is None or buf.numel() < floats:
            buf = self.torch.zeros(max(floats, 4), dtype=self.torch.float32, device=self.dev)
            self._work[key] = buf
        return buf

    def _range(self, a0, a1):
        a1 = self.n_angles if a1 is None else a1
        if not (0 <= a0 <= a1 <= self.n_angles):
            raise OperatorShapeError(f"angle range [{a0}, {a1}) outside [0, {self.n_angles})")
        return a0, a1

    def _check(self, t, numel, name):
        torch = self.torch
        if t.device != self.dev or t.dtype != torch.float32 or not t.is_contiguous():
            raise OperatorShapeError(f"{name} must be a contiguous float32 tensor on {self.dev}")
        if t.numel() != numel:
            raise OperatorShapeError(f"{name} has {t.numel()} elements, expected {numel}")

    # -- device entry points (torch tensors, stream-ordered) ---------------
    def forward(self, x, out=None, a0: int = 0, a1: int | None = None, b=None, stream=None):
        """out = A x over angles [a0, a1) (or b - A x when b is given)."""
        a0, a1 = self._range(a0, a1)
        rows = (a1 - a0) * self.det_count
        self._check(x, self.n, "x")
        if out is None:
            out = self.torch.empty(rows, dtype=self.torch.float32, device=self.dev)
        self._check(out, rows, "out")
        if b is not None:
            self._check(b, rows, "b")
        stream = self._stream(stream)
        work = self._workspace("stage", self.stage_floats, stream)
        _native.check(self._lib.ctk_forward(self.handle, x.data_ptr(), out.data_ptr(), a0, a1,
                                            _native.ptr(b), work.data_ptr(), stream.cuda_stream),
                      "ctk_forward")
        return out

    def forward_exact(self, x, out=None, a0: int = 0, a1: int | None = None, stream=None):
        """Literal fp64 Siddon for every angle (validation path)."""
        a0, a1 = self._range(a0, a1)
        rows = (a1 - a0) * self.det_count
        self._check(x, self.n, "x")
        if out is None:
            out = self.torch.empty(rows, dtype=self.torch.float32, device=self.dev)
        self._check(out, rows, "out")
        stream = self._stream(stream)
        _native.check(self._lib.ctk_forward_exact(self.handle, x.data_ptr(), out.data_ptr(),
                                                  a0, a1, stream.cuda_stream), "ctk_forward_exact")
        return out

    def back(self, u, out=None, a0: int = 0, a1: int | None = None, x0=None, stream=None):
        """out = (x0 or 0) + B u, summing angles [a0, a1)."""
        a0, a1 = self._range(a0, a1)
        self._check(u, (a1 - a0) * self.det_count, "u")
        if out is None:
            out = self.torch.empty(self.n, dtype=self.torch.float32, device=self.dev)
        self._check(out, self.n, "out")
        if x0 is not None:
            self._check(x0, self.n, "x0")
        stream = self._stream(stream)
        wf = int(self._lib.ctk_back_work_floats(self.handle, a0, a1))
        work = self._workspace("back", wf, stream) if wf > 0 else None
        _native.check(self._lib.ctk_back(self.handle, u.data_ptr(), out.data_ptr(), a0, a1,
                                         _native.ptr(x0), _native.ptr(work), stream.cuda_stream),
                      "ctk_back")
        return out

    def adjoint(self, u, out=None, a0: int = 0, a1: int | None = None, x0=None, stream=None):
        """out = (x0 or 0) + A^T u over angles [a0, a1): the exact transpose of
        the Siddon matrix (K7), i.e. the reference's matched_back."""
        a0, a1 = self._range(a0, a1)
        self._check(u, (a1 - a0) * self.det_count, "u")
        if out is None:
            out = self.torch.empty(self.n, dtype=self.torch.float32, device=self.dev)
        self._check(out, self.n, "out")
        if x0 is not None:
            self._check(x0, self.n, "x0")
        stream = self._stream(stream)
        wf = int(self._lib.ctk_adjoint_work_floats(self.handle, a0, a1))
        work = self._workspace("adjoint", wf, stream) if wf > 0 else None
        _native.check(self._lib.ctk_adjoint(self.handle, u.data_ptr(), out.data_ptr(), a0, a1,
                                            _native.ptr(x0), _native.ptr(work), stream.cuda_stream),
                      "ctk_adjoint")
        return out

    def count_segments(self, a0: int = 0, a1: int | None = None) -> tuple[int, int]:
        """(kept segments, CSR nnz) of A over angles [a0, a1) (K6)."""
        a0, a1 = self._range(a0, a1)
        stream = self._stream(None)
        counts = self.torch.zeros(2, dtype=self.torch.int64, device=self.dev)
        _native.check(self._lib.ctk_count_segments(self.handle, a0, a1, counts.data_ptr(),
                                                   stream.cuda_stream), "ctk_count_segments")
        raw, nnz = counts.cpu().tolist()
        return int(raw), int(nnz)


class _GpuOperator(LinearOperator):
    """LinearOperator whose host apply round-trips through the GPU kernel."""

    def __init__(self, rows, cols, dgeom: DeviceGeometry):
        super().__init__(rows, cols, None)
        self.dgeom = dgeom

    def _host_apply(self, v: np.ndarray) -> np.ndarray:
        torch = self.dgeom.torch
        xd = torch.from_numpy(np.ascontiguousarray(v, dtype=np.float32)).to(self.dgeom.dev)
        out = self.apply_device(xd)
        return out.cpu().numpy().astype(np.float64)


class GpuForward(_GpuOperator):
    """A: Siddon ray-driven forward projector (ctkrylov/ct.py:182-201) on the GPU."""

    kind = "forward"

    def apply_device(self, x, out=None, b=None, stream=None):
        return self.dgeom.forward(x, out=out, b=b, stream=stream)


class GpuBack(_GpuOperator):
    """B: pixel-driven linear-interpolation backprojector (ctkrylov/ct.py:204-245)."""

    kind = "back"

    def apply_device(self, u, out=None, x0=None, stream=None):
        return self.dgeom.back(u, out=out, x0=x0, stream=stream)


class GpuAdjoint(_GpuOperator):
    """A^T: exact transpose of the Siddon forward projector on the GPU (what
    ctkrylov.ct.matched_back returns for a CSR-backed forward, ct.py:248-264)."""

    kind = "adjoint"

    def apply_device(self, u, out=None, x0=None, stream=None):
        return self.dgeom.adjoint(u, out=out, x0=x0, stream=stream)


_GEOM_CACHE: dict = {}


def device_geometry(grid: ImageGrid, geometry: ParallelGeometry, device: int = 0) -> DeviceGeometry:
    """Shared DeviceGeometry per (grid, geometry, device) so A and B pair up."""
    key = (grid, geometry.angles.tobytes(), geometry.det_count, float(geometry.det_spacing),
           int(device))
    dg = _GEOM_CACHE.get(key)
    if dg is None:
        dg = DeviceGeometry(grid, geometry, device)
        _GEOM_CACHE[key] = dg
    return dg


def forward_ray_driven(grid: ImageGrid, geometry: ParallelGeometry, device: int = 0) -> GpuForward:
    """Drop-in for ctkrylov.ct.forward_ray_driven (ct.py:182): matrix-free on
    the GPU; ``sparse_matrix`` is None because no CSR is ever assembled."""
    dg = device_geometry(grid, geometry, device)
    return GpuForward(geometry.m, grid.n, dg)


def back_pixel_driven(grid: ImageGrid, geometry: ParallelGeometry, device: int = 0) -> GpuBack:
    """Drop-in for ctkrylov.ct.back_pixel_driven (ct.py:204)."""
    dg = device_geometry(grid, geometry, device)
    return GpuBack(grid.n, geometry.m, dg)


DENSE_ASSEMBLY_GUARD = 10**7             # ctkrylov/ct.py:30, desk-scale guard for dense assembly


def matched_back(forward: LinearOperator) -> LinearOperator:
    """Drop-in for ctkrylov.ct.matched_back (ct.py:248-264): the exact
    transpose of the forward projector.  For the GPU forward this is K7 (no
    matrix is ever assembled); other operators follow the reference: the
    transpose of an assembled sparse matrix, else a dense transpose under the
    desk-scale guard."""
    if isinstance(forward, GpuForward):
        return GpuAdjoint(forward.cols, forward.rows, forward.dgeom)
    mat = getattr(forward, "sparse_matrix", None)
    if mat is not None:
        mat_t = mat.T.tocsr()
        return LinearOperator(forward.cols, forward.rows, lambda v: mat_t @ v)
    if forward.rows * forward.cols > DENSE_ASSEMBLY_GUARD:
        raise GeometryError(
            "matched mode requires assembling the forward matrix; "
            f"{forward.rows}x{forward.cols} exceeds the desk-scale guard of "
            f"{DENSE_ASSEMBLY_GUARD} entries")
    dense_t = np.ascontiguousarray(forward.to_dense().T)
    return LinearOperator(forward.cols, forward.rows, lambda v: dense_t @ v)


# ---------------------------------------------------------------------------
# Problem generation on the device: ctkrylov/ct.py:99-134,
# 267-356.  Phantoms are sampled by K_phantom (bitwise numpy), the clean data
# is the GPU forward projection, and the noise is scaled on the device from
# numpy's own Gaussian draw; the host sees the reference's numpy contract.
# ---------------------------------------------------------------------------

# Modified Shepp-Logan ellipse stack (value, a, b, x0, y0, phi_degrees) on
# [-1, 1]^2 -- the published Shepp & Logan (1974) / Toft modified intensities,
# in the reference's order (ctkrylov/ct.py:99-112).
SHEPP_LOGAN_ELLIPSES = (
    (1.0, 0.69, 0.92, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.8740, 0.0, -0.0184, 0.0),
    (-0.2, 0.1100, 0.3100, 0.22, 0.0, -18.0),
    (-0.2, 0.1600, 0.4100, -0.22, 0.0, 18.0),
    (0.1, 0.2100, 0.2500, 0.0, 0.35, 0.0),
    (0.1, 0.0460, 0.0460, 0.0, 0.1, 0.0),
    (0.1, 0.0460, 0.0460, 0.0, -0.1, 0.0),
    (0.1, 0.0460, 0.0230, -0.08, -0.605, 0.0),
    (0.1, 0.0230, 0.0230, 0.0, -0.606, 0.0),
    (0.1, 0.0230, 0.0460, 0.06, -0.605, 0.0),
)


def _ellipse_table(rows) -> np.ndarray:
    """(value, a, b, x0, y0, phi_radians) rows -> the n x 7 table ctk_phantom
    takes, with cos/sin evaluated by numpy exactly as the reference does."""
    out = np.empty((len(rows), 7), dtype=np.float64)
    for i, (value, a, b, x0, y0, phi) in enumerate(rows):
        out[i] = (value, a, b, x0, y0, np.cos(phi), np.sin(phi))
    return np.ascontiguousarray(out)


def phantom_device(grid: ImageGrid, ellipses, scale: float = 1.0, device: int = 0,
                   want64: bool = True, want32: bool = True, stream=None):
    """Sample ellipses (value, a, b, x0, y0, phi in radians) at the pixel
    centres of ``grid`` divided by ``scale`` on the GPU.  Returns
    ``(img64, img32)`` CUDA tensors (either None when not requested)."""
    torch = _require_cuda(device)
    dev = torch.device("cuda", int(device))
    tab = _ellipse_table(ellipses)
    img64 = torch.empty(grid.n, dtype=torch.float64, device=dev) if want64 else None
    img32 = torch.empty(grid.n, dtype=torch.float32, device=dev) if want32 else None
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    xmin, _, _, ymax = grid.extent
    with torch.cuda.device(dev):
        _native.check(_native.load().ctk_phantom(
            grid.nx, grid.ny, float(xmin), float(ymax), float(grid.pixel_size), float(scale),
            _dptr(tab), len(tab), _native.ptr(img64), _native.ptr(img32), stream.cuda_stream),
            "ctk_phantom")
    return img64, img32


def shepp_logan(grid: ImageGrid, device: int = 0) -> np.ndarray:
    """Drop-in for ctkrylov.ct.shepp_logan (ct.py:115-134): the modified
    Shepp-Logan phantom at pixel centres, the image square mapped onto
    [-1, 1]^2; sampled on the GPU, bitwise the reference's float64 image."""
    if grid.nx != grid.ny:
        raise GeometryError(f"phantom requires a square grid, got {grid.nx}x{grid.ny}")
    scale = 0.5 * grid.nx * grid.pixel_size
    rows = [(v, a, b, x0, y0, np.deg2rad(phi)) for v, a, b, x0, y0, phi in SHEPP_LOGAN_ELLIPSES]
    img64, _ = phantom_device(grid, rows, scale, device, want32=False)
    return img64.cpu().numpy()


def add_noise_device(b_clean, level: float, seed: int, out32=None, stream=None):
    """add_noise (ctkrylov/ct.py:267-283) for a CUDA sinogram (fp32 or fp64):
    ``||e|| = level * ||b_clean||`` exactly, e from numpy's
    ``default_rng(seed).standard_normal(m)``.  Returns
    ``(b_noisy64, b_noisy32, noise_norm)``, the first two CUDA tensors."""
    if level < 0:
        raise ValueError(f"noise level must be nonnegative, got {level}")
    torch = _torch()
    dev = b_clean.device
    m = b_clean.numel()
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    b64 = torch.empty(m, dtype=torch.float64, device=dev)
    b32 = out32 if out32 is not None else torch.empty(m, dtype=torch.float32, device=dev)
    if level == 0.0:
        b64.copy_(b_clean)
        b32.copy_(b_clean)
        return b64, b32, 0.0
    g = torch.from_numpy(np.random.default_rng(seed).standard_normal(m)).to(dev)
    scratch = torch.zeros(int(_native.load().ctk_noise_scratch_bytes()) // 8,
                          dtype=torch.float64, device=dev)
    nn = torch.empty(1, dtype=torch.float64, device=dev)
    f32 = b_clean.dtype == torch.float32
    with torch.cuda.device(dev):
        _native.check(_native.load().ctk_add_noise(
            b_clean.data_ptr() if f32 else None, None if f32 else b_clean.data_ptr(),
            g.data_ptr(), m, float(level), b64.data_ptr(), b32.data_ptr(), nn.data_ptr(),
            scratch.data_ptr(), stream.cuda_stream), "ctk_add_noise")
    return b64, b32, float(nn.item())


def add_noise(b_clean, level: float, seed: int, device: int = 0) -> tuple[np.ndarray, float]:
    """Drop-in for ctkrylov.ct.add_noise (ct.py:267-283), scaled on the GPU.
    Host float64 in, host float64 out; level 0 returns a copy."""
    if level < 0:
        raise ValueError(f"noise level must be nonnegative, got {level}")
    b_clean = np.asarray(b_clean, dtype=np.float64)
    if level == 0.0:
        return b_clean.copy(), 0.0
    torch = _require_cuda(device)
    bd = torch.from_numpy(np.ascontiguousarray(b_clean)).to(torch.device("cuda", int(device)))
    b64, _, nn = add_noise_device(bd, level, seed)
    return b64.cpu().numpy(), nn


@dataclass
class CtProblem:
    """A fully populated CT test problem (ctkrylov/ct.py:286-307).  Host fields
    are numpy as in the reference; the device copies the solver consumes are
    kept alongside (``x_true_device`` / ``b_noisy_device``, fp32)."""

    grid: ImageGrid
    geometry: ParallelGeometry
    x_true: np.ndarray
    b_clean: np.ndarray
    b_noisy: np.ndarray
    noise_norm: float
    forward: LinearOperator
    back: LinearOperator
    matched: bool
    name: str = "custom"
    x_true_device: object = None
    b_noisy_device: object = None

    @property
    def m(self) -> int:
        return self.geometry.m

    @property
    def n(self) -> int:
        return self.grid.n


def make_ct_problem(nx: int, n_angles: int, det_count: int | None = None,
                    noise_level: float = 0.025, seed: int = 0, matched: bool = False,
                    name: str = "custom", device: int = 0) -> CtProblem:
    """Drop-in for ctkrylov.ct.make_ct_problem (ct.py:310-337): square
    Shepp-Logan problem on [-1, 1]^2 with the detector spanning the image
    diagonal, generated on the GPU (phantom -> K1 -> noise)."""
    if det_count is None:
        det_count = nx
    grid = ImageGrid(nx, nx, pixel_size=2.0 / nx)
    width = nx * grid.pixel_size
    det_spacing = np.sqrt(2.0) * width / det_count
    angles = np.arange(n_angles) * np.pi / n_angles
    geometry = ParallelGeometry(angles, det_count, det_spacing)
    scale = 0.5 * grid.nx * grid.pixel_size
    rows = [(v, a, b, x0, y0, np.deg2rad(phi)) for v, a, b, x0, y0, phi in SHEPP_LOGAN_ELLIPSES]
    x64, x32 = phantom_device(grid, rows, scale, device)
    forward = forward_ray_driven(grid, geometry, device)
    back = matched_back(forward) if matched else back_pixel_driven(grid, geometry, device)
    bc = forward.dgeom.forward(x32)
    b64, b32, noise_norm = add_noise_device(bc, noise_level, seed)
    return CtProblem(grid, geometry, x64.cpu().numpy(), bc.double().cpu().numpy(),
                     b64.cpu().numpy(), noise_norm, forward, back, matched, name,
                     x_true_device=x32, b_noisy_device=b32)


BUILTIN_PROBLEMS = ("tp1-like", "tp2", "tp3-desk")


def build_test_problem(name: str, matched: bool = False, seed: int = 0,
                       device: int = 0) -> CtProblem:
    """Drop-in for ctkrylov.ct.build_test_problem (ct.py:343-356)."""
    if name == "tp1-like":
        return make_ct_problem(128, 180, 128, 0.001, seed, matched, name, device)
    if name == "tp2":
        return make_ct_problem(128, 50, 128, 0.025, seed, matched, name, device)
    if name == "tp3-desk":
        return make_ct_problem(256, 50, 256, 0.015, seed, matched, name, device)
    raise GeometryError(f"unknown test problem {name!r}; choose from {BUILTIN_PROBLEMS}")


def write_pgm(path, image, shape: tuple[int, int], window=None) -> None:
    """16-bit binary PGM (ctkrylov/ct.py:359-370): values mapped linearly from
    [lo, hi] (default: the image's own range) onto 0..65535, big-endian."""
    img = np.asarray(image, dtype=np.float64).reshape(shape)
    lo, hi = window if window is not None else (img.min(), img.max())
    if hi <= lo:
        scaled = np.zeros_like(img)
    else:
        scaled = np.clip((img - lo) / (hi - lo), 0.0, 1.0)
    data = np.round(scaled * 65535).astype(">u2")
    with open(path, "wb") as f:
        f.write(f"P5\n{shape[1]} {shape[0]}\n65535\n".encode("ascii"))
        f.write(data.tobytes())


def write_csv_image(path, image, shape: tuple[int, int]) -> None:
    """Row-major CSV of an image or sinogram, repr() floats (ct.py:373-379)."""
    img = np.asarray(image, dtype=np.float64).reshape(shape)
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        for row in img:
            f.write(",".join(repr(float(v)) for v in row))
            f.write("\n")
