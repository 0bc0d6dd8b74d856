"""The C-ABI library (CPU): it loads, exports every symbol include/ctk.h
declares, rejects bad arguments before touching CUDA, and its host-side
fp64 projected solve (no GPU needed) matches the reference semantics."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_17892_b200 import _native

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "ctk.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ctk_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _native.load()
    names = declared_symbols()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers exactly the declared ABI
    assert sorted(_native.SIGNATURES) == names


def test_version_and_device_query_without_gpu():
    lib = _native.load()
    assert lib.ctk_version() >= 1
    assert _native.device_count() >= 0
    assert _native.launch_counter() >= 0


def _create(nx, ny, h, D, sp, ang=(0.0, 0.5)):
    lib = _native.load()
    c = np.cos(np.asarray(ang, float))
    s = np.sin(np.asarray(ang, float))
    off = (np.arange(max(D, 1)) - 0.5 * (D - 1)) * sp
    handle = ctypes.c_void_p()
    dp = lambda a: a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
    rc = lib.ctk_geom_create(nx, ny, h, len(ang), dp(c), dp(s), D, dp(off), sp, 0,
                             ctypes.byref(handle))
    return rc, handle


@pytest.mark.parametrize("args", [(0, 4, 1.0, 5, 1.0), (4, 4, -1.0, 5, 1.0),
                                  (4, 4, 1.0, 0, 1.0), (4, 4, 1.0, 5, 0.0)])
def test_invalid_geometry_is_rejected_before_cuda(args):
    rc, h = _create(*args)
    assert rc == _native.CTK_ERR_GEOMETRY
    assert h.value is None
    assert _native.load().ctk_last_error()


def test_error_mapping():
    from paper_2602_17892_b200.ct import GeometryError
    from paper_2602_17892_b200.linop import OperatorShapeError
    with pytest.raises(GeometryError):
        _native.check(_native.CTK_ERR_GEOMETRY)
    with pytest.raises(OperatorShapeError):
        _native.check(_native.CTK_ERR_SHAPE)
    with pytest.raises(ValueError):
        _native.check(_native.CTK_ERR_ARG)
    with pytest.raises(_native.CtkError):
        _native.check(_native.CTK_ERR_CUDA)


def test_null_arguments_rejected():
    lib = _native.load()
    assert lib.ctk_forward(None, None, None, 0, 1, None, None, None) == _native.CTK_ERR_ARG
    assert lib.ctk_back(None, None, None, 0, 1, None, None, None) == _native.CTK_ERR_ARG
    assert lib.ctk_dots(None, 4, 1, None, 8, 0, None, None, None) == _native.CTK_ERR_ARG
    assert lib.ctk_reduce_scratch_bytes(100, 1 << 20) > 100 * 8


def _native_solve(H, beta, strategy, fixed=0.0, fallback=float("nan")):
    lib = _native.load()
    k = H.shape[1]
    H = np.ascontiguousarray(H, dtype=np.float64)
    out, y = np.zeros(4), np.zeros(k)
    _native.check(lib.ctk_projected_solve(H.ctypes.data, k, beta, _native.STRATEGY_CODES[strategy],
                                          fixed, 200, fallback, out.ctypes.data, y.ctypes.data))
    return out, y


@pytest.fixture
def lapack_path():
    lib = _native.load()
    lib.ctk_set_svd_path(1)
    yield lib
    lib.ctk_set_svd_path(0)


def arnoldi_hessenberg(M, b, k):
    V = [b / np.linalg.norm(b)]
    cols = []
    for j in range(k):
        q = M @ V[j]
        h = np.zeros(j + 2)
        for _ in range(2):
            for i in range(j + 1):
                c = V[i] @ q
                h[i] += c
                q = q - c * V[i]
        h[j + 1] = np.linalg.norm(q)
        cols.append(h)
        V.append(q / h[j + 1])
    return O.hessenberg(cols, k), float(np.linalg.norm(b))


def test_fast_path_gcv_and_tikhonov_match_reference():
    """Default lock-free path (C++ bidiagonalisation + dbdsqr + Givens
    Tikhonov): the GCV choice equals the reference's on Arnoldi Hessenbergs
    of noisy ill-posed problems, and y / ||H y - beta e1|| match its lstsq."""
    rng = np.random.default_rng(11)
    n_checked = 0
    for _ in range(12):
        n = 100
        Q, _ = np.linalg.qr(rng.standard_normal((n, n)))
        M = Q @ np.diag(np.logspace(0, -rng.uniform(2, 8), n)) @ Q.T
        b = M @ rng.standard_normal(n) + 0.02 * rng.standard_normal(n)
        for k in (5, 20, 45, 80):
            H, beta = arnoldi_hessenberg(M, b, k)
            out, y = _native_solve(H, beta, "gcv")
            ref = O.lambda_selection(H, beta, "gcv")
            assert out[2] == 0.0 and out[0] == pytest.approx(ref, rel=1e-12)
            y_ref, r_ref = O.projected_tikhonov(H, beta, ref)
            np.testing.assert_allclose(y, y_ref, atol=1e-8 * max(1.0, np.abs(y_ref).max()))
            assert out[1] == pytest.approx(r_ref, rel=1e-7, abs=1e-12)
            for lam in (0.0, 0.05):
                out2, y2 = _native_solve(H, beta, "fixed", fixed=lam)
                y_ref, r_ref = O.projected_tikhonov(H, beta, lam)
                np.testing.assert_allclose(y2, y_ref, atol=1e-8 * max(1.0, np.abs(y_ref).max()))
            n_checked += 1
    assert n_checked == 48


def test_native_projected_solve_matches_reference_selection(lapack_path):
    """dgesdd path (ctk_set_svd_path(1)) vs the reference's loops: same grid
    point every time for both GCV and the ill-conditioned L-curve."""
    rng = np.random.default_rng(3)
    n = 0
    for _ in range(80):
        k = int(rng.integers(2, 70))
        H = np.triu(rng.standard_normal((k + 1, k)), -1) * np.logspace(0, -rng.uniform(1, 10), k)
        beta = float(rng.uniform(0.5, 5.0))
        for strat in ("gcv", "lcurve"):
            out, y = _native_solve(H, beta, strat)
            try:
                ref = O.lambda_selection(H, beta, strat)
            except O.OracleDegenerate:
                assert out[2] == 1.0
                continue
            assert out[2] == 0.0
            assert out[0] == pytest.approx(ref, rel=1e-12)
            y_ref, r_ref = O.projected_tikhonov(H, beta, ref)
            np.testing.assert_allclose(y, y_ref, atol=1e-7 * max(1.0, np.abs(y_ref).max()))
            n += 1
    assert n > 100


def test_native_projected_solve_golden_and_fallback(golden, lapack_path):
    d = golden("solver_cases")
    for i in range(4):
        H = d[f"lam/{i}/H"]
        assert _native_solve(H, 2.5, "gcv")[0][0] == pytest.approx(float(d[f"lam/{i}/gcv"]), rel=1e-12)
        assert _native_solve(H, 2.5, "lcurve")[0][0] == pytest.approx(float(d[f"lam/{i}/lcurve"]),
                                                                      rel=1e-12)
    # all-zero Hessenberg: degenerate curve -> fallback lambda, flagged
    out, _ = _native_solve(np.zeros((4, 3)), 1.0, "gcv", fallback=0.7)
    assert out[2] == 1.0 and out[0] == 0.7
    # plain (lambda = 0): minimum-norm least squares, rank flag
    out, y = _native_solve(np.zeros((3, 2)), 1.0, "none")
    assert out[3] == 1.0 and np.all(y == 0)
