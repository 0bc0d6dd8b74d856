"""Host fp64 regularisation-parameter selection on the projected problem.

Semantics are the reference's (ctkrylov/regparam.py): a 200-point geometric
grid over [max(s_min * 1e-4, 1e-12), s_max] (regparam.py:28-36), Tikhonov
filter factors s^2/(s^2+lam^2) on the SVD-rotated right-hand side
(regparam.py:46-70), the L-curve corner as the maximum finite-difference
curvature with ties toward larger lambda (regparam.py:82-107), and the GCV
grid minimum with ties toward larger lambda (regparam.py:110-134).

The evaluation is vectorised over the whole grid (one (grid x k) array pass
instead of the reference's 200-iteration Python loop, which costs ~5 ms per
iteration and would dominate a GPU iteration); the result is the same grid
point.  This stays on the host in fp64, as the north star prescribes.
"""

from __future__ import annotations

import numpy as np

DEFAULT_GRID_COUNT = 200
LAMBDA_FLOOR = 1e-12
CURVATURE_FLOOR = 1e-9


class DegenerateCurveError(RuntimeError):
    """The selection curve carries no usable information (regparam.py:24-25)."""


def svd_of_hessenberg(hess: np.ndarray):
    """Thin SVD, s descending: (s, U, V) like ctkrylov/arnoldi.py:133-141."""
    u, s, vt = np.linalg.svd(np.asarray(hess, dtype=np.float64), full_matrices=False)
    return s, u, vt.T


def lambda_grid(singular_values: np.ndarray, count: int = DEFAULT_GRID_COUNT) -> np.ndarray:
    s = np.asarray(singular_values, dtype=np.float64)
    top = float(s.max(initial=0.0))
    if top <= 0.0:
        raise DegenerateCurveError("all singular values are zero")
    floor_ = max(float(s[s > 0].min()) * 1e-4, LAMBDA_FLOOR)
    return np.geomspace(floor_, top, count)


def _rotated_rhs(s, u, beta):
    c = beta * np.asarray(u, dtype=np.float64)[0, :]
    outside = max(beta * beta - float(c @ c), 0.0)   # part of beta*e1 outside range(H)
    return c, outside


def _grid_norms(s, c, outside, grid):
    """(||y_lam||^2, ||H y_lam - beta e1||^2) for every lam in grid."""
    lam2 = (grid * grid)[:, None]
    denom = s * s + lam2
    sol_sq = np.sum((s * c / denom) ** 2, axis=1)
    res_sq = np.sum(((lam2 / denom) * c) ** 2, axis=1) + outside
    return sol_sq, res_sq, denom


def _last_arg(values, pick):
    """Index of the min/max, ties broken toward the LARGEST lambda."""
    rev = values[::-1]
    return len(values) - 1 - int(pick(rev))


def gcv_from_svd(s, u, beta, grid) -> float:
    c, outside = _rotated_rhs(s, u, beta)
    _, res_sq, denom = _grid_norms(s, c, outside, grid)
    trace = u.shape[0] - np.sum(s * s / denom, axis=1)
    if np.any(trace <= 0.0):
        raise DegenerateCurveError("GCV trace underflow")
    vals = res_sq / (trace * trace)
    if not np.all(np.isfinite(vals)):
        raise DegenerateCurveError("GCV values are non-finite")
    return float(grid[_last_arg(vals, np.argmin)])


def lcurve_from_svd(s, u, beta, grid) -> float:
    if not np.any(s > 0):
        raise DegenerateCurveError("all singular values are zero")
    if len(grid) < 5:
        raise DegenerateCurveError(f"need at least 5 L-curve points, got {len(grid)}")
    c, outside = _rotated_rhs(s, u, beta)
    sol_sq, res_sq, _ = _grid_norms(s, c, outside, grid)
    xr = 0.5 * np.log(np.maximum(res_sq, 1e-300))
    ys = 0.5 * np.log(np.maximum(sol_sq, 1e-300))
    dx, dy = np.gradient(xr), np.gradient(ys)
    ddx, ddy = np.gradient(dx), np.gradient(dy)
    with np.errstate(divide="ignore", invalid="ignore"):
        kappa = (dx * ddy - dy * ddx) / (dx * dx + dy * dy) ** 1.5
    ok = np.isfinite(kappa)
    if not np.any(ok):
        raise DegenerateCurveError("curvature is non-finite everywhere")
    kappa = np.where(ok, kappa, -np.inf)
    if np.max(kappa) <= CURVATURE_FLOOR:
        raise DegenerateCurveError("L-curve has no corner (curvature flat)")
    return float(grid[_last_arg(kappa, np.argmax)])


def select_lambda(hess: np.ndarray, beta: float, strategy: str,
                  fixed_value: float | None = None, grid_count: int = DEFAULT_GRID_COUNT,
                  svd=None) -> float:
    """Dispatch as ctkrylov/regparam.py:137-158; ``svd`` may carry a
    precomputed (s, U, V) of ``hess`` so the Tikhonov solve can reuse it."""
    if strategy == "none":
        return 0.0
    if strategy == "fixed":
        if fixed_value is None or fixed_value < 0:
            raise ValueError("fixed lambda strategy requires a nonnegative value")
        return float(fixed_value)
    s, u, _ = svd if svd is not None else svd_of_hessenberg(hess)
    grid = lambda_grid(s, grid_count)
    if strategy == "lcurve":
        return lcurve_from_svd(s, u, beta, grid)
    if strategy == "gcv":
        return gcv_from_svd(s, u, beta, grid)
    raise ValueError(f"unknown lambda strategy {strategy!r}")


# ---- the reference's public pieces of the selector (ctkrylov/regparam.py:40-134),
# restated on the vectorised helpers above (same values, same tie rules).

class LCurvePoint:
    """One L-curve sample (ctkrylov/regparam.py:40-43)."""

    __slots__ = ("lam", "log_residual", "log_solution")

    def __init__(self, lam: float, log_residual: float, log_solution: float):
        self.lam, self.log_residual, self.log_solution = lam, log_residual, log_solution


def tikhonov_curve_points(singular_values, left_factor, beta, grid) -> list[LCurvePoint]:
    """The projected Tikhonov L-curve on a lambda grid (regparam.py:63-79)."""
    s = np.asarray(singular_values, dtype=np.float64)
    if not np.any(s > 0):
        raise DegenerateCurveError("all singular values are zero")
    grid = np.asarray(grid, dtype=np.float64)
    c, outside = _rotated_rhs(s, left_factor, beta)
    sol_sq, res_sq, _ = _grid_norms(s, c, outside, grid)
    return [LCurvePoint(float(l), 0.5 * np.log(max(r, 1e-300)), 0.5 * np.log(max(x, 1e-300)))
            for l, r, x in zip(grid, res_sq, sol_sq)]


def lcurve_corner(points) -> float:
    """Maximum signed curvature, ties toward larger lambda (regparam.py:82-107)."""
    if len(points) < 5:
        raise DegenerateCurveError(f"need at least 5 L-curve points, got {len(points)}")
    xr = np.array([p.log_residual for p in points])
    ys = np.array([p.log_solution for p in points])
    dx, dy = np.gradient(xr), np.gradient(ys)
    ddx, ddy = np.gradient(dx), np.gradient(dy)
    with np.errstate(divide="ignore", invalid="ignore"):
        kappa = (dx * ddy - dy * ddx) / (dx * dx + dy * dy) ** 1.5
    ok = np.isfinite(kappa)
    if not np.any(ok):
        raise DegenerateCurveError("curvature is non-finite everywhere")
    kappa = np.where(ok, kappa, -np.inf)
    if np.max(kappa) <= CURVATURE_FLOOR:
        raise DegenerateCurveError("L-curve has no corner (curvature flat)")
    return float(points[_last_arg(kappa, np.argmax)].lam)


def gcv_values(singular_values, left_factor, beta, grid) -> np.ndarray:
    """GCV function res^2 / (k+1 - sum f_i)^2 on the grid (regparam.py:110-125)."""
    s = np.asarray(singular_values, dtype=np.float64)
    u = np.asarray(left_factor, dtype=np.float64)
    grid = np.asarray(grid, dtype=np.float64)
    c, outside = _rotated_rhs(s, u, beta)
    _, res_sq, denom = _grid_norms(s, c, outside, grid)
    trace = u.shape[0] - np.sum(s * s / denom, axis=1)
    if np.any(trace <= 0.0):
        raise DegenerateCurveError("GCV trace underflow")
    return res_sq / (trace * trace)


def gcv_minimize(singular_values, left_factor, beta, grid) -> float:
    """Grid minimiser of gcv_values, ties toward larger lambda (regparam.py:128-134)."""
    vals = gcv_values(singular_values, left_factor, beta, grid)
    if not np.all(np.isfinite(vals)):
        raise DegenerateCurveError("GCV values are non-finite")
    return float(np.asarray(grid, dtype=np.float64)[_last_arg(vals, np.argmin)])
