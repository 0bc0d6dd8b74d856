"""Golden fixture on an odd geometry, from the UNMODIFIED reference.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_odd.py

A 37 x 22 image of 0.8-wide pixels, 1.1-wide bins, 25 non-uniform angles (one
exactly 0, one 1e-9 rad off the other axis): A x, B u, A^T u (matched_back),
hybrid BA-GMRES with restarts, plain AB-GMRES and the Golub-Kahan solvers on
the matched pair, all through the reference's public API.  Pins the oracle
and the GPU path away from the BASELINE shapes.  Output:
tests/golden/odd_geometry.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from ctkrylov.ct import (ImageGrid, ParallelGeometry, back_pixel_driven,  # noqa: E402
                         forward_ray_driven, matched_back)
from ctkrylov.gk import run_lsmr, run_lsqr  # noqa: E402
from ctkrylov.gmres import SolverConfig, run_gmres  # noqa: E402

NX, NY, H, SP = 37, 22, 0.8, 1.1


def angles():
    rng = np.random.default_rng(77)
    a = np.sort(rng.uniform(0.05, np.pi - 0.05, 23))
    return np.unique(np.concatenate(([0.0, np.pi / 2 - 1e-9], a)))


def records_arrays(res):
    keys = ("k", "lambda_used", "residual_norm", "data_residual_norm", "proj_residual_norm",
            "solution_norm")
    return {k: np.array([getattr(r, k) for r in res.records], dtype=np.float64) for k in keys}


def main():
    ang = angles()
    D = int(np.ceil(np.hypot(NX, NY) * H / SP)) + 3
    grid, geom = ImageGrid(NX, NY, H), ParallelGeometry(ang, D, SP)
    A, B = forward_ray_driven(grid, geom), back_pixel_driven(grid, geom)
    At = matched_back(A)
    rng = np.random.default_rng(5)
    x = rng.random(grid.n).astype(np.float32).astype(np.float64)
    u = rng.random(geom.m).astype(np.float32).astype(np.float64)
    out = {"params": np.array([NX, NY, H, D, SP]), "angles": ang, "x": x, "u": u,
           "Ax": A.apply(x), "Bu": B.apply(u), "Atu": At.apply(u)}
    clean = A.apply(x)
    b = clean + 0.02 * np.linalg.norm(clean) / np.sqrt(clean.size) * rng.standard_normal(clean.size)
    b = b.astype(np.float32).astype(np.float64)
    out["b"] = b
    cases = {
        "ba_gcv_restart": (run_gmres, (A, B), dict(method="ba-hybrid", lambda_strategy="gcv",
                                                   max_iter=10, restart_period=4)),
        "ab_plain": (run_gmres, (A, B), dict(method="ab", max_iter=8)),
        "lsqr_gcv": (run_lsqr, (A, At), dict(method="lsqr-hybrid", lambda_strategy="gcv",
                                             max_iter=10)),
        "lsmr_plain": (run_lsmr, (A, At), dict(method="lsmr", max_iter=8)),
        "lsmr_gcv": (run_lsmr, (A, At), dict(method="lsmr-hybrid", lambda_strategy="gcv",
                                             max_iter=10)),
    }
    for name, (run, ops, kw) in cases.items():
        res = run(ops[0], ops[1], b, SolverConfig(**kw))
        out[f"{name}/x"] = res.x
        out[f"{name}/stop"] = np.array(res.stop_reason)
        out[f"{name}/cycles"] = np.int64(res.cycles)
        for k, v in records_arrays(res).items():
            out[f"{name}/rec/{k}"] = v
        print(name, res.stop_reason, len(res.records))
    np.savez_compressed(os.path.join(HERE, "odd_geometry.npz"), **out)


if __name__ == "__main__":
    main()
