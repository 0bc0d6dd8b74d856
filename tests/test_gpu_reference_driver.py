"""The UNMODIFIED reference driver on the GPU operators.

ctkrylov.gmres.run_gmres (installed untouched into baseline/_ref with
``pip install --target baseline/_ref``) is handed this package's
forward_ray_driven / back_pixel_driven operators -- the drop-in seam of
SURVEY row (b): ``LinearOperator(rows, cols, apply)`` with fp64 numpy in and
out (reference ctkrylov/linop.py:20-60, gmres.py:160-209).  Every projector
apply inside the reference's own loop then runs K1 / K2 on the B200.  Bars:
those of test_gpu_gmres.test_c1_ab_hybrid_gcv_50 against the reference's
own c1 run (tests/golden/c1.npz).
"""

import os
import sys

import numpy as np
import pytest

from paper_2602_17892_b200 import _native, ct, problems

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def reference_gmres():
    if not os.path.isdir(os.path.join(REF, "ctkrylov")):
        pytest.skip("unmodified reference not installed in baseline/_ref "
                    "(pip install --no-index --no-deps --target baseline/_ref <reference>)")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    import ctkrylov.gmres as rg
    assert os.path.dirname(rg.__file__).startswith(REF)
    return rg


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b)


def test_reference_run_gmres_on_gpu_projectors_c1(cuda, golden):
    rg = reference_gmres()
    spec = problems.CONFIGS["c1"]
    z = golden("c1")
    b, _ = problems.add_noise(z["Ax_true"], spec.noise, spec.noise_seed)
    b = b.astype(np.float32).astype(np.float64)
    grid = ct.ImageGrid(spec.N, spec.N, 1.0)
    geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    A, B = ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom)
    launches = _native.launch_counter()
    res = rg.run_gmres(A, B, b, rg.SolverConfig(method="ab-hybrid", lambda_strategy="gcv",
                                                max_iter=50))
    # 50 iterations x (2 A + 2 B) + the cycle start, all on the device
    assert _native.launch_counter() - launches >= 4 * 50
    assert res.stop_reason == "maxiter" and len(res.records) == 50
    rec = lambda f: np.array([getattr(r, f) for r in res.records])  # noqa: E731
    lam, lam_ref = rec("lambda_used"), z["rec/lambda_used"]
    assert np.all(np.abs(lam / lam_ref - 1.0) <= 0.01), np.abs(lam / lam_ref - 1).max()
    for f in ("data_residual_norm", "residual_norm", "proj_residual_norm", "solution_norm"):
        np.testing.assert_allclose(rec(f), z[f"rec/{f}"], rtol=1e-4, err_msg=f)
    assert rel(res.x, z["x_final"]) <= 1e-3


def test_reference_run_gmres_on_gpu_projectors_c2_plain(cuda, golden):
    rg = reference_gmres()
    spec = problems.CONFIGS["c2"]
    z = golden("c2")
    b, _ = problems.add_noise(z["Ax_true"], spec.noise, spec.noise_seed)
    b = b.astype(np.float32).astype(np.float64)
    grid = ct.ImageGrid(spec.N, spec.N, 1.0)
    geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    A, B = ct.forward_ray_driven(grid, geom), ct.back_pixel_driven(grid, geom)
    res = rg.run_gmres(A, B, b, rg.SolverConfig(method="ba", max_iter=80))
    assert len(res.records) == 80
    got = np.array([r.data_residual_norm for r in res.records])
    np.testing.assert_allclose(got, z["plain/rec/data_residual_norm"], rtol=1e-3)
    assert rel(res.x, z["plain/x_final"]) <= 1e-3
