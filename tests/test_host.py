"""Host-side logic of the product (CPU): geometry contract, solver config,
fp64 lambda selection / projected solves, input synthesis, metrics."""

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_17892_b200 import arnoldi, ct, dist, gmres, metrics, problems, regparam
from paper_2602_17892_b200.linop import LinearOperator, OperatorShapeError, compose


class TestGeometryContract:
    """ctkrylov/ct.py:37-96 validation, mirrored (tests/test_ct.py:254-265)."""

    def test_angles_must_increase(self):
        with pytest.raises(ct.GeometryError):
            ct.ParallelGeometry(np.array([0.5, 0.4]), 4, 1.0)

    def test_angles_below_pi(self):
        with pytest.raises(ct.GeometryError):
            ct.ParallelGeometry(np.array([0.0, np.pi]), 4, 1.0)

    def test_grid_positive(self):
        with pytest.raises(ct.GeometryError):
            ct.ImageGrid(0, 4)

    def test_detector_positive(self):
        with pytest.raises(ct.GeometryError):
            ct.ParallelGeometry(np.array([0.0]), 0, 1.0)

    def test_extent_and_offsets(self):
        g = ct.ImageGrid(6, 4, 0.5)
        assert g.extent == (-1.5, 1.5, -1.0, 1.0)
        X, Y = g.pixel_centers()
        assert X.shape == (4, 6) and Y[0, 0] > Y[-1, 0]        # row 0 is the top
        p = ct.ParallelGeometry(np.arange(3) * np.pi / 3, 5, 0.7)
        np.testing.assert_allclose(p.bin_offsets(), (np.arange(5) - 2) * 0.7)
        assert p.m == 15

    def test_trig_tables_are_numpy_scalar_values(self):
        p = ct.ParallelGeometry(np.arange(180) * np.pi / 180, 3, 1.0)
        c, s = ct.trig_tables(p)
        assert all(c[i] == np.cos(float(p.angles[i])) for i in range(180))
        assert abs(c[90]) < 1e-14 and s[0] == 0.0              # degenerate angles exist


class TestLinearOperator:
    def test_contract(self):
        op = LinearOperator(2, 3, lambda v: np.array([v.sum(), v[0]]))
        out = op.apply([1, 2, 3])
        assert out.dtype == np.float64 and out.shape == (2,)
        with pytest.raises(OperatorShapeError):
            op.apply(np.ones(2))
        bad = LinearOperator(2, 3, lambda v: np.ones(3))
        with pytest.raises(OperatorShapeError):
            bad.apply(np.ones(3))
        with pytest.raises(OperatorShapeError):
            LinearOperator(0, 3, lambda v: v)

    def test_compose_checks_dims(self):
        a = LinearOperator(2, 3, lambda v: v[:2])
        b = LinearOperator(3, 4, lambda v: v[:3])
        assert compose(a, b).shape == (2, 4)
        with pytest.raises(OperatorShapeError):
            compose(b, b)

    def test_to_dense(self):
        M = np.arange(6.0).reshape(2, 3)
        np.testing.assert_array_equal(LinearOperator(2, 3, lambda v: M @ v).to_dense(), M)


class TestSolverConfig:
    """ctkrylov/gmres.py:56-92 (tests/test_gmres.py:23-54)."""

    @pytest.mark.parametrize("kw,msg", [
        (dict(method="cgls"), "unknown method"),
        (dict(method="ab-hybrid"), "lambda strategy"),
        (dict(method="ab", lambda_strategy="lcurve"), "-hybrid"),
        (dict(method="ab-hybrid", lambda_strategy="fixed"), "lambda_value"),
        (dict(method="ab", stopping_rule="dp"), "noise_norm"),
        (dict(method="ab", stopping_rule="magic"), "stopping rule"),
        (dict(method="ab", max_iter=0), "max_iter"),
        (dict(method="ab", restart_period=-1), "restart_period"),
    ])
    def test_validation(self, kw, msg):
        with pytest.raises(gmres.ConfigError, match=msg):
            gmres.SolverConfig(**kw).validate()

    def test_label(self):
        cfg = gmres.SolverConfig(method="ba-hybrid", lambda_strategy="gcv", restart_period=5)
        assert cfg.label == "ba-hybrid-gcv-p5"
        assert gmres.SolverConfig(name="mine").label == "mine"

    def test_gk_method_rejected(self):
        with pytest.raises(gmres.ConfigError, match="non-GMRES"):
            gmres.run_gmres(None, None, np.ones(3), gmres.SolverConfig(method="lsqr"))

    def test_device_driver_needs_gpu_operator_pair(self):
        A = LinearOperator(3, 2, lambda v: np.ones(3))
        B = LinearOperator(2, 3, lambda v: np.ones(2))
        with pytest.raises(TypeError, match="GPU projector pair"):
            gmres.run_gmres(A, B, np.ones(3), gmres.SolverConfig(method="ab"))

    def test_dimension_mismatch(self):
        A = LinearOperator(3, 2, lambda v: np.ones(3))
        B = LinearOperator(3, 2, lambda v: np.ones(3))
        with pytest.raises(OperatorShapeError, match="projector pair"):
            gmres.run_gmres(A, B, np.ones(3), gmres.SolverConfig(method="ab"))


def random_hessenbergs(n=60, seed=3):
    rng = np.random.default_rng(seed)
    for _ in range(n):
        k = int(rng.integers(2, 60))
        H = np.triu(rng.standard_normal((k + 1, k)), -1) * np.logspace(0, -rng.uniform(1, 10), k)
        yield H, float(rng.uniform(0.5, 5.0))


class TestLambdaSelection:
    def test_vectorised_selector_matches_reference_loops(self):
        for H, beta in random_hessenbergs():
            for strat in ("gcv", "lcurve"):
                try:
                    ref = O.lambda_selection(H, beta, strat)
                except O.OracleDegenerate:
                    with pytest.raises(regparam.DegenerateCurveError):
                        regparam.select_lambda(H, beta, strat)
                    continue
                assert regparam.select_lambda(H, beta, strat) == ref

    def test_golden_reference_lambdas(self, golden):
        d = golden("solver_cases")
        for i in range(4):
            H = d[f"lam/{i}/H"]
            assert regparam.select_lambda(H, 2.5, "gcv") == d[f"lam/{i}/gcv"]
            assert regparam.select_lambda(H, 2.5, "lcurve") == d[f"lam/{i}/lcurve"]

    def test_degenerate_and_dispatch(self):
        with pytest.raises(regparam.DegenerateCurveError):
            regparam.lambda_grid(np.zeros(3))
        assert regparam.select_lambda(np.ones((2, 1)), 1.0, "none") == 0.0
        assert regparam.select_lambda(np.ones((2, 1)), 1.0, "fixed", 0.5) == 0.5
        with pytest.raises(ValueError):
            regparam.select_lambda(np.ones((2, 1)), 1.0, "magic")
        g = regparam.lambda_grid(np.array([3.0, 1e-20, 0.0]))
        assert g[0] == 1e-12 and g[-1] == 3.0 and len(g) == 200

    def test_projected_solves_match_reference_lstsq(self):
        for H, beta in random_hessenbergs(30, 5):
            for lam in (0.0, 1e-3, 0.2):
                y_ref, r_ref = O.projected_tikhonov(H, beta, lam)
                sol = arnoldi.solve_projected_tikhonov(H, beta, lam)
                scale = max(1.0, np.abs(y_ref).max())
                np.testing.assert_allclose(sol.y, y_ref, atol=1e-8 * scale)
                assert sol.proj_residual_norm == pytest.approx(r_ref, rel=1e-6, abs=1e-12)

    def test_tikhonov_closed_forms(self):
        # arnoldi tests: min (2y - 1)^2 + 4 y^2 -> y = 0.25 (tests/test_arnoldi.py)
        sol = arnoldi.solve_projected_tikhonov(np.array([[2.0], [0.0]]), 1.0, 2.0)
        assert sol.y[0] == pytest.approx(0.25)
        sol = arnoldi.solve_projected_ls(np.array([[1.0], [1.0]]), 2.0)
        assert sol.y[0] == pytest.approx(1.0)
        assert sol.proj_residual_norm == pytest.approx(np.sqrt(2.0))
        assert arnoldi.solve_projected_ls(np.zeros((3, 2)), 1.0).rank_deficient
        with pytest.raises(ValueError):
            arnoldi.solve_projected_tikhonov(np.ones((2, 1)), 1.0, -1.0)

    def test_hessenberg_assembly(self):
        cols = [np.array([1.0, 2.0]), np.array([3.0, 4.0, 5.0])]
        np.testing.assert_array_equal(arnoldi.hessenberg_from_columns(cols, 2),
                                      [[1, 3], [2, 4], [0, 5]])


class TestProblems:
    def test_phantom_is_seeded_and_fp32_representable(self):
        a = problems.random_ellipse_phantom(64, 10, 0)
        b = problems.random_ellipse_phantom(64, 10, 0)
        np.testing.assert_array_equal(a, b)
        np.testing.assert_array_equal(a, a.astype(np.float32).astype(np.float64))
        assert a.min() >= 0 and a.max() > 0.1
        assert not np.array_equal(a, problems.random_ellipse_phantom(64, 10, 1))

    def test_add_noise_exact_level(self):
        rng = np.random.default_rng(0)
        b = rng.standard_normal(500)
        noisy, norm = problems.add_noise(b, 0.02, 7)
        assert np.linalg.norm(noisy - b) / np.linalg.norm(b) == pytest.approx(0.02, abs=1e-14)
        assert norm == 0.02 * np.linalg.norm(b)
        same, _ = problems.add_noise(b, 0.02, 7)
        np.testing.assert_array_equal(noisy, same)
        clean, zero = problems.add_noise(b, 0.0, 1)
        np.testing.assert_array_equal(clean, b)
        assert zero == 0.0

    def test_configs_match_baseline(self):
        c = problems.CONFIGS
        assert (c["c1"].N, c["c1"].n_angles, c["c1"].det_count, c["c1"].max_iter) == (128, 180, 183, 50)
        assert (c["c2"].method, c["c2"].strategy, c["c2"].noise) == ("ba-hybrid", "lcurve", 0.02)
        assert (c["c5"].N, c["c5"].det_count, c["c5"].slices) == (2048, 2897, 64)
        assert problems.slice_seeds(c["c5"], 3) == (3, 1003)


class TestMetrics:
    def test_rre(self):
        assert metrics.rre([1.0, 1.0], [1.0, 0.0]) == pytest.approx(1.0)
        with pytest.raises(ValueError):
            metrics.rre([1.0], [0.0])

    def test_ssim_identity_and_direct_window(self):
        rng = np.random.default_rng(1)
        a = rng.random((12, 12))
        assert metrics.ssim(a, a, (12, 12)) == pytest.approx(1.0)
        b = a + 0.1 * rng.random((12, 12))
        # direct windowed evaluation (independent route, tests/helpers.py:123-146 style)
        L = a.max() - a.min()
        c1, c2 = (0.01 * L) ** 2, (0.03 * L) ** 2
        t = np.arange(8) - 3.5
        g = np.exp(-(t ** 2) / (2 * 1.5 ** 2))
        w = np.outer(g, g) / np.outer(g, g).sum()
        vals = []
        for i in range(5):
            for j in range(5):
                wa, wb = b[i:i + 8, j:j + 8], a[i:i + 8, j:j + 8]
                ma, mb = (w * wa).sum(), (w * wb).sum()
                va, vb = (w * wa * wa).sum() - ma ** 2, (w * wb * wb).sum() - mb ** 2
                cv = (w * wa * wb).sum() - ma * mb
                vals.append(((2 * ma * mb + c1) * (2 * cv + c2)) / ((ma ** 2 + mb ** 2 + c1) * (va + vb + c2)))
        assert metrics.ssim(b, a, (12, 12)) == pytest.approx(np.mean(vals), rel=1e-9)

    def test_stopping_rules(self):
        assert metrics.dp_should_stop(1.0, 1.0, 1.01)
        assert not metrics.dp_should_stop(1.2, 1.0, 1.01)
        assert metrics.rns_should_stop([1.0, 1.0 - 1e-6], 1e-4)
        assert not metrics.rns_should_stop([1.0], 1e-4)
        white = np.random.default_rng(2).standard_normal(4096)
        assert metrics.ncp_distance(white) < 0.05
        assert metrics.ncp_distance(np.sin(np.arange(4096) / 50.0)) > 0.5


class TestShardPlan:
    def test_interleaved_and_blocks_cover_all(self):
        for world in (1, 2, 3, 8):
            for mode in ("interleaved", "blocks"):
                parts = dist.angle_shards(1800, world, mode)
                assert len(parts) == world
                np.testing.assert_array_equal(np.sort(np.concatenate(parts)), np.arange(1800))
                assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1
        with pytest.raises(ValueError):
            dist.angle_shards(3, 4)


def test_matched_back_reference_semantics_on_host_operators():
    """ct.matched_back on non-GPU operators follows ctkrylov/ct.py:248-264:
    CSR transpose when a sparse matrix is attached, else a guarded dense
    transpose (GeometryError past the desk-scale guard)."""
    import scipy.sparse as sp
    from paper_2602_17892_b200 import ct
    from paper_2602_17892_b200.linop import LinearOperator
    rng = np.random.default_rng(0)
    M = rng.standard_normal((7, 5))
    op = LinearOperator(7, 5, lambda v: M @ v)
    At = ct.matched_back(op)
    u = rng.standard_normal(7)
    np.testing.assert_allclose(At.apply(u), M.T @ u)
    op.sparse_matrix = sp.csr_matrix(M)
    np.testing.assert_allclose(ct.matched_back(op).apply(u), M.T @ u)
    big = LinearOperator(5000, 4000, lambda v: np.zeros(5000))
    with pytest.raises(ct.GeometryError):
        ct.matched_back(big)


# ---- reference API pieces (drop-in names): linop helpers, public regparam functions

def test_dense_operator_and_transpose_contract():
    import pytest as _pt
    from paper_2602_17892_b200 import linop
    m = np.arange(6.0).reshape(2, 3)
    A = linop.dense_operator(m)
    At = linop.transpose_of(m)
    v = np.array([1.0, -2.0, 0.5])
    np.testing.assert_array_equal(A.apply(v), m @ v)
    np.testing.assert_array_equal(At.apply(np.array([1.0, 2.0])), m.T @ np.array([1.0, 2.0]))
    assert A.shape == (2, 3) and At.shape == (3, 2)
    m[0, 0] = 99.0                                     # copied and frozen
    np.testing.assert_array_equal(A.apply(v), np.arange(6.0).reshape(2, 3) @ v)
    with _pt.raises(linop.OperatorShapeError):
        linop.dense_operator(np.ones(3))
    with _pt.raises(ValueError):
        linop.dense_operator(np.array([[np.nan]]))
    with _pt.raises(linop.OperatorShapeError):
        A.apply(np.ones(2))


def test_op_norm_estimate_power_iteration():
    import pytest as _pt
    from paper_2602_17892_b200 import linop
    rng = np.random.default_rng(3)
    q, _ = np.linalg.qr(rng.standard_normal((6, 6)))
    m = q @ np.diag([5.0, 2.0, 1.0, 0.5, 0.1, 0.0]) @ q.T
    est = linop.op_norm_estimate(linop.dense_operator(m), iterations=200, seed=0)
    assert est == _pt.approx(5.0, rel=1e-10)
    assert linop.op_norm_estimate(linop.dense_operator(np.zeros((3, 3)))) == 0.0
    with _pt.raises(linop.OperatorShapeError):
        linop.op_norm_estimate(linop.dense_operator(np.ones((2, 3))))


def test_public_regparam_pieces_match_reference_selection(golden):
    """gcv_minimize / lcurve_corner(tikhonov_curve_points) reproduce the
    reference's select_lambda values stored in the golden fixture."""
    from paper_2602_17892_b200 import regparam as R
    d = golden("solver_cases")
    for i in range(4):
        H = d[f"lam/{i}/H"]
        s, u, _ = R.svd_of_hessenberg(H)
        grid = R.lambda_grid(s)
        assert R.gcv_minimize(s, u, 2.5, grid) == float(d[f"lam/{i}/gcv"])
        pts = R.tikhonov_curve_points(s, u, 2.5, grid)
        assert len(pts) == len(grid)
        assert R.lcurve_corner(pts) == float(d[f"lam/{i}/lcurve"])
        vals = R.gcv_values(s, u, 2.5, grid)
        assert vals.shape == grid.shape and np.all(vals > 0)
