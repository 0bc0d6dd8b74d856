"""Generate golden fixtures by running the UNMODIFIED reference.

Run in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Everything below calls the reference's public API (ctkrylov.ct /
ctkrylov.gmres / ctkrylov.regparam); the inputs come from
paper_2602_17892_b200.problems so the GPU tests can regenerate them on the
GPU box without the reference.  Outputs: tests/golden/*.npz (small).
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from ctkrylov.ct import (ImageGrid, ParallelGeometry, back_pixel_driven,  # noqa: E402
                         forward_ray_driven, make_ct_problem)
from ctkrylov.gmres import SolverConfig, run_gmres  # noqa: E402
from ctkrylov.regparam import select_lambda  # noqa: E402

from paper_2602_17892_b200 import problems  # noqa: E402


def geom(nx, ny, h, angles, D, sp):
    return ImageGrid(nx, ny, h), ParallelGeometry(np.asarray(angles, float), D, sp)


def small_angles(k):
    return np.arange(k) * np.pi / k


# Small operator geometries: the reference tests' own (tests/test_ct.py:67-130)
# plus degenerate-angle / non-square / edge-tap cases.
SMALL = {
    "t_siddon_4x4": (4, 4, 0.7, [0.0, 0.9, 2.1], 5, 0.8),          # tests/test_ct.py:67-72
    "t_back_5x4": (5, 4, 0.6, small_angles(4), 7, 0.5),             # tests/test_ct.py:126-130
    "t_unmatched_8x8": (8, 8, 0.3, small_angles(6), 11, 0.35),      # tests/test_ct.py:132-138
    "t_single_bin_6x6": (6, 6, 0.4, [0.7], 9, 0.4),                 # tests/test_ct.py:116-124
    "t_center_ray": (8, 8, 0.5, [0.0], 1, 0.5),                     # tests/test_ct.py:53-58
    "t_diag_ray": (6, 6, 1.0, [np.pi / 4], 1, 1.0),                 # tests/test_ct.py:60-65
    "t_miss": (4, 4, 0.5, [0.0], 3, 10.0),                          # tests/test_ct.py:95-99
    "axis_16": (16, 16, 1.0, small_angles(8), 23, 1.0),             # integer offsets, 0/45/90 deg
    "nonsquare_7x5": (7, 5, 0.5, small_angles(6), 9, 0.45),
    "edge_taps_6x6": (6, 6, 1.0, small_angles(5), 5, 1.0),          # detector narrower than image
    "wide_12x10": (12, 10, 0.8, np.sort(np.random.default_rng(5).uniform(0, np.pi, 9)), 17, 0.7),
}


def make_small():
    out = {}
    rng = np.random.default_rng(123)
    for name, (nx, ny, h, ang, D, sp) in SMALL.items():
        g, p = geom(nx, ny, h, ang, D, sp)
        A = forward_ray_driven(g, p)
        B = back_pixel_driven(g, p)
        x = rng.random(g.n).astype(np.float32).astype(np.float64)
        u = rng.random(p.m).astype(np.float32).astype(np.float64)
        out[f"{name}/params"] = np.array([nx, ny, h, D, sp], dtype=np.float64)
        out[f"{name}/angles"] = p.angles
        out[f"{name}/A_dense"] = A.to_dense()
        out[f"{name}/B_dense"] = B.to_dense()
        out[f"{name}/x"] = x
        out[f"{name}/u"] = u
        out[f"{name}/Ax"] = A.apply(x)
        out[f"{name}/Bu"] = B.apply(u)
    np.savez_compressed(os.path.join(HERE, "small_ops.npz"), **out)
    print("small_ops.npz", len(SMALL), "geometries")


def config_problem(spec):
    g, p = geom(spec.N, spec.N, 1.0, spec.angles(), spec.det_count, 1.0)
    t0 = time.time()
    A = forward_ray_driven(g, p)
    B = back_pixel_driven(g, p)
    print(f"{spec.name}: build {time.time() - t0:.1f}s nnz={A.sparse_matrix.nnz}")
    return g, p, A, B


def records_arrays(res):
    fields = ("k", "lambda_used", "residual_norm", "data_residual_norm",
              "proj_residual_norm", "solution_norm")
    arr = {f: np.array([getattr(r, f) for r in res.records], dtype=np.float64) for f in fields}
    arr["lambda_warning"] = np.array([r.lambda_warning for r in res.records], dtype=bool)
    return arr


def make_config(name, solve=True, extra_plain=False):
    spec = problems.CONFIGS[name]
    g, p, A, B = config_problem(spec)
    out = {"nnz": np.int64(A.sparse_matrix.nnz)}
    x_true = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
    u = problems.uniform_sinogram(p.m, 1)
    ximg = problems.uniform_image(g.n, 0)
    out["Ax_true"] = A.apply(x_true)
    out["Ax_uniform"] = A.apply(ximg)
    out["Bu_uniform"] = B.apply(u)
    if solve:
        b, noise_norm = problems.add_noise(out["Ax_true"], spec.noise, spec.noise_seed)
        out["noise_norm"] = np.float64(noise_norm)
        b32 = b.astype(np.float32).astype(np.float64)
        cfg = SolverConfig(method=spec.method, lambda_strategy=spec.strategy,
                           max_iter=spec.max_iter)
        t0 = time.time()
        res = run_gmres(A, B, b32, cfg)
        print(f"{name}: {spec.method}/{spec.strategy} K={spec.max_iter} {time.time() - t0:.1f}s "
              f"stop={res.stop_reason}")
        out["x_final"] = res.x.astype(np.float32)
        for k, v in records_arrays(res).items():
            out[f"rec/{k}"] = v
        if extra_plain:
            cfg = SolverConfig(method=spec.method.replace("-hybrid", ""), max_iter=spec.max_iter)
            res = run_gmres(A, B, b32, cfg)
            out["plain/x_final"] = res.x.astype(np.float32)
            for k, v in records_arrays(res).items():
                out[f"plain/rec/{k}"] = v
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(f"{name}.npz written")


def make_solver_cases():
    """Small CT solves through every driver branch (tests/test_acceptance.py:142-172 problem)."""
    prob = make_ct_problem(16, 12, 23, 0.02, 0)
    out = {"b": prob.b_noisy, "noise_norm": np.float64(prob.noise_norm),
           "A_dense": prob.forward.to_dense(), "B_dense": prob.back.to_dense()}
    cases = {
        "ab_plain": dict(method="ab", max_iter=12),
        "ba_plain": dict(method="ba", max_iter=12),
        "ab_gcv": dict(method="ab-hybrid", lambda_strategy="gcv", max_iter=15),
        "ba_gcv": dict(method="ba-hybrid", lambda_strategy="gcv", max_iter=15),
        "ab_lcurve": dict(method="ab-hybrid", lambda_strategy="lcurve", max_iter=15),
        "ba_fixed": dict(method="ba-hybrid", lambda_strategy="fixed", lambda_value=0.3, max_iter=10),
        "ab_restart": dict(method="ab-hybrid", lambda_strategy="gcv", max_iter=14, restart_period=5),
        "ab_dp": dict(method="ab", max_iter=40, stopping_rule="dp", noise_norm=prob.noise_norm),
        "ba_rns": dict(method="ba", max_iter=40, stopping_rule="rns", rns_epsilon=1e-3),
        "ba_ncp": dict(method="ba", max_iter=40, stopping_rule="ncp", ncp_threshold=0.2),
        "ab_ncp": dict(method="ab", max_iter=40, stopping_rule="ncp", ncp_threshold=0.12),
    }
    for name, kw in cases.items():
        res = run_gmres(prob.forward, prob.back, prob.b_noisy, SolverConfig(**kw))
        out[f"{name}/x"] = res.x
        out[f"{name}/stop"] = np.array(res.stop_reason)
        out[f"{name}/cycles"] = np.int64(res.cycles)
        for k, v in records_arrays(res).items():
            out[f"{name}/rec/{k}"] = v
    # Golub-Kahan solvers on the matched pair (ctkrylov/gk.py, ct.py:248-264)
    from ctkrylov.ct import matched_back
    from ctkrylov.gk import run_lsmr, run_lsqr
    At = matched_back(prob.forward)
    gk_cases = {
        "lsqr_plain": dict(method="lsqr", max_iter=12),
        "lsqr_gcv": dict(method="lsqr-hybrid", lambda_strategy="gcv", max_iter=15),
        "lsqr_lcurve": dict(method="lsqr-hybrid", lambda_strategy="lcurve", max_iter=15),
        "lsqr_dp": dict(method="lsqr", max_iter=40, stopping_rule="dp", noise_norm=prob.noise_norm),
        "lsmr_plain": dict(method="lsmr", max_iter=12),
        "lsmr_gcv": dict(method="lsmr-hybrid", lambda_strategy="gcv", max_iter=15),
    }
    for name, kw in gk_cases.items():
        run = run_lsqr if kw["method"].startswith("lsqr") else run_lsmr
        res = run(prob.forward, At, prob.b_noisy, SolverConfig(**kw))
        out[f"{name}/x"] = res.x
        out[f"{name}/stop"] = np.array(res.stop_reason)
        for k, v in records_arrays(res).items():
            out[f"{name}/rec/{k}"] = v
    # lambda selection on random Hessenbergs (ctkrylov/regparam.py:137-158)
    rng = np.random.default_rng(7)
    for i, k in enumerate((3, 8, 20, 45)):
        H = np.triu(rng.standard_normal((k + 1, k)), -1) * np.logspace(0, -6, k)
        out[f"lam/{i}/H"] = H
        out[f"lam/{i}/gcv"] = np.float64(select_lambda(H, 2.5, "gcv"))
        out[f"lam/{i}/lcurve"] = np.float64(select_lambda(H, 2.5, "lcurve"))
    np.savez_compressed(os.path.join(HERE, "solver_cases.npz"), **out)
    print("solver_cases.npz", len(cases), "cases")


def _file_bytes(path):
    with open(path, "rb") as f:
        return np.frombuffer(f.read(), dtype=np.uint8)


def synthetic_result():
    """A fixed SolveResult exercising every CSV cell kind (None, nan, inf,
    tiny/huge magnitudes), built from the reference's own dataclasses."""
    from ctkrylov.gmres import IterationRecord, SolveResult
    recs = [
        IterationRecord(1, 0.125, 3.5, 2.25, 1.0 / 3.0, 7.0, None, None, 0.5, False),
        IterationRecord(2, 1.7e-08, 1e-300, 2.0 ** -30, 0.0, 1e300, 0.9, 0.25, 1.25, True),
        IterationRecord(3, float("nan"), 4.0, float("inf"), 5.0, 6.0, 0.1, -0.5, 2.0, False),
    ]
    return SolveResult(np.arange(12.0), recs, "maxiter", 1)


def make_io():
    """Row f4 fixtures: the reference's phantom, problem builder and writers."""
    import json
    import tempfile
    from ctkrylov import ct as rct
    from ctkrylov import experiment as rexp
    from ctkrylov.gmres import SolverConfig as RCfg
    out = {}
    for nx, h in ((64, 2.0 / 64), (33, 0.37), (128, 1.0)):
        out[f"sl/{nx}"] = rct.shepp_logan(rct.ImageGrid(nx, nx, h))
    prob = rct.make_ct_problem(32, 20, 45, 0.025, seed=3)
    for k in ("x_true", "b_clean", "b_noisy"):
        out[f"mk/{k}"] = getattr(prob, k)
    out["mk/noise_norm"] = np.float64(prob.noise_norm)
    tp2 = rct.build_test_problem("tp2", seed=0)
    out["tp2/b_noisy"] = tp2.b_noisy
    out["tp2/noise_norm"] = np.float64(tp2.noise_norm)
    rng = np.random.default_rng(11)
    img = rng.standard_normal((5, 7))
    res = synthetic_result()
    with tempfile.TemporaryDirectory() as d:
        rct.write_pgm(os.path.join(d, "a.pgm"), img.ravel(), (5, 7))
        out["io/img"] = img
        out["io/pgm_auto"] = _file_bytes(os.path.join(d, "a.pgm"))
        rct.write_pgm(os.path.join(d, "b.pgm"), img.ravel(), (5, 7), (-0.5, 1.5))
        out["io/pgm_window"] = _file_bytes(os.path.join(d, "b.pgm"))
        rct.write_pgm(os.path.join(d, "c.pgm"), np.ones(35), (5, 7))
        out["io/pgm_flat"] = _file_bytes(os.path.join(d, "c.pgm"))
        rct.write_csv_image(os.path.join(d, "i.csv"), img.ravel(), (5, 7))
        out["io/csv_image"] = _file_bytes(os.path.join(d, "i.csv"))
        for method in ("ab-hybrid", "ba", "lsmr-hybrid"):
            for tim in (False, True):
                f = os.path.join(d, f"{method}_{tim}.csv")
                rexp.write_records_csv(f, res, method, tim)
                out[f"io/records/{method}/{int(tim)}"] = _file_bytes(f)
        # run_experiment on a small GPU-sized problem: manifest + CSV + PGMs
        spec = rexp.ProblemSpec(kind="ct", name="custom", nx=24, angles=18, det_count=35,
                                noise_level=0.02, seed=4)
        solvers = [RCfg(method="ab-hybrid", lambda_strategy="gcv", max_iter=8, name="abg"),
                   RCfg(method="ba", max_iter=6, stopping_rule="dp", name="badp")]
        cfg = rexp.ExperimentConfig(spec, solvers, track_metrics=True, image_export_stride=3,
                                    out_dir=Path(d))
        for mpath in rexp.run_experiment(cfg):
            label = json.load(open(mpath))["solver"]
            out[f"exp/{label}/manifest"] = _file_bytes(mpath)
            out[f"exp/{label}/csv"] = _file_bytes(os.path.join(d, f"{label}.csv"))
            out[f"exp/{label}/final_pgm"] = _file_bytes(os.path.join(d, f"{label}_final.pgm"))
        out["exp/dir"] = np.frombuffer(d.encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "problem_io.npz"), **out)
    print("problem_io.npz", len(out), "entries")


def make_solver_spread(trials=8, rel=1e-7):
    """The reference's OWN sensitivity to fp32-level input rounding on the
    driver-branch cases: each case re-run by the
    unmodified reference with its operators and data perturbed at the level
    the GPU path computes at -- (a) A, B and b rounded to fp32, (b) `trials`
    random relative perturbations of every entry of A, B and b by `rel`.
    Stored per case: the largest relative deviation, over those runs, of
    every iteration's data-residual norm from the unperturbed run, and of the
    final x.  The GPU test holds its deviation from the reference to a
    multiple of this spread where the spread exceeds the fixed bar (the
    unregularised runs deep in their noise-fitting regime)."""
    from ctkrylov.linop import dense_operator
    prob = make_ct_problem(16, 12, 23, 0.02, 0)
    Ad, Bd, b = prob.forward.to_dense(), prob.back.to_dense(), prob.b_noisy
    cases = {
        "ab_plain": dict(method="ab", max_iter=12),
        "ba_plain": dict(method="ba", max_iter=12),
        "ab_gcv": dict(method="ab-hybrid", lambda_strategy="gcv", max_iter=15),
        "ba_gcv": dict(method="ba-hybrid", lambda_strategy="gcv", max_iter=15),
        "ab_lcurve": dict(method="ab-hybrid", lambda_strategy="lcurve", max_iter=15),
        "ba_fixed": dict(method="ba-hybrid", lambda_strategy="fixed", lambda_value=0.3, max_iter=10),
        "ab_restart": dict(method="ab-hybrid", lambda_strategy="gcv", max_iter=14, restart_period=5),
        "ab_dp": dict(method="ab", max_iter=40, stopping_rule="dp", noise_norm=prob.noise_norm),
        "ba_rns": dict(method="ba", max_iter=40, stopping_rule="rns", rns_epsilon=1e-3),
        "ba_ncp": dict(method="ba", max_iter=40, stopping_rule="ncp", ncp_threshold=0.2),
        "ab_ncp": dict(method="ab", max_iter=40, stopping_rule="ncp", ncp_threshold=0.12),
    }
    rng = np.random.default_rng(77)
    variants = [(Ad.astype(np.float32).astype(np.float64), Bd.astype(np.float32).astype(np.float64),
                 b.astype(np.float32).astype(np.float64))]
    for _ in range(trials):
        variants.append((Ad * (1 + rel * rng.standard_normal(Ad.shape)),
                         Bd * (1 + rel * rng.standard_normal(Bd.shape)),
                         b * (1 + rel * rng.standard_normal(b.shape))))
    out = {"trials": np.int64(trials), "rel": np.float64(rel)}
    for name, kw in cases.items():
        cfg = SolverConfig(**kw)
        base = run_gmres(dense_operator(Ad), dense_operator(Bd), b, cfg)
        dn0 = np.array([r.data_residual_norm for r in base.records])
        dev = np.zeros(len(dn0))
        devx = 0.0
        for A_, B_, b_ in variants:
            res = run_gmres(dense_operator(A_), dense_operator(B_), b_, cfg)
            dn = np.array([r.data_residual_norm for r in res.records])
            kk = min(len(dn), len(dn0))
            dev[:kk] = np.maximum(dev[:kk], np.abs(dn[:kk] / dn0[:kk] - 1.0))
            if len(dn) != len(dn0):
                dev[kk:] = np.inf                     # stopped at another iteration
            devx = max(devx, float(np.linalg.norm(res.x - base.x) / np.linalg.norm(base.x)))
        out[f"{name}/res_spread"] = dev
        out[f"{name}/x_spread"] = np.float64(devx)
        print(f"{name}: residual spread max {dev.max():.2e} (first 12: {dev[:12].max():.2e}), "
              f"x spread {devx:.2e}")
    np.savez_compressed(os.path.join(HERE, "solver_spread.npz"), **out)


def make_lcurve_band(trials=32, deltas=(1e-15, 1e-12, 1e-7)):
    """c2 L-curve conditioning: run the reference's c2
    hybrid BA-GMRES + L-curve, capture every iteration's Hessenberg at its
    select_lambda call (ctkrylov/gmres.py:197), and re-select lambda with the
    reference's own select_lambda on fp64-rounding-level relative
    (1e-15, 1e-12) and fp32-rounding-level (1e-7, the GPU path computes in
    fp32) relative perturbations H * (1 + delta * xi).  The band [min, max]
    of those lambdas
    is the spread the reference's OWN arithmetic allows; the GPU test asserts
    that every GPU lambda lies inside it (plus 1%)."""
    import ctkrylov.gmres as rg
    spec = problems.CONFIGS["c2"]
    g, p, A, B = config_problem(spec)
    xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
    b, _ = problems.add_noise(A.apply(xt), spec.noise, spec.noise_seed)
    b32 = b.astype(np.float32).astype(np.float64)
    captured = []
    orig = rg.select_lambda

    def spy(H, beta, strategy, fixed=None, *a, **kw):
        lam = orig(H, beta, strategy, fixed, *a, **kw)
        captured.append((np.array(H, dtype=np.float64), float(beta), lam))
        return lam
    rg.select_lambda = spy
    try:
        res = run_gmres(A, B, b32, SolverConfig(method="ba-hybrid", lambda_strategy="lcurve",
                                                max_iter=spec.max_iter))
    finally:
        rg.select_lambda = orig
    rng = np.random.default_rng(2024)
    K = len(captured)
    lo, hi, moved = np.empty(K), np.empty(K), np.zeros((len(deltas), K), dtype=np.int64)
    for k, (H, beta, lam) in enumerate(captured):
        vals = [lam]
        for di, d in enumerate(deltas):
            for _ in range(trials):
                lp = orig(H * (1.0 + d * rng.standard_normal(H.shape)), beta, "lcurve")
                vals.append(lp)
                moved[di, k] += abs(lp / lam - 1.0) > 1e-3
        lo[k], hi[k] = min(vals), max(vals)
    lam_ref = np.array([c[2] for c in captured])
    assert np.array_equal(lam_ref, [r.lambda_used for r in res.records])
    np.savez_compressed(os.path.join(HERE, "c2_lcurve_band.npz"), lam_ref=lam_ref, band_lo=lo,
                        band_hi=hi, moved=moved, deltas=np.array(deltas), trials=np.int64(trials))
    print("c2_lcurve_band.npz: iterations whose corner moves under 1e-15:",
          int(np.sum(moved[0] > 0)), "of", K)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "solver", "c1", "c2", "io"]
    if "io" in which:
        make_io()
    if "small" in which:
        make_small()
    if "solver" in which:
        make_solver_cases()
    if "c1" in which:
        make_config("c1")
    if "c2" in which:
        make_config("c2", extra_plain=True)
    if "lcurve" in which:
        make_lcurve_band()
    if "spread" in which:
        make_solver_spread()
