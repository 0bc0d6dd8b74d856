"""GPU parity of row f4: on-device problem generation and experiment outputs.

* K_phantom (ctk_phantom) is bitwise the reference's shepp_logan
  (ctkrylov/ct.py:115-134, golden fixtures) and the harness's random-ellipse
  recipe (the oracle's sampler / problems.random_ellipse_phantom), up to the
  c5 size (2048^2).
* make_ct_problem / build_test_problem on the GPU vs the reference's:
  x_true bitwise, b_clean / b_noisy within the projector bar (1e-5 rel-L2,
  fp32 A), noise_norm to 1e-6.
* ctk_add_noise on fp64 input vs the reference's add_noise: 1e-12 (only the
  norm summation order differs).
* run_experiment end to end vs the reference's files: same manifest keys,
  stop reasons, iteration counts and cycles; records and final PGM within
  the solver parity bars.
"""

import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_2602_17892_b200 import ct, experiment, problems
from paper_2602_17892_b200.gmres import SolverConfig

pytestmark = pytest.mark.gpu


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_shepp_logan_bitwise(cuda, golden):
    d = golden("problem_io")
    for nx, h in ((64, 2.0 / 64), (33, 0.37), (128, 1.0)):
        img = ct.shepp_logan(ct.ImageGrid(nx, nx, h))
        np.testing.assert_array_equal(img, d[f"sl/{nx}"], err_msg=f"{nx}")


def test_shepp_logan_nonsquare_rejected(cuda):
    with pytest.raises(ct.GeometryError):
        ct.shepp_logan(ct.ImageGrid(8, 6, 1.0))


@pytest.mark.parametrize("N,E,seed", [(256, 10, 0), (1024, 20, 0), (2048, 10, 63)])
def test_random_ellipse_phantom_bitwise(cuda, N, E, seed):
    img64, img32 = problems.random_ellipse_phantom_device(N, E, seed)
    host = problems.random_ellipse_phantom(N, E, seed)
    np.testing.assert_array_equal(img32.double().cpu().numpy(), host)
    rows = [(rho, a, b, cx, cy, phi) for cx, cy, a, b, phi, rho in problems.ellipse_params(N, E, seed)]
    if N <= 1024:
        np.testing.assert_array_equal(img64.cpu().numpy(), O.phantom(N, N, 1.0, rows))


def test_phantom_nonsquare_grid_against_oracle(cuda):
    rows = [(0.7, 3.0, 1.5, 0.5, -1.0, 0.3), (-0.2, 2.0, 2.5, -1.0, 0.25, 2.0)]
    grid = ct.ImageGrid(13, 9, 0.6)
    img64, img32 = ct.phantom_device(grid, rows)
    np.testing.assert_array_equal(img64.cpu().numpy(), O.phantom(13, 9, 0.6, rows))
    assert img64.abs().sum().item() > 0


def test_make_ct_problem_matches_reference(cuda, golden):
    d = golden("problem_io")
    prob = ct.make_ct_problem(32, 20, 45, 0.025, seed=3)
    np.testing.assert_array_equal(prob.x_true, d["mk/x_true"])
    assert rel(prob.b_clean, d["mk/b_clean"]) <= 1e-5
    assert rel(prob.b_noisy, d["mk/b_noisy"]) <= 1e-5
    assert abs(prob.noise_norm / float(d["mk/noise_norm"]) - 1) <= 1e-6
    # exact relative level of the noise actually added
    e = prob.b_noisy - prob.b_clean
    assert abs(np.linalg.norm(e) / np.linalg.norm(prob.b_clean) - 0.025) <= 1e-6
    assert prob.m == 20 * 45 and prob.n == 32 * 32
    assert prob.b_noisy_device.numel() == prob.m


def test_build_test_problem_tp2(cuda, golden):
    d = golden("problem_io")
    prob = ct.build_test_problem("tp2", seed=0)
    assert rel(prob.b_noisy, d["tp2/b_noisy"]) <= 1e-5
    assert abs(prob.noise_norm / float(d["tp2/noise_norm"]) - 1) <= 1e-6
    with pytest.raises(ct.GeometryError):
        ct.build_test_problem("tp9")


def test_add_noise_fp64_input(cuda, golden):
    d = golden("problem_io")
    b, nn = ct.add_noise(d["mk/b_clean"], 0.025, 3)
    assert rel(b, d["mk/b_noisy"]) <= 1e-12
    assert abs(nn / float(d["mk/noise_norm"]) - 1) <= 1e-12
    b0, n0 = ct.add_noise(d["mk/b_clean"], 0.0, 3)
    np.testing.assert_array_equal(b0, d["mk/b_clean"])
    assert n0 == 0.0
    with pytest.raises(ValueError):
        ct.add_noise(d["mk/b_clean"], -0.1, 3)


def test_add_noise_large_device(cuda):
    torch = cuda
    m = 5_214_600                                   # c5 sinogram
    rng = np.random.default_rng(2)
    bc = torch.from_numpy(rng.random(m).astype(np.float32)).cuda()
    b64, b32, nn = ct.add_noise_device(bc, 0.01, 1000)
    ref, nref = O.add_noise(bc.double().cpu().numpy(), 0.01, 1000)
    assert rel(b64.cpu().numpy(), ref) <= 1e-12
    assert abs(nn / nref - 1) <= 1e-12
    np.testing.assert_array_equal(b32.cpu().numpy(), b64.cpu().numpy().astype(np.float32))


def _csv_cols(raw):
    lines = raw.decode().splitlines()
    head = lines[0].split(",")
    rows = [ln.split(",") for ln in lines[1:]]
    return head, {h: np.array([float(r[i]) if r[i] else np.nan for r in rows])
                  for i, h in enumerate(head)}


def test_run_experiment_matches_reference(cuda, golden, tmp_path):
    d = golden("problem_io")
    spec = experiment.ProblemSpec(kind="ct", name="custom", nx=24, angles=18, det_count=35,
                                  noise_level=0.02, seed=4)
    solvers = [SolverConfig(method="ab-hybrid", lambda_strategy="gcv", max_iter=8, name="abg"),
               SolverConfig(method="ba", max_iter=6, stopping_rule="dp", name="badp")]
    cfg = experiment.ExperimentConfig(spec, solvers, track_metrics=True, image_export_stride=3,
                                      out_dir=tmp_path)
    paths = experiment.run_experiment(cfg)
    assert [p.name for p in paths] == ["abg.manifest.json", "badp.manifest.json"]
    for p in paths:
        man = json.loads(p.read_text())
        label = man["solver"]
        ref = json.loads(np.asarray(d[f"exp/{label}/manifest"], np.uint8).tobytes().decode())
        assert sorted(man) == sorted(ref)
        for k in ("solver", "method", "config", "seed", "stop_reason", "cycles", "iterations",
                  "min_rre_iteration"):
            if k == "config":
                assert {a: b for a, b in man[k].items() if a != "noise_norm"} == \
                    {a: b for a, b in ref[k].items() if a != "noise_norm"}
            else:
                assert man[k] == ref[k], k
        assert man["problem"]["kind"] == ref["problem"]["kind"]
        assert abs(man["problem"]["noise_norm"] / ref["problem"]["noise_norm"] - 1) <= 1e-5
        assert abs(man["final"]["data_residual"] / ref["final"]["data_residual"] - 1) <= 1e-4
        assert abs(man["final"]["rre"] / ref["final"]["rre"] - 1) <= 1e-4
        assert abs(man["min_rre"] / ref["min_rre"] - 1) <= 1e-4
        assert [p.split("/")[-1] for p in man["images"]] == \
            [p.split("/")[-1] for p in ref["images"]]
        head, ours = _csv_cols((tmp_path / f"{label}.csv").read_bytes())
        rhead, theirs = _csv_cols(np.asarray(d[f"exp/{label}/csv"], np.uint8).tobytes())
        assert head == rhead
        for col in ("data_residual", "ba_residual", "sol_norm", "rre", "ssim"):
            a, b = ours[col], theirs[col]
            assert np.array_equal(np.isnan(a), np.isnan(b)), col
            ok = ~np.isnan(b)
            assert np.all(np.abs(a[ok] - b[ok]) <= 1e-4 * np.abs(b[ok]) + 1e-7), col
        pg = (tmp_path / f"{label}_final.pgm").read_bytes()
        rpg = np.asarray(d[f"exp/{label}/final_pgm"], np.uint8).tobytes()
        hdr = b"P5\n24 24\n65535\n"
        assert pg[:len(hdr)] == hdr == rpg[:len(hdr)]
        a = np.frombuffer(pg[len(hdr):], ">u2").astype(np.int64)
        b = np.frombuffer(rpg[len(hdr):], ">u2").astype(np.int64)
        assert np.max(np.abs(a - b)) <= 8            # 65535 levels; x within 1e-4
