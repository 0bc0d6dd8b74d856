"""Row f4 on-disk formats (CPU): the PGM / image-CSV / records-CSV / manifest
writers reproduce, byte for byte, files the unmodified reference wrote
(tests/golden/problem_io.npz, made by tests/golden/make_golden.py io)."""

import json
import math

import numpy as np

from paper_2602_17892_b200 import ct, experiment
from paper_2602_17892_b200.gmres import IterationRecord, SolveResult, SolverConfig


def _bytes(arr):
    return np.asarray(arr, dtype=np.uint8).tobytes()


def _read(path):
    with open(path, "rb") as f:
        return f.read()


def synthetic_result():
    # same values as make_golden.synthetic_result (reference dataclasses there)
    recs = [
        IterationRecord(1, 0.125, 3.5, 2.25, 1.0 / 3.0, 7.0, None, None, 0.5, False),
        IterationRecord(2, 1.7e-08, 1e-300, 2.0 ** -30, 0.0, 1e300, 0.9, 0.25, 1.25, True),
        IterationRecord(3, float("nan"), 4.0, float("inf"), 5.0, 6.0, 0.1, -0.5, 2.0, False),
    ]
    return SolveResult(np.arange(12.0), recs, "maxiter", 1)


def test_pgm_and_image_csv_bytes(golden, tmp_path):
    d = golden("problem_io")
    img = d["io/img"].ravel()
    ct.write_pgm(tmp_path / "a.pgm", img, (5, 7))
    assert _read(tmp_path / "a.pgm") == _bytes(d["io/pgm_auto"])
    ct.write_pgm(tmp_path / "b.pgm", img, (5, 7), (-0.5, 1.5))
    assert _read(tmp_path / "b.pgm") == _bytes(d["io/pgm_window"])
    ct.write_pgm(tmp_path / "c.pgm", np.ones(35), (5, 7))
    assert _read(tmp_path / "c.pgm") == _bytes(d["io/pgm_flat"])
    ct.write_csv_image(tmp_path / "i.csv", img, (5, 7))
    assert _read(tmp_path / "i.csv") == _bytes(d["io/csv_image"])


def test_records_csv_bytes(golden, tmp_path):
    d = golden("problem_io")
    res = synthetic_result()
    for method in ("ab-hybrid", "ba", "lsmr-hybrid"):
        for tim in (False, True):
            p = tmp_path / f"{method}_{tim}.csv"
            experiment.write_records_csv(p, res, method, tim)
            assert _read(p) == _bytes(d[f"io/records/{method}/{int(tim)}"]), (method, tim)
    cols = experiment.read_records_csv(tmp_path / "ba_True.csv")
    assert tuple(cols) == experiment.CSV_COLUMNS
    assert np.isnan(cols["rre"][0]) and cols["rre"][1] == 0.9
    assert cols["ba_residual"][2] == 4.0 and math.isinf(cols["data_residual"][2])


def test_manifest_layout_matches_reference(golden, tmp_path):
    """manifest_dict + write_manifest on the reference run's own records give
    the reference's manifest bytes (paths and timings are the run's)."""
    d = golden("problem_io")
    for label in ("abg", "badp"):
        ref = json.loads(_bytes(d[f"exp/{label}/manifest"]).decode())
        cols = {}
        lines = _bytes(d[f"exp/{label}/csv"]).decode().splitlines()
        head = lines[0].split(",")
        assert tuple(head) == experiment.CSV_COLUMNS
        rows = [ln.split(",") for ln in lines[1:]]
        f = lambda s: float(s) if s else None          # noqa: E731
        recs = []
        for r in rows:
            cols = dict(zip(head, r))
            recs.append(IterationRecord(int(cols["k"]), f(cols["lambda"]),
                                        f(cols["ba_residual"]) or 0.0, f(cols["data_residual"]),
                                        f(cols["proj_residual"]), f(cols["sol_norm"]),
                                        f(cols["rre"]), f(cols["ssim"]), ref["elapsed_s"]))
        res = SolveResult(np.zeros(1), recs, ref["stop_reason"], ref["cycles"])
        cfg = SolverConfig(**{k: v for k, v in ref["config"].items()})
        spec = experiment.ProblemSpec(kind=ref["problem"]["kind"], name=ref["problem"]["name"],
                                      matched=ref["problem"]["matched"])
        man = experiment.manifest_dict(label, cfg, spec, ref["problem"]["noise_norm"], ref["seed"],
                                       res, ref["csv"], ref["images"])
        p = tmp_path / f"{label}.manifest.json"
        experiment.write_manifest(p, man)
        assert _read(p) == _bytes(d[f"exp/{label}/manifest"]), label
