"""Experiment outputs: per-iteration CSV, JSON manifest, PGM images (row f4).

Mirrors the on-disk formats of ctkrylov/experiment.py so downstream tooling
reads our runs unchanged: the fixed CSV columns (experiment.py:26-27), the
record writer/reader (experiment.py:194-222), and the per-solver manifest and
image exports of run_experiment (experiment.py:225-289).  Given the same
records the files are byte-identical to the reference's
(tests/test_experiment_io.py against fixtures the reference wrote).

The problem is built on the GPU (ct.make_ct_problem / build_test_problem)
and every solve is the device-resident driver.  The INI front end
(parse_config) and the CLI around it stay out of scope.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field, replace
from pathlib import Path

import numpy as np

from . import ct
from .gk import run_lsmr, run_lsqr
from .gmres import GK_METHODS, GMRES_METHODS, SolveResult, SolverConfig, run_gmres

CSV_COLUMNS = ("k", "lambda", "data_residual", "ba_residual", "proj_residual",
               "sol_norm", "rre", "ssim", "elapsed_s")
OUTPUT_ENV_VAR = "CTKRYLOV_OUT"


class ConfigParseError(ValueError):
    """Invalid experiment description (ctkrylov/experiment.py:31-32)."""


@dataclass
class ProblemSpec:
    """The [problem] section (ctkrylov/experiment.py:35-46); CT kinds only --
    dense test matrices have no projector to put on the GPU."""

    kind: str = "ct"
    name: str = "tp2"
    nx: int | None = None
    angles: int | None = None
    det_count: int | None = None
    noise_level: float | None = None
    matched: bool = False
    seed: int = 0


@dataclass
class ExperimentConfig:
    """ctkrylov/experiment.py:49-56."""

    problem: ProblemSpec
    solvers: list[SolverConfig]
    track_metrics: bool = True
    image_export_stride: int = 0
    out_dir: Path = field(default_factory=lambda: Path("."))
    include_timings: bool = False


@dataclass
class BuiltProblem:
    A: object
    B: object
    b: np.ndarray
    x_true: np.ndarray | None
    noise_norm: float
    image_shape: tuple[int, int] | None
    ct_problem: ct.CtProblem | None = None


def build_problem(spec: ProblemSpec, seed: int | None = None, device: int = 0) -> BuiltProblem:
    """ctkrylov/experiment.py:145-171 for CT problems, generated on the GPU."""
    seed = spec.seed if seed is None else seed
    if spec.kind != "ct":
        raise ConfigParseError(f"problem kind {spec.kind!r} is not supported on the GPU path")
    if spec.name in ct.BUILTIN_PROBLEMS:
        prob = ct.build_test_problem(spec.name, spec.matched, seed, device)
    else:
        if spec.nx is None or spec.angles is None:
            raise ConfigParseError(
                "custom ct problem needs 'nx' and 'angles' (or use a built-in name)")
        prob = ct.make_ct_problem(
            spec.nx, spec.angles, spec.det_count,
            spec.noise_level if spec.noise_level is not None else 0.025,
            seed, spec.matched, spec.name, device)
    return BuiltProblem(prob.forward, prob.back, prob.b_noisy, prob.x_true, prob.noise_norm,
                        (prob.grid.ny, prob.grid.nx), prob)


def run_solver(built: BuiltProblem, cfg: SolverConfig, track_metrics: bool) -> SolveResult:
    """ctkrylov/experiment.py:174-185."""
    if cfg.stopping_rule == "dp" and cfg.noise_norm is None:
        cfg = replace(cfg, noise_norm=built.noise_norm)
    x_true = built.x_true if track_metrics else None
    if cfg.method in GMRES_METHODS:
        return run_gmres(built.A, built.B, built.b, cfg, x_true=x_true,
                         image_shape=built.image_shape)
    if cfg.method in GK_METHODS:
        runner = run_lsqr if cfg.method.startswith("lsqr") else run_lsmr
        return runner(built.A, built.B, built.b, cfg, x_true=x_true,
                      image_shape=built.image_shape)
    raise ConfigParseError(f"unknown solver method {cfg.method!r}")


def _fmt(v) -> str:
    return "" if v is None else repr(float(v))


def write_records_csv(path, result: SolveResult, method: str,
                      include_timings: bool = False) -> None:
    """One row per IterationRecord under CSV_COLUMNS (experiment.py:194-211):
    repr() floats, empty cells for absent values, ``ba_residual`` only for
    methods whose residual lives in image space (BA, LSMR)."""
    ba_like = method.startswith("ba") or method.startswith("lsmr")
    with open(path, "w", encoding="utf-8", newline="\n") as f:
        f.write(",".join(CSV_COLUMNS) + "\n")
        for r in result.records:
            cells = [str(r.k), _fmt(r.lambda_used), _fmt(r.data_residual_norm),
                     _fmt(r.residual_norm) if ba_like else "", _fmt(r.proj_residual_norm),
                     _fmt(r.solution_norm), _fmt(r.rre), _fmt(r.ssim),
                     _fmt(r.elapsed) if include_timings else ""]
            f.write(",".join(cells) + "\n")


def read_records_csv(path) -> dict[str, np.ndarray]:
    """Columns of a records CSV as float arrays, NaN for empty cells."""
    with open(path, encoding="utf-8") as f:
        header = f.readline().strip().split(",")
        rows = [line.strip().split(",") for line in f if line.strip()]
    return {name: np.array([float(row[i]) if row[i] else np.nan for row in rows])
            for i, name in enumerate(header)}


def manifest_dict(label: str, cfg: SolverConfig, problem: ProblemSpec, noise_norm: float,
                  seed: int, result: SolveResult, csv_path, image_paths) -> dict:
    """The per-solver manifest (experiment.py:255-282): same keys, values and
    None-dropping of the solver config (x0 excluded)."""
    rres = [r.rre for r in result.records if r.rre is not None]
    last = result.records[-1]
    return {
        "solver": label,
        "method": cfg.method,
        "config": {k: v for k, v in cfg.__dict__.items() if k != "x0" and v is not None},
        "problem": {"kind": problem.kind, "name": problem.name, "matched": problem.matched,
                    "noise_norm": noise_norm},
        "seed": seed,
        "stop_reason": result.stop_reason,
        "cycles": result.cycles,
        "iterations": len(result.records),
        "min_rre": min(rres) if rres else None,
        "min_rre_iteration": int(np.argmin(rres)) + 1 if rres else None,
        "final": {"data_residual": last.data_residual_norm, "rre": last.rre, "ssim": last.ssim},
        "elapsed_s": last.elapsed,
        "csv": str(csv_path),
        "images": list(image_paths),
    }


def write_manifest(path, manifest: dict) -> None:
    with open(path, "w", encoding="utf-8") as f:
        json.dump(manifest, f, indent=2, sort_keys=True)
        f.write("\n")


def run_experiment(config: ExperimentConfig, seed: int | None = None,
                   device: int = 0) -> list[Path]:
    """Every solver of ``config`` on one GPU-built problem; writes
    ``<label>.csv``, ``<label>_kNNNN.pgm`` snapshots, ``<label>_final.pgm``
    and ``<label>.manifest.json`` per solver (experiment.py:225-289) and
    returns the manifest paths."""
    out_dir = Path(config.out_dir)
    out_dir.mkdir(parents=True, exist_ok=True)
    built = build_problem(config.problem, seed, device)
    actual_seed = config.problem.seed if seed is None else seed
    manifests = []
    for cfg in config.solvers:
        label = cfg.label
        if config.image_export_stride and built.image_shape is not None:
            cfg = replace(cfg, snapshot_stride=config.image_export_stride)
        result = run_solver(built, cfg, config.track_metrics)
        csv_path = out_dir / f"{label}.csv"
        write_records_csv(csv_path, result, cfg.method, config.include_timings)
        image_paths = []
        if built.image_shape is not None:
            window = None
            if built.x_true is not None:
                window = (float(built.x_true.min()), float(built.x_true.max()))
            for k, snap in sorted(result.snapshots.items()):
                p = out_dir / f"{label}_k{k:04d}.pgm"
                ct.write_pgm(p, snap, built.image_shape, window)
                image_paths.append(str(p))
            p = out_dir / f"{label}_final.pgm"
            ct.write_pgm(p, result.x, built.image_shape, window)
            image_paths.append(str(p))
        manifest = manifest_dict(label, cfg, config.problem, built.noise_norm, actual_seed,
                                 result, csv_path, image_paths)
        manifest_path = out_dir / f"{label}.manifest.json"
        write_manifest(manifest_path, manifest)
        manifests.append(manifest_path)
    return manifests


def load_manifest(path) -> dict:
    """ctkrylov/experiment.py:292-304: the manifest plus ``_csv_path``."""
    path = Path(path)
    if not path.exists():
        raise FileNotFoundError(f"manifest not found: {path}")
    with open(path, encoding="utf-8") as f:
        manifest = json.load(f)
    csv_path = Path(manifest["csv"])
    if not csv_path.is_absolute():
        csv_path = path.parent / csv_path.name
    if not csv_path.exists():
        raise FileNotFoundError(f"CSV referenced by manifest not found: {csv_path}")
    manifest["_csv_path"] = csv_path
    return manifest


def default_out_dir() -> Path:
    return Path(os.environ.get(OUTPUT_ENV_VAR, "."))
