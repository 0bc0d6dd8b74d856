"""Benchmark: hybrid AB-/BA-GMRES projector path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2]
                    [--impl ours|reference]

Metric (BASELINE.json): A+B projected rays/s through hybrid GMRES, plus
hybrid iterations/s and the HBM-roofline fraction of the dominant kernel.

* A "step" is one full hybrid solve of the workload (c2 by default:
  BA-GMRES + L-curve, 80 iterations, 256^2 image, 360 angles x 363 bins,
  seeded random-ellipse phantom, 2% noise).  Projected rays
  per step = K * (A+B applies per iteration) * m  (BA: 2A+1B, AB: 2A+2B;
  cycle-start applies excluded).
* ``value``: device-resident solve (b already in HBM, x left in HBM), timed
  with CUDA events on the solve stream, L2 flushed (256 MiB write) before
  every timed step.  ``e2e``: the same solve through the public API
  ``run_gmres(A, B, b_numpy, cfg)`` with host b in and host x out, wall-clock
  with the copies inside the timed region.
* ``roofline``: the projector kernel with the largest share of the timed
  region, algorithmic bytes per launch (A: 4 nnz + 4 m, B: 8 n na + 4 n)
  over its mean CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline`` (rank 0, N = 1): the oracle port (oracle/, the
  reference's algorithm restated in C + numpy, CSR A as the reference builds
  it) on a bounded sample of the same workload using all host cores.
* Multi-GPU (torchrun): weak scaling by independent slices -- rank r solves
  its own seeded slice, no data-path collective (the c5 pattern); the step
  time is the max over ranks.
* ``--impl reference``: the CPU reference arm (oracle port, all host cores)
  on the same workload/metric; rank 0 only under torchrun.
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# exact reference CSR nnz(A) per config (c1, c2 also re-derived
# by K6 / golden fixtures at run time).
REF_NNZ = {"c1": 3755161, "c2": 30038914, "c3": 240316558, "c4": 1922526218,
           "c5": 9612625979}

CPU_SAMPLE_ITERS = {"c1": 25, "c2": 12, "c3": 2, "c4": 1, "c5": 1}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c2", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    return ap.parse_args()


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def applies_per_iter(method):
    return (2, 2) if method.startswith("ab") else (2, 1)   # (A, B)


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < 8:
                    continue
                try:
                    sm.append(float(parts[0]))
                    mx = max(mx, float(parts[1]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[4:8]):
                    if v.lower() == "active":
                        reasons.add(nm)
        except Exception:
            pass
        finally:
            try:
                os.unlink(self.path)
            except Exception:
                pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        busy = [v for v in sm if v > 0.5 * mx] or sm
        return {"sm_mhz": float(np.median(busy)), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------
# CPU arm: the oracle port (reference algorithm, host cores)
# ----------------------------------------------------------------------------

def cpu_sample(spec, iters=None, threads=0):
    """Time the oracle port on a bounded sample of the workload.

    Returns dict(value rays/s, iters/s, cores, sample description)."""
    from oracle import oracle as O
    from paper_2602_17892_b200 import problems

    threads = threads or len(os.sched_getaffinity(0))
    if spec.N >= 1024:
        return cpu_sample_subset(spec, threads)
    g = O.Geometry(spec.N, spec.N, 1.0, spec.angles(), spec.det_count, 1.0)
    t0 = time.perf_counter()
    A = O.CsrForward(g, nthreads=threads)
    build_s = time.perf_counter() - t0
    if spec.method is None:           # c3 microbench: A + B applies
        x = problems.uniform_image(g.n, 0)
        u = problems.uniform_sinogram(g.m, 1)
        reps = iters or CPU_SAMPLE_ITERS[spec.name]
        t0 = time.perf_counter()
        for _ in range(reps):
            A(x)
            O.back(g, u, threads)
        dt = time.perf_counter() - t0
        return dict(value=2 * reps * g.m / dt, iters_per_s=None, cores=threads,
                    sample=f"{reps}x (A + B) applies at {spec.name}, CSR build {build_s:.1f}s excluded",
                    seconds=dt)
    xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
    b, _ = problems.add_noise(A(xt), spec.noise, spec.noise_seed)
    b = b.astype(np.float32).astype(np.float64)
    K = iters or CPU_SAMPLE_ITERS[spec.name]
    t0 = time.perf_counter()
    O.gmres(A, lambda u: O.back(g, u, threads), b, spec.method, spec.strategy, K)
    dt = time.perf_counter() - t0
    na, nb = applies_per_iter(spec.method)
    return dict(value=K * (na + nb) * g.m / dt, iters_per_s=K / dt, cores=threads,
                sample=(f"first {K} of {spec.max_iter} {spec.method}/{spec.strategy} iterations at "
                        f"{spec.name} (oracle port: CSR A + C back + numpy MGS/lambda), "
                        f"CSR build {build_s:.1f}s excluded"), seconds=dt)


def cpu_sample_subset(spec, threads, stride=None):
    """c4/c5: the full CSR would need ~23 GB (c4) / ~115 GB (c5 per slice), so
    time the reference algorithm (CSR A + pixel-driven B) on a strided angle
    subset and extrapolate linearly in angles (SURVEY.md §8d protocol)."""
    from oracle import oracle as O
    from paper_2602_17892_b200 import problems

    stride = stride or max(1, spec.n_angles // 24)
    sub = spec.angles()[::stride]
    g = O.Geometry(spec.N, spec.N, 1.0, sub, spec.det_count, 1.0)
    A = O.CsrForward(g, nthreads=threads)
    x = problems.uniform_image(g.n, 0)
    u = problems.uniform_sinogram(g.m, 1)
    t0 = time.perf_counter()
    A(x)
    ta = time.perf_counter() - t0
    t0 = time.perf_counter()
    O.back(g, u, threads)
    tb = time.perf_counter() - t0
    scale = spec.n_angles / len(sub)
    ta, tb = ta * scale, tb * scale                 # extrapolated full-geometry applies
    na, nb = applies_per_iter(spec.method) if spec.method else (1, 1)
    per_iter = na * ta + nb * tb
    return dict(value=(na + nb) * spec.m / per_iter, iters_per_s=1.0 / per_iter, cores=threads,
                sample=(f"extrapolated: A (CSR) and B applies on {len(sub)} of {spec.n_angles} "
                        f"angles at {spec.name}, scaled x{scale:.1f}; {na}A+{nb}B per iteration, "
                        f"orthogonalisation/lambda excluded"), seconds=ta + tb)


def run_reference(args, spec, rank, world):
    if rank != 0:
        return
    steps, warm = args.steps, args.warmup
    # each step is a bounded sample of the workload; keep the whole run short
    iters = max(1, CPU_SAMPLE_ITERS[spec.name] // 2)
    if spec.N >= 1024:
        steps, warm = min(steps, 2), 0
    vals, secs = [], []
    for i in range(warm + steps):
        r = cpu_sample(spec, iters=iters)
        if i >= warm:
            vals.append(r["value"])
            secs.append(r["seconds"])
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": metric_name(spec), "value": value, "unit": "rays/s",
        "n_gpus": world, "steps": steps, "warmup": warm,
        "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(spec, world),
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": r["cores"], "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def metric_name(spec):
    if spec.method is None:
        return f"A+B projected rays/s ({spec.name} projector microbenchmark)"
    return f"A+B projected rays/s (hybrid {spec.method.split('-')[0].upper()}-GMRES solve, {spec.name})"


def workload_config(spec, world):
    cfg = {"workload": f"{spec.name}: {spec.N}x{spec.N} px, {spec.n_angles} angles, "
                       f"{spec.det_count} bins"
                       + (f", {spec.method} {spec.strategy}, {spec.max_iter} it, "
                          f"{int(spec.noise * 100)}% noise" if spec.method else ", 100 A + 100 B"),
           "n": spec.n, "m": spec.m, "slices_per_gpu": 1,
           "parallelism": f"weak x{world} (independent slices)" if world > 1 else "single GPU",
           "l2": "flushed (256 MiB write) before every timed step"}
    return cfg


# ----------------------------------------------------------------------------
# GPU arm
# ----------------------------------------------------------------------------

def main():
    args = parse()
    from paper_2602_17892_b200 import problems
    spec = problems.CONFIGS[args.workload]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, spec, rank, world)
        return

    import torch
    from paper_2602_17892_b200 import _native, ct, gmres

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (libctk has no CPU path)")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)

    grid = ct.ImageGrid(spec.N, spec.N, 1.0)
    geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    A = ct.forward_ray_driven(grid, geom, device=local)
    B = ct.back_pixel_driven(grid, geom, device=local)
    dg = A.dgeom
    raw, nnz = dg.count_segments()
    bytes_A = 4 * nnz + 4 * dg.m
    bytes_B = 8 * dg.n * dg.n_angles + 4 * dg.n
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def l2_flush():
        with torch.cuda.stream(stream):
            flush.fill_(1.0)

    hbm_peak, peak_src = measured_peak()
    result = {}

    if spec.method is None:
        # c3 projector microbenchmark: a step = 1 A + 1 B apply
        x = torch.from_numpy(problems.uniform_image(dg.n, 0).astype(np.float32)).to(dev)
        u = torch.from_numpy(problems.uniform_sinogram(dg.m, 1).astype(np.float32)).to(dev)
        y = torch.empty(dg.m, dtype=torch.float32, device=dev)
        xo = torch.empty(dg.n, dtype=torch.float32, device=dev)

        def step():
            dg.forward(x, out=y, stream=stream)
            dg.back(u, out=xo, stream=stream)
        rays_per_step = executed_per_step = 2 * dg.m
        iters_per_step = None
    else:
        pseed, nseed = problems.slice_seeds(spec, rank) if spec.slices > 1 else (
            spec.phantom_seed + rank, spec.noise_seed + 1000 * rank)
        xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, pseed)
        with torch.cuda.stream(stream):
            xd = torch.from_numpy(xt.astype(np.float32)).to(dev)
            clean = dg.forward(xd, stream=stream)
        stream.synchronize()
        b_host, _ = problems.add_noise(clean.cpu().numpy().astype(np.float64), spec.noise, nseed)
        b_host = b_host.astype(np.float32).astype(np.float64)
        b_dev = torch.from_numpy(b_host.astype(np.float32)).to(dev)
        cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy,
                                 max_iter=spec.max_iter)
        na, nb = applies_per_iter(spec.method)
        rays_per_step = spec.max_iter * (na + nb) * dg.m
        # applies this path actually runs: 1A + 1B per Arnoldi step, plus the
        # cycle start (AB: A x0; BA: A x0 and B of the residual)
        executed_per_step = (2 * spec.max_iter + (1 if spec.method.startswith("ab") else 2)) * dg.m
        iters_per_step = spec.max_iter

        def step():
            result["last"] = gmres.run_gmres(A, B, b_dev, cfg, stream=stream,
                                             keep_on_device=True)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        l2_flush()
        step()
    barrier()

    def timed_steps():
        tot = 0.0
        for _ in range(args.steps):
            l2_flush()
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            step()
            e1.record(stream)
            e1.synchronize()
            tot += e0.elapsed_time(e1)
        barrier()
        return tot

    launches0 = _native.launch_counter()
    with ClockSampler(local) as clocks:
        total_ms = timed_steps()
    launches = _native.launch_counter() - launches0
    # Per-kernel durations for the roofline: the same K steps again with CUDA
    # events around every libctk projector / orthogonalisation call on its
    # own stream (kept out of the timed steps above, whose events would
    # otherwise add their own overhead to `value`).
    _native.profile_begin()
    prof_total_ms = timed_steps()
    prof = _native.profile_end()
    t_local = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
    total_ms = float(t_local.item())
    ms_per_step = total_ms / args.steps
    value = world * rays_per_step * args.steps / (total_ms / 1e3)

    ksum = {k: (n, ms) for k, (n, ms, _) in prof.items()}
    shares = {k: tot for k, (_, _, tot) in prof.items() if k in ("forward", "back")}
    dom = max(shares, key=shares.get)
    n_l, ms_l = ksum[dom]
    alg = bytes_A if dom == "forward" else bytes_B
    achieved = alg / (ms_l / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "k_forward (+k_stage where not fused) (A)"
                if dom == "forward" else "k_back (B)",
                "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic_from_profiles(spec, dom),
                "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
                "launches_timed": n_l, "mean_launch_ms": round(ms_l, 5),
                "share_of_step": round(shares[dom] / max(prof_total_ms, 1e-9), 4),
                "measured": f"CUDA events around each launch over {args.steps} profiled steps "
                            "run after the timed ones (same workload, L2 flushed per step)"}
    kernels = {}
    for k, (n, ms) in ksum.items():
        kernels[k] = {"launches": n, "mean_ms": round(ms, 5)}
        if k in ("forward", "back"):
            kernels[k]["gbs"] = round((bytes_A if k == "forward" else bytes_B) / (ms / 1e3) / 1e9, 1)
            kernels[k]["rays_per_s"] = dg.m / (ms / 1e3)

    e2e = None
    if not args.no_e2e and spec.method is not None:
        # public API, host buffers: b numpy in, x numpy out, copies inside the timed region
        for _ in range(args.warmup):          # first-use costs (pinned staging buffers)
            gmres.run_gmres(A, B, b_host, cfg, stream=stream)
        walls = []
        for _ in range(args.steps):
            l2_flush()
            barrier()
            t0 = time.perf_counter()
            res = gmres.run_gmres(A, B, b_host, cfg, stream=stream)
            walls.append(time.perf_counter() - t0)
        barrier()
        wt = torch.tensor([float(np.sum(walls))], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * rays_per_step * args.steps / wt.item(), "unit": "rays/s",
               "h2d_bytes_per_step": int(res.transfer["h2d_bytes"]),
               "d2h_bytes_per_step": int(res.transfer["d2h_bytes"]),
               "timing": "wall clock around run_gmres(A, B, b_numpy, cfg) incl. H2D/D2H"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            c = cpu_sample(spec)
            cpu = {"value": c["value"], "unit": "rays/s", "cores": c["cores"], "kind": "port",
                   "sample": c["sample"]}
            if c.get("iters_per_s") is not None:
                cpu["iters_per_s"] = c["iters_per_s"]
        except Exception as exc:  # the baseline is reported, never the product
            cpu = {"value": None, "unit": "rays/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": metric_name(spec), "value": value, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random-ellipse phantom / uniform inputs, SURVEY.md §8d)",
            "config": workload_config(spec, world),
            "iters_per_s": (world * iters_per_step * args.steps / (total_ms / 1e3)
                            if iters_per_step else None),
            "roofline": roofline, "kernels": kernels, "nnz_A": nnz,
            "rays_counted": ("2*m per step (1 A + 1 B apply)" if spec.method is None else
                             f"{spec.max_iter} iterations x "
                             f"{'2A+2B' if spec.method.startswith('ab') else '2A+1B'} applies x m "
                             "per solve: the reference algorithm's projector work "
                             "(gmres.py:189,207,209); this path executes the Arnoldi "
                             "1A+1B per iteration and gets x_k and b - A x_k by linearity "
                             "from rows kept during the Arnoldi step"),
            "rays_executed_per_s": (value * executed_per_step / rays_per_step
                                    if rays_per_step else None),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
            "clocks": clocks.summary(),
        }
        if spec.slices > 1:      # batched slices (c5): one slice solve per rank per step
            line["slices_per_s"] = world * args.steps / (total_ms / 1e3)
        if "last" in result:
            last = result["last"]
            line["solve"] = {"stop_reason": last.stop_reason, "iterations": len(last.records),
                             "final_data_residual": last.records[-1].data_residual_norm}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def traffic_from_profiles(spec, dom):
    """dram bytes per launch of the dominant kernel from a committed ncu capture."""
    path = os.path.join(ROOT, "profiles", f"ncu_{spec.name}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(dom, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


if __name__ == "__main__":
    main()
