"""Benchmark: hybrid AB-/BA-GMRES projector path on B200 (one JSON line).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5]
                    [--slices-per-gpu S] [--impl ours|reference]

Metric (BASELINE.json): A+B projected rays/s through hybrid GMRES, plus
hybrid iterations/s, slices/s and the HBM-roofline fraction of the dominant
kernel.

* Default workload: c5, the largest configuration -- batched hybrid
  BA-GMRES + GCV, 60 iterations, 2048^2 px, 1800 angles x 2897 bins, seeded
  random-ellipse phantom per slice, 1% noise -- at 8 slices per GPU (the
  config's 64 slices over 8 B200; slice s has seeds (s, 1000 + s)).  A "step"
  is the full hybrid solve of every slice of this GPU, issued from S host
  threads at once (each with its own stream pair; slices never communicate).
  Projected rays per step = S * K * (A+B applies per iteration) * m
  (BA: 2A+1B, AB: 2A+2B; cycle-start applies excluded).
  ``--workload c1..c4`` run one solve (or the c3 A+B microbenchmark) per step.
* ``value``: device-resident solves (b already in HBM, x left in HBM), timed
  with CUDA events (e0 before every slice stream starts, e1 after all have
  joined), L2 flushed (256 MiB write) before every timed step; the inputs
  (4.2M-px images, 5.2M-sample sinograms, a 2.3 GB Krylov basis per slice)
  are far larger than L2 anyway.  ``e2e``: the same solves through the
  public API ``run_gmres(A, B, b_numpy, cfg)`` with host b in and host x out,
  wall-clock with the copies inside the timed region.
* ``roofline``: the projector kernel with the largest share of the timed
  region, algorithmic bytes per launch (A: 4 nnz + 4 m, B: 8 n na + 4 n)
  over its mean CUDA-event duration, against MEASURED_PEAKS.json hbm_gbs.
* ``cpu_baseline`` (rank 0, N = 1): the oracle port (oracle/, the
  reference's algorithm restated in C + numpy, CSR A as the reference builds
  it) on a bounded sample of the same workload using all host cores.
* Multi-GPU (torchrun): weak scaling by independent slices -- rank r solves
  its own seeded slices r*S .. r*S+S-1, no data-path collective (the c5
  pattern); the step time is the max over ranks.
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
    ap.add_argument("--workload", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--slices-per-gpu", type=int, default=0,
                    help="concurrent independent slices per GPU (default: 8 for c5, else 1)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--shard", default="none", choices=["none", "angles"],
                    help="angles: one problem split by projection angle over the ranks "
                         "(strong scaling; c3 A+B microbenchmark or a c1/c2/c4 solve)")
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

class CpuSample:
    """One bounded, repeatable sample of the workload on the host cores (the
    oracle port: the reference's algorithm restated -- CSR A as the reference
    assembles it, pixel-driven B, numpy MGS/lambda).  Set-up (CSR assembly)
    happens once in the constructor; run() is one timed sample and returns
    rays/s in the workload's metric (reference applies per iteration).

    * c1/c2: the first `iters` iterations of the hybrid solve;
    * c3: `reps` x (A + B) applies;
    * c4/c5: A (CSR) and B applies on a strided angle subset, extrapolated
      linearly in angles to the full geometry (the full CSR needs ~23 GB at
      c4, ~115 GB per slice at c5); orthogonalisation / lambda excluded."""

    def __init__(self, spec, threads=0, iters=None):
        from oracle import oracle as O
        from paper_2602_17892_b200 import problems
        self.O, self.spec = O, spec
        self.threads = threads or len(os.sched_getaffinity(0))
        t0 = time.perf_counter()
        if spec.N >= 1024:
            stride = max(1, spec.n_angles // 18)
            self.sub = spec.angles()[::stride]
            g = O.Geometry(spec.N, spec.N, 1.0, self.sub, spec.det_count, 1.0)
            self.x = problems.uniform_image(g.n, 0)
            self.u = problems.uniform_sinogram(g.m, 1)
        else:
            g = O.Geometry(spec.N, spec.N, 1.0, spec.angles(), spec.det_count, 1.0)
        self.g = g
        self.A = O.CsrForward(g, nthreads=self.threads)
        self.build_s = time.perf_counter() - t0
        if spec.method is None:
            self.x = problems.uniform_image(g.n, 0)
            self.u = problems.uniform_sinogram(g.m, 1)
            self.reps = iters or CPU_SAMPLE_ITERS[spec.name]
        elif spec.N < 1024:
            xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
            b, _ = problems.add_noise(self.A(xt), spec.noise, spec.noise_seed)
            self.b = b.astype(np.float32).astype(np.float64)
            self.iters = iters or CPU_SAMPLE_ITERS[spec.name]

    def run(self):
        """One timed sample; adds the effective core count (process CPU time
        / wall time over the sample)."""
        c0, w0 = time.process_time(), time.perf_counter()
        r = self._run()
        r["cpu_time_over_wall"] = round((time.process_time() - c0) / (time.perf_counter() - w0), 2)
        return r

    def _run(self):
        O, spec, g, th = self.O, self.spec, self.g, self.threads
        if spec.N >= 1024:
            t0 = time.perf_counter()
            self.A(self.x)
            ta = time.perf_counter() - t0
            t0 = time.perf_counter()
            O.back(g, self.u, th)
            tb = time.perf_counter() - t0
            scale = spec.n_angles / len(self.sub)
            ta, tb = ta * scale, tb * scale
            na, nb = applies_per_iter(spec.method) if spec.method else (1, 1)
            per_iter = na * ta + nb * tb
            return dict(value=(na + nb) * spec.m / per_iter, iters_per_s=1.0 / per_iter,
                        cores=th, seconds=(ta + tb) / scale,
                        sample=(f"extrapolated: A (CSR) and B applies on {len(self.sub)} of "
                                f"{spec.n_angles} angles at {spec.name}, scaled x{scale:.1f}; "
                                f"{na}A+{nb}B per iteration, orthogonalisation/lambda excluded; "
                                f"CSR build {self.build_s:.1f}s excluded"))
        if spec.method is None:
            t0 = time.perf_counter()
            for _ in range(self.reps):
                self.A(self.x)
                O.back(g, self.u, th)
            dt = time.perf_counter() - t0
            return dict(value=2 * self.reps * g.m / dt, iters_per_s=None, cores=th, seconds=dt,
                        sample=f"{self.reps}x (A + B) applies at {spec.name}, "
                               f"CSR build {self.build_s:.1f}s excluded")
        K = self.iters
        t0 = time.perf_counter()
        O.gmres(self.A, lambda u: O.back(g, u, th), self.b, spec.method, spec.strategy, K)
        dt = time.perf_counter() - t0
        na, nb = applies_per_iter(spec.method)
        return dict(value=K * (na + nb) * g.m / dt, iters_per_s=K / dt, cores=th, seconds=dt,
                    sample=(f"first {K} of {spec.max_iter} {spec.method}/{spec.strategy} "
                            f"iterations at {spec.name} (oracle port: CSR A + C back + numpy "
                            f"MGS/lambda), CSR build {self.build_s:.1f}s excluded"))


def cpu_sample(spec, iters=None, threads=0):
    """One sample (bench's cpu_baseline leg)."""
    return CpuSample(spec, threads, iters).run()


def run_reference(args, spec, rank, world):
    """CPU reference arm: the oracle port on all host cores.  Exactly
    args.warmup untimed + args.steps timed samples (each a bounded sample of
    the workload, see CpuSample); rank 0 only."""
    if rank != 0:
        return
    spg = args.slices_per_gpu or (8 if spec.slices > 1 else 1)
    smp = CpuSample(spec, iters=max(1, CPU_SAMPLE_ITERS[spec.name] // 2))
    vals, secs = [], []
    for i in range(args.warmup + args.steps):
        r = smp.run()
        if i >= args.warmup:
            vals.append(r["value"])
            secs.append(r["seconds"])
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": metric_name(spec, spg), "value": value, "unit": "rays/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * float(np.mean(secs)), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(spec, world, spg),
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": r["cores"], "kind": "port",
                         "sample": r["sample"], "cpu_time_over_wall": r["cpu_time_over_wall"],
                         "cpu_env": cpu_env()},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_env():
    """Host-core context of a CPU number."""
    keys = ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS")
    return {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
            **{k: os.environ.get(k) for k in keys}}


def metric_name(spec, spg=1):
    if spec.method is None:
        return f"A+B projected rays/s ({spec.name} projector microbenchmark)"
    what = f"{spg} concurrent slice solves" if spg > 1 else "solve"
    return (f"A+B projected rays/s (hybrid {spec.method.split('-')[0].upper()}-GMRES {what}, "
            f"{spec.name})")


def workload_config(spec, world, spg=1):
    cfg = {"workload": f"{spec.name}: {spec.N}x{spec.N} px, {spec.n_angles} angles, "
                       f"{spec.det_count} bins"
                       + (f", {spec.method} {spec.strategy}, {spec.max_iter} it, "
                          f"{int(spec.noise * 100)}% noise" if spec.method else ", 100 A + 100 B")
                       + (f", {spg} independent slices per GPU" if spg > 1 else ""),
           "n": spec.n, "m": spec.m, "slices_per_gpu": spg,
           "parallelism": (f"weak x{world} (independent slices)" if world > 1 else "single GPU")
                          + (f", {spg} concurrent slice solves per GPU" if spg > 1 else ""),
           "l2": "flushed (256 MiB write) before every timed step; per-slice inputs and "
                 "Krylov basis exceed L2"}
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
    if args.shard == "angles":
        return main_sharded(args, spec, world, rank, local, torch, dist, stream)

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

    spg = args.slices_per_gpu or (8 if spec.slices > 1 else 1)
    if spec.method is None:
        # c3 projector microbenchmark: a step = 1 A + 1 B apply
        spg = 1
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
        b_hosts, b_devs = [], []
        for i in range(spg):
            sidx = rank * spg + i                   # global slice index
            pseed, nseed = problems.slice_seeds(spec, sidx) if spec.slices > 1 else (
                spec.phantom_seed + sidx, spec.noise_seed + 1000 * sidx)
            _, x32 = problems.random_ellipse_phantom_device(spec.N, spec.ellipses, pseed,
                                                            device=local, stream=stream)
            with torch.cuda.stream(stream):
                clean = dg.forward(x32, stream=stream)
            stream.synchronize()
            b_host, _ = problems.add_noise(clean.cpu().numpy().astype(np.float64), spec.noise,
                                           nseed)
            b_host = b_host.astype(np.float32).astype(np.float64)
            b_hosts.append(b_host)
            b_devs.append(torch.from_numpy(b_host.astype(np.float32)).to(dev))
        cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy,
                                 max_iter=spec.max_iter)
        na, nb = applies_per_iter(spec.method)
        rays_per_step = spg * spec.max_iter * (na + nb) * dg.m
        # applies this path actually runs: 1A + 1B per Arnoldi step, plus the
        # cycle start (AB: A x0; BA: A x0 and B of the residual)
        executed_per_step = spg * (2 * spec.max_iter
                                   + (1 if spec.method.startswith("ab") else 2)) * dg.m
        iters_per_step = spg * spec.max_iter
        # one caller stream per slice; a persistent pool of spg host threads
        # (the solver's per-thread stream pairs and workspaces are reused)
        callers = [torch.cuda.Stream(dev) for _ in range(spg)]
        from concurrent.futures import ThreadPoolExecutor
        tpool = ThreadPoolExecutor(max_workers=spg) if spg > 1 else None

        def solve_all(bs, on_device):
            for c in callers:
                c.wait_stream(stream)

            def one(i):
                return gmres.run_gmres(A, B, bs[i], cfg, stream=callers[i],
                                       keep_on_device=on_device)
            outs = list(tpool.map(one, range(spg))) if tpool else [one(0)]
            for c in callers:
                stream.wait_stream(c)
            return outs

        def step():
            result["last"] = solve_all(b_devs, True)[-1]

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        l2_flush()
        step()
    barrier()

    def timed_steps(n_steps):
        tot = 0.0
        for _ in range(n_steps):
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
        total_ms = timed_steps(args.steps)
    launches = _native.launch_counter() - launches0
    # Per-kernel durations for the roofline: CUDA events around every libctk
    # projector / orthogonalisation call on its own stream, in a separate
    # pass after the timed one (so the events add nothing to `value`), with
    # one slice at a time (concurrent slices share the SMs, which would
    # stretch each launch's own duration).
    spg_timed = spg
    if spec.method is not None and spg > 1:
        prof_bs = b_devs[:1]

        def prof_step():
            gmres.run_gmres(A, B, prof_bs[0], cfg, stream=stream, keep_on_device=True)
    else:
        prof_step = step
    _native.profile_begin()
    prof_total_ms = 0.0
    for _ in range(max(1, min(args.steps, 3))):
        l2_flush()
        torch.cuda.synchronize(dev)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        prof_step()
        e1.record(stream)
        e1.synchronize()
        prof_total_ms += e0.elapsed_time(e1)
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
                "binding": traffic_from_profiles(spec, dom, "binding") or
                "gathers served on chip (frac > 1 on algorithmic gather bytes); see profiles/",
                "measured": "CUDA events around each launch on its stream over "
                            f"{max(1, min(args.steps, 3))} profiled single-slice solves run "
                            "after the timed steps (same workload, L2 flushed per solve)"}
    kernels = {}
    for k, (n, ms) in ksum.items():
        kernels[k] = {"launches": n, "mean_ms": round(ms, 5)}
        if k in ("forward", "back"):
            kernels[k]["gbs"] = round((bytes_A if k == "forward" else bytes_B) / (ms / 1e3) / 1e9, 1)
            kernels[k]["rays_per_s"] = dg.m / (ms / 1e3)

    e2e = None
    if not args.no_e2e and spec.method is not None:
        # public API, host buffers: b numpy in, x numpy out, copies inside the timed region
        for _ in range(min(args.warmup, 2)):   # first-use costs (pinned staging buffers)
            solve_all(b_hosts, False)
        walls = []
        res = None
        for _ in range(args.steps):
            l2_flush()
            barrier()
            t0 = time.perf_counter()
            outs = solve_all(b_hosts, False)
            walls.append(time.perf_counter() - t0)
            res = outs
        barrier()
        wt = torch.tensor([float(np.sum(walls))], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        e2e = {"value": world * rays_per_step * args.steps / wt.item(), "unit": "rays/s",
               "h2d_bytes_per_step": int(sum(r.transfer["h2d_bytes"] for r in res)),
               "d2h_bytes_per_step": int(sum(r.transfer["d2h_bytes"] for r in res)),
               "timing": (f"wall clock around {spg} concurrent run_gmres(A, B, b_numpy, cfg) "
                          "calls incl. H2D/D2H")}
        if spec.slices > 1:
            e2e["slices_per_s"] = world * spg * args.steps / wt.item()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            c = cpu_sample(spec)
            cpu = {"value": c["value"], "unit": "rays/s", "cores": c["cores"], "kind": "port",
                   "sample": c["sample"], "cpu_time_over_wall": c["cpu_time_over_wall"],
                   "cpu_env": cpu_env()}
            if c.get("iters_per_s") is not None:
                cpu["iters_per_s"] = c["iters_per_s"]
        except Exception as exc:  # the baseline is reported, never the product
            cpu = {"value": None, "unit": "rays/s", "cores": 0, "kind": "port",
                   "sample": f"failed: {exc}"}

    if rank == 0:
        line = {
            "metric": metric_name(spec, spg), "value": value, "unit": "rays/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded random-ellipse phantom / uniform inputs, SURVEY.md §8d)",
            "config": workload_config(spec, world, spg),
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
        if spec.slices > 1:      # batched slices (c5): spg slice solves per rank per step
            line["slices_per_s"] = world * spg * args.steps / (total_ms / 1e3)
        if "last" in result:
            last = result["last"]
            line["solve"] = {"stop_reason": last.stop_reason, "iterations": len(last.records),
                             "final_data_residual": last.records[-1].data_residual_norm}
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def main_sharded(args, spec, world, rank, local, torch, dist, stream):
    """--shard angles: ONE problem split by projection angle over the ranks
    (SURVEY row e; strong scaling, total work fixed).  A is sharded by angle
    with a replicated image; B's partial images are summed over ranks (peer
    exchange fused into K2 when the ranks map each other's memory, else NCCL);
    AB Krylov vectors are sharded in measurement space with fp64 all-reduces
    of the Gram-Schmidt dots; all collectives are issued by libctk's C++
    driver (dist.NativeComm + run_gmres(..., comm=)).  c3: a step = A + the
    summed B of the full geometry; c1/c2/c4: a step = one full hybrid solve."""
    from paper_2602_17892_b200 import _native, ct, dist as cdist, gmres, problems

    dev = torch.device("cuda", local)
    grid = ct.ImageGrid(spec.N, spec.N, 1.0)
    geom = ct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    idx = cdist.angle_shards(spec.n_angles, world)[rank]
    A, B = cdist.sharded_projectors(grid, geom, idx, device=local)
    dg = A.dgeom
    comm = cdist.NativeComm(dg)
    D = spec.det_count
    m_full = spec.m
    raw, nnz_local = dg.count_segments()
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    result = {}
    if spec.method is None:
        x = torch.from_numpy(problems.uniform_image(dg.n, 0).astype(np.float32)).to(dev)
        u_full = problems.uniform_sinogram(m_full, 1)
        u = torch.from_numpy(cdist.local_rows(u_full, D, idx).astype(np.float32)).to(dev)
        y = torch.empty(dg.m, dtype=torch.float32, device=dev)
        img = torch.empty(dg.n, dtype=torch.float32, device=dev)

        def step():
            dg.forward(x, out=y, stream=stream)
            comm.back(u, out=img, stream=stream)
        rays_per_step = 2 * m_full
        iters_per_step = None
    else:
        # b of the FULL geometry (bitwise the single-GPU bench's), this rank's rows
        Af = ct.forward_ray_driven(grid, geom, device=local)
        xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
        with torch.cuda.stream(stream):
            clean = Af.dgeom.forward(torch.from_numpy(xt.astype(np.float32)).to(dev), stream=stream)
        stream.synchronize()
        b_full, _ = problems.add_noise(clean.cpu().numpy().astype(np.float64), spec.noise,
                                       spec.noise_seed)
        b_full = b_full.astype(np.float32).astype(np.float64)
        del Af, clean
        b_host = cdist.local_rows(b_full, D, idx)
        b_dev = torch.from_numpy(b_host.astype(np.float32)).to(dev)
        cfg = gmres.SolverConfig(method=spec.method, lambda_strategy=spec.strategy,
                                 max_iter=spec.max_iter)
        na_, nb_ = applies_per_iter(spec.method)
        rays_per_step = spec.max_iter * (na_ + nb_) * m_full
        iters_per_step = spec.max_iter

        def step():
            result["last"] = gmres.run_gmres(A, B, b_dev, cfg, stream=stream,
                                             keep_on_device=True, comm=comm)

    def barrier():
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()

    def timed(n_steps):
        tot = 0.0
        for _ in range(n_steps):
            with torch.cuda.stream(stream):
                flush.fill_(1.0)
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
        total_ms = timed(args.steps)
    launches = _native.launch_counter() - launches0
    _native.profile_begin()
    timed(max(1, min(args.steps, 2)))
    prof = _native.profile_end()
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = rays_per_step * args.steps / (total_ms / 1e3)
    hbm_peak, peak_src = measured_peak()
    kernels = {k: {"launches": n, "mean_ms": round(ms, 5)} for k, (n, ms, _) in prof.items()}
    bytes_A = 4 * nnz_local + 4 * dg.m
    roofline = None
    if "forward" in prof:
        n_l, ms_l, _ = prof["forward"]
        ach = bytes_A / (ms_l / 1e3) / 1e9
        roofline = {"bound": "hbm", "kernel": "k_forward (this rank's angles)",
                    "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                    "frac": round(ach / hbm_peak, 4), "traffic": None, "peak_source": peak_src,
                    "algorithmic_bytes_per_launch": bytes_A, "launches_timed": n_l,
                    "mean_launch_ms": round(ms_l, 5)}
    e2e = None
    if spec.method is not None and not args.no_e2e:
        gmres.run_gmres(A, B, b_host, cfg, stream=stream, comm=comm)     # pinned buffers
        walls = []
        res = None
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            res = gmres.run_gmres(A, B, b_host, cfg, stream=stream, comm=comm)
            walls.append(time.perf_counter() - t0)
        barrier()
        wt = torch.tensor([float(np.sum(walls))], dtype=torch.float64, device=dev)
        if dist is not None:
            dist.all_reduce(wt, op=dist.ReduceOp.MAX)
        e2e = {"value": rays_per_step * args.steps / wt.item(), "unit": "rays/s",
               "h2d_bytes_per_step": int(res.transfer["h2d_bytes"]),
               "d2h_bytes_per_step": int(res.transfer["d2h_bytes"]),
               "timing": "wall clock around run_gmres(A_rank, B_rank, b_rank_numpy, cfg, "
                         "comm=) incl. H2D/D2H, max over ranks"}
    if rank == 0:
        cfgd = workload_config(spec, world)
        cfgd["parallelism"] = (f"angle-sharded x{world} ("
                               + ("peer-memory exchange" if comm.xchg is not None else "NCCL")
                               + " for B's partial images)")
        line = {
            "metric": metric_name(spec) + ", angle-sharded", "value": value, "unit": "rays/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, SURVEY.md §8d)",
            "config": cfgd, "shard": {"angles_per_rank": int(len(idx)), "mode": "interleaved"},
            "iters_per_s": (iters_per_step * args.steps / (total_ms / 1e3)
                            if iters_per_step else None),
            "roofline": roofline, "kernels": kernels, "e2e": e2e, "cpu_baseline": None,
            "gpu_launches": int(launches), "clocks": clocks.summary(),
        }
        if "last" in result:
            last = result["last"]
            line["solve"] = {"stop_reason": last.stop_reason, "iterations": len(last.records),
                             "final_data_residual": last.records[-1].data_residual_norm}
        print(json.dumps(line), flush=True)
    comm.close()
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


def traffic_from_profiles(spec, dom, field="dram_bytes_per_launch"):
    """A field of the dominant kernel's committed ncu capture (profiles/)."""
    path = os.path.join(ROOT, "profiles", f"ncu_{spec.name}.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(dom, {}).get(field)
    except Exception:
        return None


if __name__ == "__main__":
    main()
