"""Time the UNMODIFIED reference (ctkrylov from baseline/_ref) on the host
cores (VERDICT r01 missing 8): c1 and c2 hybrid solves in
full (all iterations), c3 A and B applies, each beside the oracle port that
bench.py uses as its CPU arm, with the CPU context (cpu count, affinity,
BLAS/OMP env, process CPU time / wall time).  One JSON line per item.

    python tools/time_reference_cpu.py [c1] [c2] [c3]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402

import ctkrylov.ct as rct  # noqa: E402
import ctkrylov.gmres as rg  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2602_17892_b200 import problems  # noqa: E402

ENV = {"cpu_count": os.cpu_count(), "affinity": len(os.sched_getaffinity(0)),
       **{k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                          "MKL_NUM_THREADS")}}


def timed(fn):
    c0, w0 = time.process_time(), time.perf_counter()
    out = fn()
    wall = time.perf_counter() - w0
    return out, wall, (time.process_time() - c0) / wall


def emit(**kw):
    kw["cpu_env"] = ENV
    print(json.dumps(kw), flush=True)


def ref_ops(spec):
    g = rct.ImageGrid(spec.N, spec.N, 1.0)
    p = rct.ParallelGeometry(spec.angles(), spec.det_count, 1.0)
    (A, B), build, _ = timed(lambda: (rct.forward_ray_driven(g, p), rct.back_pixel_driven(g, p)))
    return A, B, build


def solve(name):
    spec = problems.CONFIGS[name]
    A, B, build = ref_ops(spec)
    xt = problems.random_ellipse_phantom(spec.N, spec.ellipses, spec.phantom_seed)
    b, _ = problems.add_noise(A.apply(xt), spec.noise, spec.noise_seed)
    b = b.astype(np.float32).astype(np.float64)
    cfg = rg.SolverConfig(method=spec.method, lambda_strategy=spec.strategy, max_iter=spec.max_iter)
    res, wall, util = timed(lambda: rg.run_gmres(A, B, b, cfg))
    na, nb = (2, 2) if spec.method.startswith("ab") else (2, 1)
    K = len(res.records)
    emit(impl="reference (unmodified ctkrylov)", workload=name, what=f"{spec.method}/{spec.strategy}",
         iterations=K, seconds=wall, iters_per_s=K / wall, rays_per_s=K * (na + nb) * spec.m / wall,
         build_s=build, cpu_time_over_wall=round(util, 2))
    # the oracle port on the same problem (bench.py's CPU arm), all host cores
    g = O.Geometry(spec.N, spec.N, 1.0, spec.angles(), spec.det_count, 1.0)
    Ao = O.CsrForward(g)
    res_o, wall_o, util_o = timed(lambda: O.gmres(Ao, lambda u: O.back(g, u), b, spec.method,
                                                  spec.strategy, spec.max_iter))
    emit(impl="oracle port (bench.py CPU arm)", workload=name, iterations=len(res_o.records),
         seconds=wall_o, iters_per_s=len(res_o.records) / wall_o,
         rays_per_s=len(res_o.records) * (na + nb) * spec.m / wall_o,
         cpu_time_over_wall=round(util_o, 2), cores=ENV["affinity"])


def applies(name, reps=3):
    spec = problems.CONFIGS[name]
    A, B, build = ref_ops(spec)
    x = problems.uniform_image(spec.n, 0)
    u = problems.uniform_sinogram(spec.m, 1)
    _, ta, ua = timed(lambda: [A.apply(x) for _ in range(reps)])
    _, tb, ub = timed(lambda: [B.apply(u) for _ in range(reps)])
    emit(impl="reference (unmodified ctkrylov)", workload=name, what="A and B applies",
         A_ms=1e3 * ta / reps, B_ms=1e3 * tb / reps,
         A_rays_per_s=spec.m * reps / ta, B_rays_per_s=spec.m * reps / tb, build_s=build,
         cpu_time_over_wall_A=round(ua, 2), cpu_time_over_wall_B=round(ub, 2))


if __name__ == "__main__":
    which = sys.argv[1:] or ["c1", "c2", "c3"]
    for w in which:
        (applies if w == "c3" else solve)(w)
