"""Phase breakdown of the streamed Gram-corrected Gram-Schmidt step (k_gs_stream).

Needs libctk.so built with CTK_NVCC_EXTRA=-DCTK_GS_PROF.  Builds a basis of
k + 1 orthonormal rows directly (QR-free: random rows orthogonalised by the
kernel itself over steps 0..k-1), times step k with CUDA events (L2 flushed)
and prints the per-phase durations (median / max over CTAs) from the
globaltimer stamps of that launch, with each sweep's achieved HBM GB/s.

    CTK_NVCC_EXTRA=-DCTK_GS_PROF python -m paper_2602_17892_b200.build --force
    GS_KS=10,30,50 python tools/gs_stream_phase_prof.py 2086560 4194304
"""
import ctypes
import os
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_2602_17892_b200 import _native
from paper_2602_17892_b200.arnoldi import DeviceBasis

lib = _native.load()
try:
    rd = lib.ctk_gs_prof_read
    rd.argtypes = [ctypes.c_void_p]
except AttributeError:          # plain build: event timings only
    rd = None
PH = [(0, 1, "pdl_wait"), (1, 2, "sweepA"), (2, 3, "grid_sync"), (3, 4, "reduce"),
      (4, 5, "gram_coefs"), (5, 6, "sweepC"), (6, 7, "tail")]
Ls = [int(a) for a in sys.argv[1:]] or [2086560]
KS = [int(a) for a in os.environ.get('GS_KS', '10,30,50').split(',')]
REPS = int(os.environ.get('GS_REPS', '5'))
buf = np.zeros(160 * 16, dtype=np.uint64)
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
for L in Ls:
    kmax = max(KS) + REPS
    B = DeviceBasis(L, kmax + 3, torch.device('cuda', 0), torch)
    h = torch.zeros(kmax + 8, dtype=torch.float64, device='cuda')
    st = torch.zeros(4, dtype=torch.float64, device='cuda')
    s = torch.cuda.current_stream()
    v = torch.randn(L, device='cuda')
    B.W[0, :L] = v / v.norm()
    done = 0
    for k0 in sorted(KS):
        for j in range(done, k0):
            B.cgs2_step(j, torch.randn(L, device='cuda'), h, st, s)
        times = []
        # the Gram path needs the chain of steps 0, 1, ... on one basis: time
        # REPS consecutive steps k0, k0 + 1, ... (the stamps are the last one's)
        for k in range(k0, k0 + REPS):
            q = torch.randn(L, device='cuda')
            flush.fill_(1.0)
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            B.cgs2_step(k, q, h, st, s)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3)
        done = k0 + REPS
        k = k0 + REPS - 1
        if rd is None:
            sweep_bytes = 4.0 * L * (k + 2)
            print(f"L={L} k={k}: {times[-1]:.1f} us/step (events), "
                  f"{2 * sweep_bytes / times[-1] / 1e3:.0f} GB/s on 2 sweeps")
            continue
        rd(buf.ctypes.data)
        T = buf.reshape(160, 16).astype(np.int64)
        G = int((T[:, 1] > 0).sum())
        T = T[:G]
        t = float(times[-1])
        sweep_bytes = 4.0 * L * (k + 2)
        print(f"L={L} k={k} G={G}: {t:.1f} us/step (events), 2 sweeps = "
              f"{2 * sweep_bytes / 1e9:.3f} GB -> {2 * sweep_bytes / t / 1e3:.0f} GB/s overall")
        print("   " + " ".join(f"{n:>11s}" for _, _, n in PH))
        d = np.stack([(T[:, b] - T[:, a]) / 1e3 for a, b, _ in PH], axis=1)
        print("med" + " ".join(f"{x:11.2f}" for x in np.median(d, axis=0)))
        print("max" + " ".join(f"{x:11.2f}" for x in d.max(axis=0)))
        span = (T[:, 7].max() - T[:, 0].min()) / 1e3
        a = np.median(d[:, 1]); c = np.median(d[:, 5])
        print(f"   kernel span {span:.1f} us; sweepA {sweep_bytes / a / 1e3:.0f} GB/s, "
              f"sweepC {sweep_bytes / c / 1e3:.0f} GB/s")
