"""Phase breakdown of the Gram-corrected SMEM Gram-Schmidt step (k_gs_smem).

Needs libctk.so built with CTK_NVCC_EXTRA=-DCTK_GS_PROF.  Runs the chain of
steps 0..k on one basis (so step k takes the Gram path), times step k with
CUDA events, and prints per-phase durations (median / max over CTAs) from
the globaltimer stamps of that launch.

    CTK_NVCC_EXTRA=-DCTK_GS_PROF python -m paper_2602_17892_b200.build --force
    GS_KS=20,40,79 python tools/gs_gram_phase_prof.py 65536
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
rd = lib.ctk_gs_prof_read
rd.argtypes = [ctypes.c_void_p]
PH = [(0, 1, "pdl_wait"), (1, 2, "load"), (2, 3, "dots2"), (3, 4, "grid_sync"),
      (4, 6, "reduce"), (6, 5, "gram_coefs"), (5, 10, "update"), (10, 11, "tail")]
Ls = [int(a) for a in sys.argv[1:]] or [65536]
KS = [int(a) for a in os.environ.get('GS_KS', '20,40,79').split(',')]
REPS = int(os.environ.get('GS_REPS', '20'))
buf = np.zeros(160 * 16, dtype=np.uint64)
for L in Ls:
    for k in KS:
        B = DeviceBasis(L, k + 3, torch.device('cuda', 0), torch)
        v = torch.randn(L, device='cuda')
        h = torch.zeros(k + 8, dtype=torch.float64, device='cuda')
        st = torch.zeros(4, dtype=torch.float64, device='cuda')
        s = torch.cuda.current_stream()
        times = []
        for rep in range(REPS):
            B.W[0, :L] = v / v.norm()
            for j in range(k):
                B.cgs2_step(j, torch.randn(L, device='cuda'), h, st, s)
            q = torch.randn(L, device='cuda')
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            B.cgs2_step(k, q, h, st, s)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3)
        rd(buf.ctypes.data)
        T = buf.reshape(160, 16).astype(np.int64)
        G = int((T[:, 1] > 0).sum())
        T = T[:G]
        print(f"L={L} k={k} G={G}: {np.median(times):.1f} us/step (events, launch included)")
        print("   " + " ".join(f"{n:>12s}" for _, _, n in PH))
        d = np.stack([(T[:, b] - T[:, a]) / 1e3 for a, b, _ in PH], axis=1)
        print("med" + " ".join(f"{x:12.2f}" for x in np.median(d, axis=0)))
        print("max" + " ".join(f"{x:12.2f}" for x in d.max(axis=0)))
