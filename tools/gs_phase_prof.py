"""Phase breakdown of the SMEM-resident Gram-Schmidt step (k_gs_smem).

Needs libctk.so built with CTK_NVCC_EXTRA=-DCTK_GS_PROF (globaltimer stamps
per CTA at every phase boundary of the last launch).  Prints, per (L, k), the
median / max over CTAs of each phase's duration and the spread of arrival.

    CTK_NVCC_EXTRA=-DCTK_GS_PROF python -m paper_2602_17892_b200.build --force
    python tools/gs_phase_prof.py 32940 65536
"""
import ctypes
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_2602_17892_b200 import _native
from paper_2602_17892_b200.arnoldi import DeviceBasis

lib = _native.load()
rd = lib.ctk_gs_prof_read
rd.argtypes = [ctypes.c_void_p]
NAMES = ["pdl_wait", "load", "dots1", "sync1", "reduce1", "update1", "dots2", "sync2",
         "reduce2", "update2", "tail"]
Ls = [int(a) for a in sys.argv[1:]] or [32940, 65536]
import os
KS = [int(a) for a in os.environ.get('GS_KS', '1,20,40,80').split(',')]
REPS = int(os.environ.get('GS_REPS', '50'))
buf = np.zeros(160 * 16, dtype=np.uint64)
for L in Ls:
    for k in KS:
        B = DeviceBasis(L, k + 3, torch.device('cuda', 0), torch)
        # orthonormal rows (as in a solve: the ||q2|| shortcut applies)
        Qm, _ = torch.linalg.qr(torch.randn(L, k + 1, device='cuda', dtype=torch.float64))
        B.W[:k + 1, :L] = Qm.T.float()
        q = torch.randn(L, device='cuda')
        h = torch.zeros(k + 8, dtype=torch.float64, device='cuda')
        st = torch.zeros(4, dtype=torch.float64, device='cuda')
        s = torch.cuda.current_stream()
        for _ in range(20):
            B.cgs2_step(k, q, h, st, s)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(REPS):
            B.cgs2_step(k, q, h, st, s)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / REPS * 1e3
        B.cgs2_step(k, q, h, st, s)
        torch.cuda.synchronize()
        rd(buf.ctypes.data)
        T = buf.reshape(160, 16).astype(np.int64)
        G = int((T[:, 1] > 0).sum())
        T = T[:G]
        t0 = T[:, 0].min()
        rel = (T - t0) / 1e3
        d = np.diff(T[:, :12], axis=1) / 1e3       # us per phase
        print(f"L={L} k={k} G={G}: {us:.1f} us/step (events); entry spread "
              f"{rel[:, 0].max():.2f} us, end (CTA0) {rel[0, 11]:.2f} us")
        print("   " + " ".join(f"{n:>9s}" for n in NAMES))
        print("med" + " ".join(f"{v:9.2f}" for v in np.median(d[:, :11], axis=0)))
        print("max" + " ".join(f"{v:9.2f}" for v in d[:, :11].max(axis=0)))
