"""Microbenchmark of one CGS2 step (ctk_cgs2_step) at given L and k."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2602_17892_b200.arnoldi import DeviceBasis
Ls = [int(a) for a in sys.argv[1:]] or [32940, 65536, 130680, 1048576]
for L in Ls:
    for k in (1, 10, 40, 80):
        B = DeviceBasis(L, k + 3, torch.device('cuda', 0), torch)
        B.W[:k + 1] = torch.randn(k + 1, B.ld, device='cuda')
        q0 = torch.randn(L, device='cuda')
        q = q0.clone()
        h = torch.zeros(k + 8, dtype=torch.float64, device='cuda'); st = torch.zeros(4, dtype=torch.float64, device='cuda')
        s = torch.cuda.current_stream()
        for _ in range(5): B.cgs2_step(k, q, h, st, s)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): B.cgs2_step(k, q, h, st, s)
        e1.record(); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 50 * 1e3
        gb = 4 * L * (4 * (k + 1) + 4) / us / 1e3
        print(f"L={L:8d} k={k:3d}  {us:7.1f} us  {gb:7.1f} GB/s")
