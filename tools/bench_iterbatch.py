"""Isolated timing of ctk_iterate_batch (batched iterate norms, K4) at c4 / c5
sizes: CUDA events, L2 flushed before each call, GB/s on the bytes it reads
(the k_max rows of X and AX plus x0 / d0).

    python tools/bench_iterbatch.py [c4|c5 ...]
"""
import json
import sys

sys.path.insert(0, '.')
import numpy as np
import torch

from paper_2602_17892_b200 import _native, problems

lib = _native.load()
peak = json.load(open('MEASURED_PEAKS.json'))['hbm_gbs']
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
for name in sys.argv[1:] or ['c4', 'c5']:
    spec = problems.CONFIGS[name]
    ab = spec.method.startswith('ab')
    Lx, Lr = spec.n, spec.m
    for k0 in (10, 30, 50):
        nb = 8
        rows = k0 + nb + 2
        ldx, ldr = (Lx + 3) // 4 * 4, (Lr + 3) // 4 * 4
        X = torch.randn(rows, ldx, device='cuda')
        AX = torch.randn(rows, ldr, device='cuda')
        x0 = torch.randn(Lx, device='cuda')
        d0 = torch.randn(Lr, device='cuda')
        Y = torch.randn(nb, rows, dtype=torch.float64, device='cuda')
        x = torch.zeros(Lx, device='cuda')
        r = torch.zeros(Lr, device='cuda')
        norms = torch.zeros(2 * nb, dtype=torch.float64, device='cuda')
        cap = rows + 2
        scratch = torch.zeros(int(lib.ctk_reduce_scratch_bytes(cap, Lr)) // 8 + 1,
                              dtype=torch.float64, device='cuda')
        st = torch.cuda.current_stream()

        def call():
            _native.check(lib.ctk_iterate_batch(X.data_ptr(), ldx, x0.data_ptr(), x.data_ptr(), Lx,
                                                AX.data_ptr(), ldr, d0.data_ptr(), r.data_ptr(), Lr,
                                                k0, nb, Y.data_ptr(), rows, norms.data_ptr(),
                                                scratch.data_ptr(), cap, st.cuda_stream))
        for _ in range(3):
            call()
        ts = []
        for _ in range(10):
            flush.fill_(1.0)
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            call()
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts))
        kmax = k0 + nb - 1
        by = 4 * (kmax * (Lx + Lr) + Lx + Lr) + 4 * (Lx + Lr)     # reads + last-iterate writes
        print(json.dumps({'config': name, 'k_max': kmax, 'ms': round(ms, 4),
                          'GBps': round(by / ms / 1e6, 1), 'frac': round(by / ms / 1e6 / peak, 3)}))
        del X, AX
