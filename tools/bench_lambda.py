"""Host cost of one native projected solve (SVD + lambda grid + Tikhonov) vs k."""
import ctypes, os, sys, time
sys.path.insert(0, '.')
import numpy as np
from threadpoolctl import threadpool_limits
from paper_2602_17892_b200 import _native
L = _native.load()
print('cpus', os.cpu_count(), len(os.sched_getaffinity(0)))
rng = np.random.default_rng(0)
with threadpool_limits(limits=1, user_api='blas'):
    for k in (10, 20, 40, 60, 80, 100):
        H = np.triu(rng.standard_normal((k + 1, k)), -1)
        out = np.zeros(4); y = np.zeros(k)
        for strat in (3, 2):
            L.ctk_projected_solve(H.ctypes.data, k, 2.0, strat, 0.0, 200, float('nan'), out.ctypes.data, y.ctypes.data)
            t = time.perf_counter()
            for _ in range(20):
                L.ctk_projected_solve(H.ctypes.data, k, 2.0, strat, 0.0, 200, float('nan'), out.ctypes.data, y.ctypes.data)
            print(k, 'gcv' if strat == 3 else 'lcurve', '%.0f us' % ((time.perf_counter() - t) / 20 * 1e6))
