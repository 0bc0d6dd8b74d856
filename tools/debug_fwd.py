import sys, numpy as np
sys.path.insert(0, '.')
import torch
from oracle import oracle as O
from paper_2602_17892_b200 import ct, problems
d = np.load('tests/golden/small_ops.npz')
names = sorted({k.split('/')[0] for k in d.files})
for nm in names:
    nx, ny, h, D, sp = d[f'{nm}/params']; ang = d[f'{nm}/angles']
    g = ct.DeviceGeometry(ct.ImageGrid(int(nx), int(ny), h), ct.ParallelGeometry(ang, int(D), sp), 0)
    y = g.forward(torch.from_numpy(d[f'{nm}/x'].astype(np.float32)).cuda()).cpu().numpy().reshape(len(ang), -1)
    ref = d[f'{nm}/Ax'].reshape(len(ang), -1)
    err = np.abs(y - ref).max(axis=1) / max(1e-30, np.abs(ref).max())
    print(nm, ' '.join(f'{e:.1e}' for e in err))
spec = problems.CONFIGS['c1']
g = ct.DeviceGeometry(ct.ImageGrid(128, 128, 1.0), ct.ParallelGeometry(spec.angles(), 183, 1.0), 0)
z = np.load('tests/golden/c1.npz')
xt = problems.random_ellipse_phantom(128, 10, 0)
y = g.forward(torch.from_numpy(xt.astype(np.float32)).cuda()).cpu().numpy().reshape(180, -1)
ref = z['Ax_true'].reshape(180, -1)
err = np.linalg.norm(y - ref, axis=1) / np.linalg.norm(ref, axis=1)
bad = np.where(err > 1e-5)[0]
print('c1 bad angles', bad[:40], err[bad[:10]])
