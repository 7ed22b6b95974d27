"""Averaged screen-space position-gradient norms of the 3-D fit (bench c9 scene) after N steps:
the scale tau_pos must be set at for the 3-D densifier to select a few percent of the model."""
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2412_13547_b200 as P  # noqa: E402
from paper_2412_13547_b200 import scene3d as S3  # noqa: E402

W, H, n, views = 1920, 1080, 1_000_000, 8
ctx = P.Context(0)
fx = 0.5 * W / math.tan(math.radians(30))
cams = [S3.Camera.look_at((0.3 * math.cos(a), 0.2 * math.sin(a), 0.0), (0.0, 0.0, 4.5), (0, -1, 0), 60.0, W, H)
        for a in np.linspace(0, 2 * math.pi, views, endpoint=False)]
cam0 = S3.Camera(np.eye(3), np.zeros(3), fx, fx, W / 2, H / 2, W, H)
dm = S3.DeviceModel3D.from_host(S3.GaussianModel3D.synthetic(1, n, cam0), ctx)
tm = S3.DeviceModel3D.from_host(S3.GaussianModel3D.synthetic(2, n, cam0), ctx)
targets = [tm.render(c).colors.reshape(H, W, 3).copy() for c in cams]
tm.close()
for it in range(int(sys.argv[1]) if len(sys.argv) > 1 else 100):
    pat = P.DilationPattern(2, it % 2, (it // 2) % 2, W, H) if it < 60 else None
    dm.fit_step(cams[it % views], pat, (0.0, 0.0, 0.0), targets[it % views], it + 1, 1000, 3.0)
pos, col, vis = dm.stats()
avg = pos / np.maximum(vis, 1)
cavg = col / np.maximum(vis, 1)
q = [0.5, 0.75, 0.9, 0.95, 0.99]
print("visited", float((vis > 0).mean()), "pos avg quantiles", [float(np.quantile(avg[vis > 0], x)) for x in q])
print("col avg quantiles", [float(np.quantile(cavg[vis > 0], x)) for x in q])
