"""Run-to-run spread of the C9 fit loop (bench.py measure_fit3d's setup): per-iteration host wall
times of trainer.step() and device time per 50 iterations, to tell host stalls from GPU time.
python tools/c9_probe.py [--runs 1]"""
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2412_13547_b200 as P  # noqa: E402
from paper_2412_13547_b200 import scene3d as S3  # noqa: E402

cfg = bench.CONFIGS["c9"]
W, H, n, p, iters, views = cfg["W"], cfg["H"], cfg["n"], cfg["p"], cfg["iters"], cfg["views"]
ctx = P.Context(0)
fx = 0.5 * W / math.tan(math.radians(30))
cams = [S3.Camera.look_at((0.3 * math.cos(a), 0.2 * math.sin(a), 0.0), (0.0, 0.0, 4.5), (0, -1, 0), 60.0, W, H)
        for a in np.linspace(0, 2 * math.pi, views, endpoint=False)]
cam0 = S3.Camera(np.eye(3), np.zeros(3), fx, fx, W / 2, H / 2, W, H)
dm = S3.DeviceModel3D.from_host(S3.GaussianModel3D.synthetic(1, n, cam0), ctx)
tm = S3.DeviceModel3D.from_host(S3.GaussianModel3D.synthetic(2, n, cam0), ctx)
targets = [torch.from_numpy(tm.render(c).colors.reshape(H, W, 3).copy()).cuda().contiguous() for c in cams]
tm.close()
tcfg = P.train_config(total_iters=iters, warmup_iters=100, densify_interval=20, densify_until=400,
                      batch_final_iters=50, batch_size=4, dilation_p=p, n_views=views, m_final=1.5 * n, seed=1)
tcfg.densify.tau_pos = 6e-8
trainer = S3.Trainer3D(dm, cams, 3.0, tcfg)
trainer.set_targets([t.data_ptr() for t in targets])
stream = torch.cuda.ExternalStream(ctx.L.tgsx_get_stream(ctx.h))
torch.cuda.synchronize()
ctx.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(iters // 50 + 1)]
host = []
t0 = time.perf_counter()
ev[0].record(stream)
for it in range(iters):
    a = time.perf_counter()
    rep = trainer.step()
    host.append((time.perf_counter() - a, it + 1, int(rep.densified)))
    if (it + 1) % 50 == 0:
        ev[(it + 1) // 50].record(stream)
ctx.synchronize()
wall = time.perf_counter() - t0
seg = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(ev) - 1)]
host.sort(reverse=True)
print({"wall_s": round(wall, 3), "device_ms_per_50": [round(x, 1) for x in seg],
       "host_top": [(round(h * 1e3, 2), i, d) for h, i, d in host[:8]],
       "host_median_ms": round(float(np.median([h for h, _, _ in host])) * 1e3, 3)}, flush=True)
