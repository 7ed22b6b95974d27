"""Per-phase timing of the bench C8 schedule (warm-up / densify window / post-densify / batched
finale) and per-stage CUDA-event totals, to see where the fit loop spends its time beyond the
per-iteration kernels."""
import json
import math
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2412_13547_b200 as P  # noqa: E402

cfg = bench.CONFIGS["c8"]
W, H, n, p, iters = cfg["W"], cfg["H"], cfg["n"], cfg["p"], cfg["iters"]
ctx = P.Context(0)
host = P.GaussianModel.synthetic(1, n, W, H)
tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(2, n, W, H), ctx)
clean = torch.from_numpy(tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3)).cuda()
tm.close()
targets = []
for v in range(cfg["views"]):
    g = torch.Generator(device="cuda").manual_seed(2000 + v)
    targets.append((clean + 0.02 * torch.randn(clean.shape, generator=g, device="cuda")).clamp(0, 1).contiguous())
tcfg = P.train_config(total_iters=iters, warmup_iters=100, densify_interval=20, densify_until=600,
                      batch_final_iters=100, batch_size=4, dilation_p=p, n_views=cfg["views"], m_final=1.5 * n, seed=1)
tcfg.densify.tau_pos = 5e-8
dm = P.DeviceModel.from_host(host, ctx)
tr = P.Trainer(dm, W, H, tcfg)
tr.set_targets([t.data_ptr() for t in targets])
stream = torch.cuda.ExternalStream(ctx.L.tgsx_get_stream(ctx.h))
prof = "--profile" in sys.argv
if prof:
    ctx.profile(True)
torch.cuda.synchronize()
bounds = [0, 100, 600, 900, 1000]
evs = [torch.cuda.Event(enable_timing=True) for _ in bounds]
import time
t0 = time.time()
walls = []
for k in range(len(bounds) - 1):
    evs[k].record(stream)
    tw = time.time()
    for it in range(bounds[k], bounds[k + 1]):
        tr.step()
    walls.append(time.time() - tw)
evs[-1].record(stream)
evs[-1].synchronize()
out = {"phases_ms": [evs[k].elapsed_time(evs[k + 1]) for k in range(len(bounds) - 1)],
       "host_enqueue_s": walls, "total_s": time.time() - t0}
if prof:
    pr = ctx.profile_read()
    out["stages_ms_total"] = {k: round(v[0], 2) for k, v in pr.items() if v[1]}
    out["stages_launches"] = {k: v[1] for k, v in pr.items() if v[1]}
print(json.dumps(out))
