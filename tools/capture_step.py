"""Runs `--warmup` + `--steps` fused fit steps of a bench config (same model / target as bench.py)
and prints each step's counters (blend ops, evaluations, pairs) as one JSON line — the work of the
launches an ncu capture of this command selects with `-s 2*warmup -c 2` (forward + backward of
the first step after the warm-up)."""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
CFG = {"c1": (10_000, 256, 256, 1), "c2": (1_000_000, 1920, 1080, 1), "c3": (3_000_000, 3840, 2160, 2)}

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c2")
ap.add_argument("--warmup", type=int, default=3)
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2412_13547_b200 as P  # noqa: E402

n, W, H, p = CFG[a.config]
ctx = P.Context(0)
dm = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, n, W, H), ctx)
tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(2, n, W, H), ctx)
tgt = torch.from_numpy(tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3)).cuda()
tm.close()
loss = torch.zeros(1, device="cuda")
torch.cuda.synchronize()
bg = (C.c_float * 3)(0, 0, 0)
diag = float(np.hypot(W, H))
for it in range(a.warmup + a.steps):
    ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
    pat = P.DilationPattern(p, ox, oy, W, H).c()
    args = P._lib.AdamArgs(it + 1, 10000, diag)
    ctx.check(ctx.L.tgsx_fit_step(ctx.h, dm.h, C.byref(pat), bg, C.c_void_p(tgt.data_ptr()), C.byref(args),
                                  C.c_void_p(loss.data_ptr())))
    ctx.synchronize()
    print(json.dumps({"config": a.config, "step": it, "warmup": it < a.warmup, **ctx.counters()}), flush=True)
