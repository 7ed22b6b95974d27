"""A/B helper: per-stage CUDA-event times of the fit step for one or more library builds.

python tools/stages.py [--configs c2,c3] [--steps 50] LIB [LIB ...]
Each LIB (a libtgsx.so path, e.g. exp/<name>/libtgsx.so or the in-tree build) runs in its own
process (TGSX_LIB), from the same initial model as bench.py, and prints one line per config:
stage ms per step + counters; a build with TGSX_BWD_STATS also reports the backward's
union-row statistics."""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CFG = {"c1": (10_000, 256, 256, 1), "c2": (1_000_000, 1920, 1080, 1), "c3": (3_000_000, 3840, 2160, 2)}


def child(cfgs, steps):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    import paper_2412_13547_b200 as P
    L = P._lib.load()
    stats = getattr(L, "tgsx_debug_bwd_stats", None) if hasattr(L, "tgsx_debug_bwd_stats") else None
    ctx = P.Context(0)
    for name in cfgs:
        n, W, H, p = CFG[name]
        diag = float(np.hypot(W, H))
        dm = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, n, W, H), ctx)
        tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(2, n, W, H), ctx)
        tgt = torch.from_numpy(tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3)).cuda()
        tm.close()
        loss = torch.zeros(1, device="cuda")
        bg = (C.c_float * 3)(0, 0, 0)

        def step(it):
            ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
            pat = P.DilationPattern(p, ox, oy, W, H).c()
            a = P._lib.AdamArgs(it + 1, 10000, diag)
            ctx.check(ctx.L.tgsx_fit_step(ctx.h, dm.h, C.byref(pat), bg, C.c_void_p(tgt.data_ptr()),
                                          C.byref(a), C.c_void_p(loss.data_ptr())))
        for it in range(3):
            step(it)
        torch.cuda.synchronize()
        if stats:
            buf = (C.c_uint64 * 16)()
            stats(buf)
        ctx.profile(True)
        for it in range(3, 3 + steps):
            step(it)
        torch.cuda.synchronize()
        prof = ctx.profile_read()
        ctx.profile(False)
        out = {"config": name, "lib": os.environ.get("TGSX_LIB", "in-tree")}
        out["ms"] = {k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items() if v[1]}
        out["total_ms"] = round(sum(v[0] for v in prof.values()) / steps, 4)
        out["counters"] = ctx.counters()
        if stats:
            stats(buf)
            s = [b / steps for b in buf]
            out["bwd"] = {"group_chunks": s[0], "rows": s[1], "blends": s[2], "u0u1": s[3],
                          "rounds": s[4], "chunks": s[5], "box_blends": s[6], "quarter_rows": s[7], "lane_max": s[8], "lane_sum": s[9],
                          "row_util": s[2] / max(64 * s[1], 1), "lockstep_util": s[3] / max(2 * s[1], 1)}
        print(json.dumps(out), flush=True)
        dm.close()


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="c2,c3")
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.configs.split(","), a.steps)
        sys.exit(0)
    for lib in a.libs or ["in-tree"]:
        env = dict(os.environ)
        if lib != "in-tree":
            env["TGSX_LIB"] = os.path.abspath(lib)
        subprocess.call([sys.executable, __file__, "--child", "--configs", a.configs, "--steps", str(a.steps)],
                        env=env)
