"""A/B helper: device time of tgsx_loss (dense pattern, SSIM weight 0.2 -> L1 + SSIM stats + SSIM
gradient + finalize) on device-resident images, per library build.

python tools/loss_bench.py [--sizes 1920x1080,3840x2160] [--iters 200] LIB [LIB ...]"""
import argparse
import ctypes as C
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(sizes, iters):
    sys.path.insert(0, ROOT)
    import torch
    import paper_2412_13547_b200 as P
    ctx = P.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    g = torch.Generator(device="cuda").manual_seed(1)
    for s in sizes:
        W, H = (int(v) for v in s.split("x"))
        rgb = torch.rand(H * W * 3, device="cuda", generator=g)
        tgt = torch.rand(H * W * 3, device="cuda", generator=g)
        grad = torch.empty_like(rgb)
        loss = torch.zeros(1, device="cuda")
        pat = P.DilationPattern(1, 0, 0, W, H).c()

        def run():
            ctx.check(ctx.L.tgsx_loss(ctx.h, C.byref(pat), C.c_void_p(rgb.data_ptr()), C.c_void_p(tgt.data_ptr()),
                                      C.c_float(0.2), C.c_void_p(loss.data_ptr()), C.c_void_p(grad.data_ptr())))
        for _ in range(5):
            run()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(iters):
            run()
        b.record()
        torch.cuda.synchronize()
        print(json.dumps({"lib": os.environ.get("TGSX_LIB", "in-tree"), "size": s,
                          "ms": round(a.elapsed_time(b) / iters, 4), "loss": float(loss.item()),
                          "grad_sum": float(grad.double().abs().sum().item())}), flush=True)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1920x1080,3840x2160")
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--child", action="store_true")
    ap.add_argument("libs", nargs="*")
    a = ap.parse_args()
    if a.child:
        child(a.sizes.split(","), a.iters)
        sys.exit(0)
    for lib in a.libs or ["in-tree"]:
        env = dict(os.environ)
        if lib != "in-tree":
            env["TGSX_LIB"] = os.path.abspath(lib)
        subprocess.call([sys.executable, __file__, "--child", "--sizes", a.sizes, "--iters", str(a.iters)], env=env)
