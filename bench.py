"""Benchmark: Turbo-GS fit iterations/s on B200 (BASELINE.json metric).

Workload (N=1, BASELINE.json configs[1], "C2"): synthetic 1M Gaussians (seed 1), 1920x1080,
dense (p=1) single-view fit step = preprocess -> onesweep binning -> blend forward + fused L1
-> blend backward -> chain rule + densify stats + Adam, through libtgsx. The loss target is the
render of the seed-2 synthetic scene. `--config c3` runs configs[2] (3M Gaussians, 3840x2160,
dilated p=2 with cycled offsets). With N>1 ranks (torchrun) every rank fits its own view per
step and the per-Gaussian step buffer (9 grads + densify stats) is all-reduced over NCCL
before the identical Adam on every rank (view-batch data parallelism).

Timing: W warm-up steps, then K steps bracketed by barrier + synchronize, timed with CUDA
events on the library's stream, max over ranks. Working set per step (model state + moments
+ pairs + partials, >600 MB at C2) exceeds the 126 MB L2, so no explicit flush.

`--impl reference` times the reference CPU path on this host (oracle/_ref: the unmodified
reference render/backward compiled from /root/reference, + the oracle's restated L1/Adam)
on the same workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    "c2": dict(workload="C2: synthetic 1M Gaussians, 1920x1080, p=1 single-view fit step "
                        "(fwd + L1 + bwd + densify stats + Adam)",
               n=1_000_000, W=1920, H=1080, p=1),
    "c3": dict(workload="C3: synthetic 3M Gaussians, 3840x2160, dilated p=2 (cycled offsets) "
                        "fit step (fwd + L1 + bwd + densify stats + Adam)",
               n=3_000_000, W=3840, H=2160, p=2),
}
METRIC = "fit iters/sec (fwd+bwd+Adam) at 1080p and 4K dilated, 1M–3M Gaussians"


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.th = threading.Thread(target=self.run, daemon=True)

    def run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index),
                                      f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.th.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        self.th.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "fallback": True}


# ---------------------------------------------------------------------------- reference arm
def run_reference(args, cfg):
    rank, world, _ = env_rank()
    if rank != 0:
        return
    from oracle import bind as B
    threads = os.cpu_count() or 1
    W, H, n, p = cfg["W"], cfg["H"], cfg["n"], cfg["p"]
    impl = "ref_native" if B.ref_available() else "oracle"
    B.set_math(False)
    s = B.synthetic_scene(1, n, W, H)
    t = B.synthetic_scene(2, n, W, H)
    target, _, _, _ = B.render(t, 1, 0, 0, W, H, impl=impl, threads=threads)
    target = target.reshape(H, W, 3)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)
    diag = float(np.hypot(W, H))

    def step(it):
        ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
        rgb, _, _, _ = B.render(s, p, ox, oy, W, H, impl=impl, threads=threads)
        _, dl = B.l1_loss(rgb, p, ox, oy, W, H, target)
        g, _ = B.backward(s, p, ox, oy, W, H, dl, impl=impl, threads=threads)
        B.adam_step(s, g, m1, m2, B.adam_config(it + 1, 10000, diag))

    for i in range(args.warmup):
        step(i)
    t0 = time.perf_counter()
    for i in range(args.steps):
        step(args.warmup + i)
    dt = time.perf_counter() - t0
    v = args.steps / dt
    kind = "reference" if impl != "oracle" else "port"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "gaussians": n, "width": W, "height": H, "p": p},
            "cpu_baseline": {"value": v, "unit": "iters/s", "cores": threads, "kind": kind,
                             "sample": f"{args.steps} full fit iterations on {threads} host threads "
                                       "(reference render+backward from oracle/_ref, restated L1+Adam)"},
            "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_sample(cfg, iters=2):
    """Bounded CPU sample of the same workload (oracle/_ref, all host threads)."""
    from oracle import bind as B
    threads = os.cpu_count() or 1
    W, H, n, p = cfg["W"], cfg["H"], cfg["n"], cfg["p"]
    impl = "ref_native" if B.ref_available() else "oracle"
    B.set_math(False)
    s = B.synthetic_scene(1, n, W, H)
    t = B.synthetic_scene(2, n, W, H)
    target, _, _, _ = B.render(t, 1, 0, 0, W, H, impl=impl, threads=threads)
    target = target.reshape(H, W, 3)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)
    diag = float(np.hypot(W, H))
    times = []
    for it in range(iters + 1):
        ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
        t0 = time.perf_counter()
        rgb, _, _, _ = B.render(s, p, ox, oy, W, H, impl=impl, threads=threads)
        _, dl = B.l1_loss(rgb, p, ox, oy, W, H, target)
        g, _ = B.backward(s, p, ox, oy, W, H, dl, impl=impl, threads=threads)
        B.adam_step(s, g, m1, m2, B.adam_config(it + 1, 10000, diag))
        times.append(time.perf_counter() - t0)
    med = statistics.median(times[1:])  # first iteration absorbs the blend-order sort
    return {"value": 1.0 / med, "unit": "iters/s", "cores": threads,
            "kind": "reference" if impl != "oracle" else "port",
            "sample": f"median of {iters} full fit iterations after 1 warm-up, same config "
                      "(reference render+backward from oracle/_ref, restated L1+Adam)"}


# ---------------------------------------------------------------------------- tgsx arm
def run_tgsx(args, cfg):
    import torch
    import paper_2412_13547_b200 as P

    rank, world, local = env_rank()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    W, H, n, p = cfg["W"], cfg["H"], cfg["n"], cfg["p"]
    diag = float(np.hypot(W, H))
    ctx = P.Context(local)
    stream = torch.cuda.ExternalStream(ctx.L.tgsx_get_stream(ctx.h))
    host = P.GaussianModel.synthetic(1, n, W, H)
    dm = P.DeviceModel.from_host(host, ctx)
    # target: render of the seed-2 scene on the GPU (+ per-rank noise for N>1 distinct views)
    tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(2, n, W, H), ctx)
    tgt = tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3)
    tm.close()
    target = torch.from_numpy(tgt).cuda()
    if world > 1:
        g = torch.Generator(device="cuda").manual_seed(1000 + rank)
        target = target + 0.02 * torch.randn(target.shape, generator=g, device="cuda")
    target = target.contiguous()
    loss_dev = torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    step_ptr, step_floats = dm.step_buffer()

    class _CudaArray:
        # zero-copy torch view of the library's [12][cap] step buffer, all-reduced by NCCL
        __cuda_array_interface__ = {"shape": (step_floats,), "typestr": "<f4",
                                    "data": (step_ptr, False), "version": 3, "stream": None}

    step_tensor = torch.as_tensor(_CudaArray(), device="cuda") if world > 1 else None
    bg = (C.c_float * 3)(0, 0, 0)

    def one_step(it, tptr, lptr):
        ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
        pat = P.DilationPattern(p, ox, oy, W, H).c()
        a = P._lib.AdamArgs(it + 1, 10000, diag)
        if world == 1:
            ctx.check(ctx.L.tgsx_fit_step(ctx.h, dm.h, C.byref(pat), bg, tptr, C.byref(a), lptr))
        else:
            ctx.check(ctx.L.tgsx_view_accumulate(ctx.h, dm.h, C.byref(pat), bg, tptr, lptr))
            with torch.cuda.stream(stream):
                dist.all_reduce(step_tensor)
            ctx.check(ctx.L.tgsx_apply_step(ctx.h, dm.h, world, C.byref(a)))

    tptr = C.c_void_p(target.data_ptr())
    lptr = C.c_void_p(loss_dev.data_ptr())
    for i in range(args.warmup):
        one_step(i, tptr, lptr)
    ctx.synchronize()

    def timed(fn, steps, base):
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ctx.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            fn(base + i)
        e1.record(stream)
        e1.synchronize()
        ctx.synchronize()
        ms = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms

    # device-resident run (the `value`), with live per-stage CUDA events
    launches0 = ctx.launches
    ctx.profile(True)
    with ClockSampler(local) as clk:
        ms = timed(lambda it: one_step(it, tptr, lptr), args.steps, args.warmup)
    stages = ctx.profile_read()
    ctx.profile(False)
    launches = ctx.launches - launches0
    counters = ctx.counters()
    # e2e through the public API with host buffers: pinned target H2D + loss D2H every step
    h_target = torch.from_numpy(tgt).pin_memory() if world == 1 else target.cpu().pin_memory()
    h_loss = torch.zeros(1).pin_memory()
    e2e_ms = timed(lambda it: one_step(it, C.c_void_p(h_target.data_ptr()),
                                       C.c_void_p(h_loss.data_ptr())), args.steps,
                   args.warmup + args.steps)
    if rank != 0:
        dist.barrier()
        dist.destroy_process_group()
        return
    value = world * args.steps / (ms / 1e3)
    e2e = world * args.steps / (e2e_ms / 1e3)
    clocks = clk.summary()
    peaks = measured_peaks()
    # roofline of the dominant kernel (per launch: stage ms / launch count)
    per = {k: (v[0] / max(v[1], 1), v[1]) for k, v in stages.items() if v[1]}
    dom = max(per, key=lambda k: per[k][0] * per[k][1])
    dom_ms = per[dom][0]
    E, Bl, K = counters["evals"], counters["blend_ops"], counters["pairs"]
    f_mhz = clocks["sm_mhz"] or peaks.get("clocks_under_load", {}).get("sm_mhz_median", 1342.0)
    fp32_peak = 148 * 128 * 2 * f_mhz * 1e6 / 1e12  # TFLOP/s at the sampled SM clock
    if dom in ("blend_backward", "blend_forward"):
        flops = (2 * E + 77 * Bl) if dom == "blend_backward" else (2 * E + 20 * Bl)
        achieved = flops / (dom_ms / 1e3) / 1e12
        roof = {"kernel": dom, "bound": "fp32", "achieved": achieved, "peak": fp32_peak,
                "unit": "TFLOP/s", "frac": achieved / fp32_peak, "traffic": None,
                "peak_note": "148 SM x 128 FP32 lanes x 2 x median sampled SM clock "
                             "(MEASURED_PEAKS.json has no FP32 figure)",
                "work_note": f"algorithmic flops per launch 2E+{77 if dom == 'blend_backward' else 20}Bl "
                             f"with E={E} evaluations, Bl={Bl} blends (SURVEY.md §8d)"}
    else:
        nb = {"chain_adam": 400 * n, "preprocess": 108 * n, "radix_sort": 32 * K,
              "duplicate": 8 * K + 20 * n}.get(dom, 0)
        achieved = nb / (dom_ms / 1e3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": None}
    line = {"metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": cfg["workload"], "gaussians": n, "width": W, "height": H,
                       "p": p, "views_per_step": world,
                       "l2": "per-step working set > 126 MB L2 (no explicit flush)"},
            "clocks": clocks,
            "e2e": {"value": e2e, "unit": "iters/s", "h2d_bytes_per_step": W * H * 12,
                    "d2h_bytes_per_step": 4},
            "gpu_launches": launches,
            "roofline": roof,
            "stages_ms_per_step": {k: v[0] / args.steps for k, v in stages.items() if v[1]},
            "counters": {"pairs": K, "evals": E, "blend_ops": Bl}}
    if world == 1 and not args.no_cpu_baseline:
        try:
            line["cpu_baseline"] = cpu_baseline_sample(cfg)
        except Exception as e:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "error": str(e)}
    print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="tgsx", choices=["tgsx", "reference"])
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "tgsx" else args.warmup
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg)
    else:
        run_tgsx(args, cfg)


if __name__ == "__main__":
    main()
