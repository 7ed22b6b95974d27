"""Generates the committed golden fixtures from the UNMODIFIED reference (oracle/_ref, built
from /root/reference by oracle/Makefile). Run in the build container (needs /root/reference):

    python tests/golden/make_golden.py

Fixtures (small, seeded, see SURVEY.md §8d generator):
  c1_small.npz  — 2000 Gaussians, 128x96: render (p=1 and p=2 offsets (1,0)), backward with
                  seeded dL/dC, stats after backward, per-tile lists, prepared splats, sorted
                  order; reference built with the correctly-rounded libm interposer (ref_cr)
                  and with glibc libm (ref_native).
  fd64.npz      — fp64 render/backward of 8x8 scenes with 5 Gaussians (SPEC.md:671 oracle).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import bind as B  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def scene_arrays(s):
    return {f"scene_{f}": getattr(s, f) for f in B.ALL_FIELDS}


def main():
    B.build()
    assert B.ref_available(), "oracle/_ref not built (needs /root/reference)"
    W, H, n = 128, 96, 2000
    s = B.synthetic_scene(7, n, W, H)
    out = dict(scene_arrays(s), W=W, H=H)
    rng = np.random.default_rng(11)
    for kind in ("cr", "native"):
        impl = f"ref_{kind}"
        for tag, (p, ox, oy) in (("p1", (1, 0, 0)), ("p2", (2, 1, 0))):
            rgb, T, ops, _ = B.render(s, p, ox, oy, W, H, (0.1, 0.2, 0.3), impl=impl)
            out[f"{kind}_{tag}_rgb"] = rgb
            out[f"{kind}_{tag}_T"] = T
            out[f"{kind}_{tag}_ops"] = np.uint64(ops)
            dl = rng.normal(size=rgb.shape).astype(np.float32) * 1e-3
            out[f"{kind}_{tag}_dLdC"] = dl
            s2 = s.copy().ensure_stats()
            g, _ = B.backward(s2, p, ox, oy, W, H, dl, (0.1, 0.2, 0.3), impl=impl)
            out[f"{kind}_{tag}_grads"] = g
            out[f"{kind}_{tag}_pos_acc"] = s2.pos_acc
            out[f"{kind}_{tag}_col_acc"] = s2.col_acc
            out[f"{kind}_{tag}_visit"] = s2.visit
        off, items = B.tile_grid(s, 1, W, H, impl=impl)
        out[f"{kind}_tiles_offsets"] = off
        out[f"{kind}_tiles_items"] = items
        prep = B.prepare(s, 1, impl=impl)
        for k, v in prep.items():
            out[f"{kind}_prep_{k}"] = v
    out["sorted_order"] = B.sorted_order(s, impl="ref_cr")
    np.savez_compressed(os.path.join(OUT, "c1_small.npz"), **out)

    # fp64 finite-difference fixture: 8x8 image, 5 Gaussians, 20 scenes
    fd = {}
    for i in range(20):
        t = B.synthetic_scene(100 + i, 5, 8, 8)
        t.lsx[:] = np.float32(0.2) + t.lsx * np.float32(0.3)
        t.lsy[:] = np.float32(0.2) + t.lsy * np.float32(0.3)
        for f in B.ALL_FIELDS:
            fd[f"s{i}_{f}"] = getattr(t, f)
        for p in (1, 2):
            pat = (p, 0, 0)
            rgb, T, _, _ = B.render(t, *pat, 8, 8, (0.2, 0.3, 0.4), impl="ref_native", dtype=np.float64)
            dl = np.random.default_rng(i).normal(size=rgb.shape)
            t2 = t.copy()
            g, _ = B.backward(t2, *pat, 8, 8, dl, (0.2, 0.3, 0.4), impl="ref_native", dtype=np.float64)
            fd[f"s{i}_p{p}_rgb"] = rgb
            fd[f"s{i}_p{p}_dLdC"] = dl
            fd[f"s{i}_p{p}_grads"] = g
    np.savez_compressed(os.path.join(OUT, "fd64.npz"), **fd)
    for f in ("c1_small.npz", "fd64.npz"):
        print(f, os.path.getsize(os.path.join(OUT, f)), "bytes")


if __name__ == "__main__":
    main()
