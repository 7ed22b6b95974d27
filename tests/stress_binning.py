"""Stress the binning chain (depth sort -> preprocess -> scan -> duplicate -> onesweep ->
ranges) with many random shapes/sizes in one process, several contexts and models alive at
once; every result is validated against the CPU oracle. Run on the GPU box:

    python tests/stress_binning.py [iterations]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bind as B  # noqa: E402
import paper_2412_13547_b200 as P  # noqa: E402
from tests.helpers import model_from_scene  # noqa: E402


def main(iters):
    B.set_math(True)
    rng = np.random.default_rng(int(time.time()))
    ctxs = [P.Context(0) for _ in range(2)]
    keep = []
    fails = 0
    for it in range(iters):
        ctx = ctxs[it % 2]
        W = int(rng.integers(1, 700))
        H = int(rng.integers(1, 500))
        n = int(rng.integers(0, 60000))
        p = int(rng.integers(1, 4))
        s = B.synthetic_scene(int(rng.integers(1 << 30)), n, W, H)
        if it % 5 == 0 and n:
            s.id = rng.permutation(np.arange(n, dtype=np.uint64) * 3 + 7)
        dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
        if it % 7 == 0:
            keep.append(dm)  # keep some models (and their memory) alive
        try:
            off, items = dm.stage_tile_lists(p, W, H)
        except Exception as e:  # noqa: BLE001
            print("ERROR", it, W, H, n, p, e, flush=True)
            fails += 1
            continue
        roff, ritems = B.tile_grid(s, p, W, H)
        if not (np.array_equal(off, roff) and np.array_equal(items, ritems)):
            print("MISMATCH", it, W, H, n, p, flush=True)
            fails += 1
        if it % 3 == 0 and n:
            ox, oy = int(rng.integers(0, p)), int(rng.integers(0, p))
            if ox < W and oy < H:
                out = dm.render(P.DilationPattern(p, ox, oy, W, H))
                ref = B.render(s, p, ox, oy, W, H)
                if np.abs(out.colors - ref[0]).max(initial=0) > 2e-3:
                    print("RENDER MISMATCH", it, flush=True)
                    fails += 1
        if len(keep) > 6:
            keep.pop(0).close()
    print(f"stress done: {iters} iterations, {fails} failures", flush=True)
    return fails


if __name__ == "__main__":
    sys.exit(1 if main(int(sys.argv[1]) if len(sys.argv) > 1 else 300) else 0)
