"""The C++ drop-in (tgs::render<float> / tgs::backward<float> with the reference's signatures,
paper_2412_13547_b200/shim/tgs_gpu_rasterizer.cpp) driven through the reference's own public
API (tests/shim_check.cpp, built against /root/reference headers in the build container), checked
against the CPU oracle on the same scene."""
import os
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import frac_close

pytestmark = pytest.mark.gpu
BIN = os.path.join(os.path.dirname(__file__), "_bin", "shim_check")


@pytest.mark.skipif(not os.path.exists(BIN), reason="shim_check not built (needs reference headers)")
def test_cpp_shim_render_backward_match_oracle():
    B.set_math(True)
    with tempfile.TemporaryDirectory() as d:
        out = os.path.join(d, "o.bin")
        r = subprocess.run([BIN, out], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0, r.stdout + r.stderr
        raw = open(out, "rb").read()
    n, P = np.frombuffer(raw[:16], np.int64)
    ops = int(np.frombuffer(raw[16:24], np.uint64)[0])
    o = 24
    rgb = np.frombuffer(raw[o:o + 12 * P], np.float32).reshape(P, 3)
    o += 12 * P
    T = np.frombuffer(raw[o:o + 4 * P], np.float32)
    o += 4 * P
    g = np.frombuffer(raw[o:o + 36 * n], np.float32).reshape(9, n)
    o += 36 * n
    pos = np.frombuffer(raw[o:o + 4 * n], np.float32)
    o += 8 * n
    visit = np.frombuffer(raw[o:o + 8 * n], np.int64)
    # same scene through the oracle: reference Pcg32(7, 1), generator order of shim_check.cpp
    W, H = 160, 112
    s = B.synthetic_scene(7, int(n), W, H)
    rrgb, rT, rops, _ = B.render(s, 2, 1, 0, W, H, (0.1, 0.2, 0.3))
    assert np.abs(rgb - rrgb).max() <= 2e-3 and (np.abs(rgb - rrgb).max(1) > 1e-5).mean() <= 1e-3
    assert abs(ops - rops) <= 2
    rng_vals = B.Pcg32(9, 1)
    dl = np.array([[rng_vals.uniform() for _ in range(3)] for _ in range(P)])
    dl = (-1e-3 + 2e-3 * dl).astype(np.float32)
    gr, _ = B.backward(s.copy(), 2, 1, 0, W, H, dl, (0.1, 0.2, 0.3))
    for q in range(9):
        scale = np.abs(gr[q]).max()
        assert frac_close(g[q], gr[q], 1e-3, 1e-5 * scale) >= 0.995, q
    s2 = s.copy().ensure_stats()
    B.backward(s2, 2, 1, 0, W, H, dl, (0.1, 0.2, 0.3))
    assert np.abs(visit - s2.visit).sum() <= 3
    assert np.allclose(pos, s2.pos_acc, rtol=2e-3, atol=1e-9)
