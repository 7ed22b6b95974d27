"""The SSIM window literals compiled into csrc/loss.cu (module-initialised constant memory) equal
the window the oracle forms at run time (oracle/tgs_oracle.c or_loss: float(g_i / sum g),
g_i = exp(-i^2 / 4.5) in double, summed in order)."""
import math
import os
import re

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_ssim_window_literals_match_formula():
    src = open(os.path.join(ROOT, "paper_2412_13547_b200", "csrc", "loss.cu")).read()
    body = re.search(r"__constant__ float c_win\[2 \* kR \+ 1\] = \{(.*?)\};", src, re.S).group(1)
    lits = [float.fromhex(t.strip().rstrip("f")) for t in body.split(",") if t.strip()]
    g = [math.exp(-(i * i) / (2.0 * 1.5 * 1.5)) for i in range(-5, 6)]
    s = 0.0
    for v in g:
        s += v
    want = [float(np.float32(v / s)) for v in g]
    assert lits == want
