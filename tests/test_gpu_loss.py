"""compute_loss on the device against the oracle restatement (or_loss, itself
pinned by the SPEC examples and finite differences in tests/test_spec_kats.py): dense patterns
(1-w) L1 + w (1 - SSIM), dilated patterns L1 only; and the dense SSIM term inside the fused fit
views. FP32 on the device vs FP64 in the oracle: loss within 1e-5 relative, gradients within
1e-3 relative (plus 1e-3 of the largest component)."""
import math

import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import frac_close, model_from_scene, target_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def _close(a, b):
    scale = np.abs(b).max(initial=0.0)
    return frac_close(a, b, 1e-3, 1e-3 * scale)


@pytest.mark.parametrize("W,H,w", [(16, 16, 0.2), (37, 23, 0.2), (64, 48, 1.0), (200, 120, 0.2)])
def test_dense_loss_matches_oracle(P, ctx, W, H, w):
    rng = np.random.default_rng(W * H)
    rgb = rng.random((W * H, 3)).astype(np.float32)
    tgt = np.clip(rgb.reshape(H, W, 3) + rng.normal(0, 0.1, (H, W, 3)), 0, 1).astype(np.float32)
    loss, g = P.compute_loss(ctx, rgb, tgt, P.DilationPattern(1, 0, 0, W, H), w)
    rl, rg = B.loss(rgb, 1, 0, 0, W, H, tgt, w)
    assert abs(loss - rl) <= 1e-5 * abs(rl)
    assert _close(g, rg) == 1.0


def test_identical_and_dilated(P, ctx):
    W, H = 40, 30
    t = np.random.default_rng(1).random((H, W, 3)).astype(np.float32)
    loss, g = P.compute_loss(ctx, t.reshape(-1, 3), t, P.DilationPattern(1, 0, 0, W, H), 0.2)
    assert abs(loss) < 1e-6 and np.abs(g).max() < 1e-9
    pat = P.DilationPattern(2, 1, 0, W, H)
    x = np.random.default_rng(2).random((pat.active_count(), 3)).astype(np.float32)
    loss, g = P.compute_loss(ctx, x, t, pat, 0.2)  # dilated: L1 only
    rl, rg = B.l1_loss(x, 2, 1, 0, W, H, t)
    assert abs(loss - rl) <= 1e-6 * rl and np.array_equal(g, rg)
    with pytest.raises(ValueError):
        P.compute_loss(ctx, x, t, pat, 1.5)


def test_fullsize_1080p_loss(P, ctx):
    W, H = 1920, 1080
    rng = np.random.default_rng(5)
    tgt = rng.random((H, W, 3)).astype(np.float32)
    rgb = np.clip(tgt.reshape(-1, 3) + rng.normal(0, 0.05, (W * H, 3)), 0, 1).astype(np.float32)
    loss, g = P.compute_loss(ctx, rgb, tgt, P.DilationPattern(1, 0, 0, W, H), 0.2)
    rl, rg = B.loss(rgb, 1, 0, 0, W, H, tgt, 0.2)
    assert abs(loss - rl) <= 1e-5 * abs(rl)
    assert _close(g, rg) >= 0.9999


def test_fused_dense_view_with_ssim_matches_oracle(P, ctx):
    """view_accumulate on a dense view with lambda_ssim = 0.2: loss == oracle compute_loss of the
    render, and one Adam step on the accumulated gradient == oracle backward(dL/dC) + Adam."""
    W, H, n = 96, 80, 1500
    s = B.synthetic_scene(1, n, W, H).ensure_stats()
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    target = target_image(2, n, W, H)
    diag = math.hypot(W, H)
    ctx.set_ssim_weight(0.2)
    try:
        loss = dm.view_accumulate(P.DilationPattern(1, 0, 0, W, H), (0, 0, 0), target)
        dm.apply_step(1, 1, 100, diag)
    finally:
        ctx.set_ssim_weight(0.0)
    B.set_math(True)
    rgb = B.render(s, 1, 0, 0, W, H)[0]
    rl, dl = B.loss(rgb, 1, 0, 0, W, H, target, 0.2)
    assert abs(loss - rl) <= 2e-5 * rl
    g, _ = B.backward(s, 1, 0, 0, W, H, dl)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)
    B.adam_step(s, g, m1, m2, B.adam_config(1, 100, diag))
    h = dm.download()
    for i, f in enumerate(B.PARAM_FIELDS):
        assert frac_close(h.params[i], getattr(s, f), 1e-6, 1e-6) >= 0.995, f
