"""GPU parity for the rest of the fit path — densify / prune / audit, batched views — and
size-independent properties at BASELINE.json's full sizes (C2: 1M Gaussians at 1080p; C3: 3M
at 4K dilated)."""
import math
import os

import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import frac_close, model_from_scene, scene_from_model, target_image

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


@pytest.fixture(autouse=True)
def cr_math():
    B.set_math(True)
    yield


def stat_scene(seed, n, W=96, H=96):
    rng = np.random.default_rng(seed)
    s = B.synthetic_scene(seed, n, W, H).ensure_stats()
    s.accum[:] = rng.integers(0, 4, n)
    s.visit[:] = rng.integers(0, 12, n)
    s.window[:] = rng.integers(0, 8, n)
    s.tau_v[:] = rng.choice([1.0, 2.5, 5.0, 8.0], n)
    s.pos_acc[:] = (rng.random(n) * 6e-4 * s.accum).astype(np.float32)
    s.col_acc[:] = (rng.random(n) * 6e-2 * s.accum).astype(np.float32)
    s.rop[:] = rng.uniform(-6, 3, n).astype(np.float32)
    return s


@pytest.mark.parametrize("seed,budget_extra,rng_seed", [(1, 10**6, 5), (2, 37, 11), (3, 0, 2), (4, 500, 13)])
def test_densify_matches_oracle(P, ctx, seed, budget_extra, rng_seed):
    n = 6000
    s = stat_scene(seed, n)
    rng = np.random.default_rng(seed)
    m1 = rng.normal(size=(9, n)).astype(np.float32)
    m2 = rng.random((9, n)).astype(np.float32)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    dm.set_moments(m1, m2)
    budget = n + budget_extra
    gpu_rng = P.Pcg32(rng_seed, 3)
    rep = dm.densify(budget, gpu_rng.state, P.densify_config(tau_pos=2e-4))
    orng = B.Pcg32(rng_seed, 3)
    out, spawned, pruned, ncand, (om1, om2) = B.densify_event(s, n + max(0, budget - n) + 16,
                                                              B.densify_config(2e-4), budget, orng,
                                                              m1, m2)
    assert (rep.candidates, rep.spawned, rep.pruned, rep.count_after) == (ncand, spawned, pruned, out.n)
    assert tuple(gpu_rng.state) == orng.state  # RNG advanced exactly like the sequential draws
    h = dm.download()
    assert np.array_equal(h.id, out.id) and dm.next_id() == out.next_id
    for i, f in enumerate(B.ALL_FIELDS):
        if f in ("px", "py"):
            # child positions: FP64 sin/cos/exp on the device vs glibc (1-ulp double drift)
            assert np.allclose(h.params[i], getattr(out, f), rtol=0, atol=1e-4), f
            assert frac_close(h.params[i], getattr(out, f), 0, 0) >= 0.999
        else:
            assert np.array_equal(h.params[i], getattr(out, f)), f
    assert np.array_equal(h.accum_count, out.accum) and np.array_equal(h.visit_count, out.visit)
    assert np.array_equal(h.pos_grad_norm_accum, out.pos_acc)
    assert np.array_equal(h.visit_thresholds, out.tau_v)
    g1, g2 = dm.moments()
    assert np.array_equal(g1, om1) and np.array_equal(g2, om2)


def test_visit_audit_matches_oracle(P, ctx):
    s = stat_scene(7, 3000)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    dm.visit_audit()
    B.visit_audit(s)
    h = dm.download()
    assert np.array_equal(h.visit_thresholds, s.tau_v) and np.all(h.window_visit_count == 0)


def test_batched_views_match_oracle(P, ctx):
    """4 views (the 4 offsets of p=2) accumulated then one Adam step on the mean
    == oracle: per-view backward (stats per call) + componentwise mean + Adam."""
    W, H, n = 96, 80, 1500
    s = B.synthetic_scene(1, n, W, H).ensure_stats()
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    target = target_image(2, n, W, H)
    diag = math.hypot(W, H)
    gsum = np.zeros((9, n), np.float32)
    losses = []
    for v in range(4):
        ox, oy = P.next_offsets(2, v)
        losses.append(dm.view_accumulate(P.DilationPattern(2, ox, oy, W, H), (0, 0, 0), target))
        rgb = B.render(s, 2, ox, oy, W, H)[0]
        loss, dl = B.l1_loss(rgb, 2, ox, oy, W, H, target)
        assert abs(losses[-1] - loss) <= 1e-5 * loss
        g, _ = B.backward(s, 2, ox, oy, W, H, dl)  # stats accumulate per call, like the reference
        gsum += g
    dm.apply_step(4, 1, 100, diag)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)
    B.adam_step(s, (gsum / np.float32(4)).astype(np.float32), m1, m2, B.adam_config(1, 100, diag))
    h = dm.download()
    assert np.array_equal(h.visit_count, s.visit) or np.abs(h.visit_count - s.visit).sum() <= 3
    for i, f in enumerate(B.PARAM_FIELDS):
        assert frac_close(h.params[i], getattr(s, f), 1e-6, 1e-6) >= 0.995, f
    assert np.allclose(h.pos_grad_norm_accum, s.pos_acc, rtol=2e-3, atol=1e-9)


def test_binning_reuse_invalidated_by_every_model_change(P, ctx):
    """Views of an unchanged model share one binning; each parameter / order change must drop it.
    After render -> adam_step / apply_step / densify / upload, the next render equals the oracle
    render of the changed scene."""
    W, H, n = 80, 64, 1200
    s = B.synthetic_scene(4, n, W, H).ensure_stats()
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    diag = math.hypot(W, H)
    pat = P.DilationPattern(2, 1, 0, W, H)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)

    def check():
        # render first (a stale binning would be used here), then compare with the oracle
        # render of the device's current parameters
        got = dm.render(pat, (0.1, 0.2, 0.3)).colors
        ref = B.render(scene_from_model(dm.download()), 2, 1, 0, W, H, (0.1, 0.2, 0.3))[0]
        assert np.abs(got - ref).max() <= 2e-3 and (np.abs(got - ref).max(axis=1) > 1e-5).mean() <= 1e-3

    dm.render(pat, (0.1, 0.2, 0.3))  # binning cached
    check()
    # explicit-gradient Adam (large steps so that tile rectangles change)
    g = np.random.default_rng(0).normal(size=(9, n)).astype(np.float32) * 50
    dm.render(pat, (0.1, 0.2, 0.3))
    dm.adam_step(g, 1, 100, diag)
    B.adam_step(s, g, m1, m2, B.adam_config(1, 100, diag))
    check()
    # batched views + apply_step
    target = target_image(5, n, W, H)
    gsum = np.zeros((9, n), np.float32)
    for v in range(2):
        ox, oy = P.next_offsets(2, v)
        dm.view_accumulate(P.DilationPattern(2, ox, oy, W, H), (0, 0, 0), target)
        rgb = B.render(s, 2, ox, oy, W, H)[0]
        _, dl = B.l1_loss(rgb, 2, ox, oy, W, H, target)
        gsum += B.backward(s, 2, ox, oy, W, H, dl)[0]
    dm.apply_step(2, 2, 100, diag)
    check()
    # densify (spawn + prune change n and the blend order)
    dm.render(pat, (0.1, 0.2, 0.3))
    dm.densify(dm.size() + 200, P.Pcg32(3, 1).state, P.densify_config(tau_pos=1e-9))
    check()
    # upload of a different scene
    dm.render(pat, (0.1, 0.2, 0.3))
    dm.upload(model_from_scene(B.synthetic_scene(9, n, W, H)))
    check()


# ------------------------------------------------------------------ full-size properties
FULL = {"c2": (1_000_000, 1920, 1080, 1), "c3": (3_000_000, 3840, 2160, 2)}


@pytest.fixture(scope="module")
def c2(P, ctx):
    n, W, H, p = FULL["c2"]
    s = B.synthetic_scene(1, n, W, H)
    return s, P.DeviceModel.from_host(model_from_scene(s), ctx)


def test_fullsize_c2_binning_bitexact(c2):
    s, dm = c2
    n, W, H, p = FULL["c2"]
    got, orig = dm.stage_prepare(1)
    ref = B.prepare(s, 1)
    assert np.array_equal(orig, ref["orig"])
    for i, k in enumerate(B.PREP_FIELDS):
        assert np.array_equal(got[i], ref[k]), k
    off, items = dm.stage_tile_lists(1, W, H)
    roff, ritems = B.tile_grid(s, 1, W, H)
    assert np.array_equal(off, roff) and np.array_equal(items, ritems)


def test_fullsize_c3_tile_counts_bitexact(P, ctx):
    n, W, H, p = FULL["c3"]
    s = B.synthetic_scene(1, n, W, H)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    off, items = dm.stage_tile_lists(2, W, H)
    roff, ritems = B.tile_grid(s, 2, W, H)
    assert np.array_equal(off, roff)
    assert np.array_equal(items, ritems)


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not present")
def test_fullsize_c2_render_backward_vs_reference(c2):
    """C2 at full size against the unmodified reference (CR build, all host threads)."""
    s, dm = c2
    n, W, H, p = FULL["c2"]
    import paper_2412_13547_b200 as P
    pat = P.DilationPattern(1, 0, 0, W, H)
    out = dm.render(pat)
    rgb, T, ops, _ = B.render(s, 1, 0, 0, W, H, impl="ref_cr", threads=os.cpu_count())
    d = np.abs(out.colors - rgb).max(1)
    assert (d > 1e-5).mean() <= 1e-4 and d.max() <= 2e-3
    assert abs(out.blend_op_count - ops) <= 1e-5 * ops
    dl = (np.random.default_rng(0).normal(size=rgb.shape) * 1e-7).astype(np.float32)
    g = dm.backward(pat, (0, 0, 0), dl).rows()
    s2 = s.copy()
    gr, _ = B.backward(s2, 1, 0, 0, W, H, dl, impl="ref_cr", threads=os.cpu_count())
    for q in range(9):
        scale = np.abs(gr[q]).max()
        assert frac_close(g[q], gr[q], 1e-3, 1e-5 * scale) >= 0.999, q


def test_fullsize_restriction_property(P, c2):
    """SPEC.md:221 / acceptance #2: with the same low-pass p, dilated values equal the dense
    render at the active pixels — bit-exactly (per-pixel arithmetic is independent of p)."""
    s, dm = c2
    n, W, H, _ = FULL["c2"]
    dense = dm.render(P.DilationPattern(1, 0, 0, W, H), opts=P.RenderOptions(lowpass_p=2))
    img = dense.colors.reshape(H, W, 3)
    for ox, oy in ((0, 0), (1, 1)):
        pat = P.DilationPattern(2, ox, oy, W, H)
        d = dm.render(pat)  # lowpass = pattern p = 2
        xs, ys = pat.active_pixels()
        assert np.array_equal(d.colors, img[ys, xs])


def test_fullsize_determinism_and_linearity(P, c2):
    """The backward has no atomics: two runs are bit-identical. Gradients are linear in dL/dC."""
    s, dm = c2
    n, W, H, p = FULL["c2"]
    pat = P.DilationPattern(1, 0, 0, W, H)
    rng = np.random.default_rng(1)
    a = (rng.normal(size=(pat.active_count(), 3)) * 1e-7).astype(np.float32)
    b = (rng.normal(size=(pat.active_count(), 3)) * 1e-7).astype(np.float32)
    ga = dm.backward(pat, (0, 0, 0), a, update_stats=False).rows()
    ga2 = dm.backward(pat, (0, 0, 0), a, update_stats=False).rows()
    assert np.array_equal(ga, ga2)
    gb = dm.backward(pat, (0, 0, 0), b, update_stats=False).rows()
    gab = dm.backward(pat, (0, 0, 0), a + b, update_stats=False).rows()
    for q in range(9):
        scale = np.abs(gab[q]).max()
        assert frac_close(gab[q], ga[q] + gb[q], 1e-4, 1e-6 * scale) >= 0.999


def test_fullsize_conservation(P, ctx):
    """sum of blend weights + T = 1: with colour ~c everywhere and background 1,
    C = c (1 - T) + T."""
    n, W, H, p = FULL["c2"]
    s = B.synthetic_scene(3, n, W, H)
    s.cr[:] = s.cg[:] = s.cb[:] = 12.0
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    out = dm.render(P.DilationPattern(1, 0, 0, W, H), (1.0, 1.0, 1.0))
    c = np.float32(1.0) / (np.float32(1.0) + np.float32(np.exp(-12.0)))
    T = out.final_transmittance.astype(np.float64)
    assert np.abs(out.colors[:, 0] - (c * (1 - T) + T)).max() <= 2e-6


def test_fullsize_c3_fit_step_runs(P, ctx):
    """C3 (3M Gaussians, 4K, dilated p=2 with cycled offsets): fused steps run and lower the
    loss against the seed-2 target."""
    n, W, H, p = FULL["c3"]
    dm = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, n, W, H), ctx)
    tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(2, n, W, H), ctx)
    target = tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3)
    tm.close()
    diag = math.hypot(W, H)
    losses = []
    for it in range(8):
        ox, oy = P.next_offsets(2, it)
        losses.append(dm.fit_step(P.DilationPattern(2, ox, oy, W, H), (0, 0, 0), target, it + 1, 1000, diag))
    assert all(np.isfinite(losses)) and np.mean(losses[4:]) < np.mean(losses[:4])


@pytest.mark.parametrize("p,ox,oy", [(2, 1, 1), (3, 2, 2), (3, 0, 1)])
def test_dilated_host_target_stages_active_rows(P, ctx, p, ox, oy):
    """A host target of a dilated view is staged as its active rows only (1/p of the image over
    PCIe); the fused step must equal the same step with the full device-resident target, bit for
    bit (odd heights: the last active row)."""
    import torch
    W, H, n = 70, 53, 800
    s = B.synthetic_scene(3, n, W, H).ensure_stats()
    target = target_image(4, n, W, H)
    pat = P.DilationPattern(p, ox, oy, W, H)
    diag = math.hypot(W, H)
    a = P.DeviceModel.from_host(model_from_scene(s), ctx)
    b = P.DeviceModel.from_host(model_from_scene(s), ctx)
    la = a.fit_step(pat, (0, 0, 0), np.ascontiguousarray(target), 1, 100, diag)   # host: rows only
    dev = torch.from_numpy(np.ascontiguousarray(target)).cuda()
    torch.cuda.synchronize()
    lb = b.fit_step(pat, (0, 0, 0), dev.data_ptr(), 1, 100, diag)                # device: full image
    assert la == lb
    ha, hb = a.download(), b.download()
    assert np.array_equal(ha.params.view(np.uint32), hb.params.view(np.uint32))
