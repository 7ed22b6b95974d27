"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded
inputs (SURVEY.md §8c parity definition).

Bit-exact: prepared splats, blend order, tile counts, per-tile lists, Adam given equal
gradients, chain rule given equal screen-space sums, densify/prune selections given equal
statistics. Within stated FP32 tolerance: colours / transmittance / gradients (the blend uses
a fast exp2 and FMA; the backward recovers T by division), with the few pixels whose
termination test sits at T == 1e-4 reported explicitly.
"""
import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import frac_close, model_from_scene, render_check, scene_from_model, target_image

pytestmark = pytest.mark.gpu

# colour / transmittance tolerance (abs) for all but threshold pixels
RGB_ATOL = 1e-5
# gradient tolerance: |gpu - ref| <= GRAD_RTOL |ref| + GRAD_ATOL_REL * max|ref| per component
GRAD_RTOL = 1e-3
GRAD_ATOL_REL = 1e-5


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


def make(P, ctx, seed, n, W, H):
    s = B.synthetic_scene(seed, n, W, H)
    m = model_from_scene(s)
    dm = P.DeviceModel.from_host(m, ctx)
    return s, m, dm


@pytest.mark.parametrize("lowpass", [1, 2, 3])
def test_prepare_bitexact(P, ctx, lowpass):
    s, m, dm = make(P, ctx, 1, 10000, 256, 256)
    got, orig = dm.stage_prepare(lowpass)
    ref = B.prepare(s, lowpass)
    assert np.array_equal(orig, ref["orig"])
    for i, k in enumerate(B.PREP_FIELDS):
        assert np.array_equal(got[i].view(np.uint32), ref[k].view(np.uint32)), k


def test_sorted_order_ties_and_ids(P, ctx):
    s = B.synthetic_scene(3, 5000, 128, 128)
    # quantised depths create many ties; shuffled non-monotone ids exercise the id pre-sort
    s.depth = np.round(s.depth * 16).astype(np.float32) / 16
    s.depth[::7] = -0.0
    rng = np.random.default_rng(0)
    s.id = rng.permutation(np.arange(10, 10 + s.n)).astype(np.uint64)
    m = model_from_scene(s)
    dm = P.DeviceModel.from_host(m, ctx)
    assert np.array_equal(dm.stage_sorted_order(), B.sorted_order(s))
    if B.ref_available():
        assert np.array_equal(dm.stage_sorted_order(), B.sorted_order(s, impl="ref_cr"))


@pytest.mark.parametrize("W,H,n,lowpass", [(256, 256, 10000, 1), (250, 170, 3000, 2),
                                           (33, 17, 50, 1), (1920, 1080, 50000, 1)])
def test_tile_lists_bitexact(P, ctx, W, H, n, lowpass):
    s, m, dm = make(P, ctx, 5, n, W, H)
    off, items = dm.stage_tile_lists(lowpass, W, H)
    roff, ritems = B.tile_grid(s, lowpass, W, H)
    assert np.array_equal(off, roff)
    assert np.array_equal(items, ritems)


def test_tile_lists_long_list_fallback(P, ctx):
    """A tile list longer than the per-tile warp sort (kSegCap = 1024) takes the
    onesweep radix-sort path; the lists must still equal the reference's."""
    W, H, n = 64, 64, 6000
    s = B.synthetic_scene(11, n, W, H)
    rng = np.random.default_rng(1)
    s.px[:] = (8.0 + rng.uniform(-2, 2, n)).astype(np.float32)
    s.py[:] = (8.0 + rng.uniform(-2, 2, n)).astype(np.float32)
    s.lsx[:] = np.float32(0.0)
    s.lsy[:] = np.float32(0.0)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    off, items = dm.stage_tile_lists(1, W, H)
    roff, ritems = B.tile_grid(s, 1, W, H)
    assert np.diff(roff.astype(np.int64)).max() > 1024
    assert np.array_equal(off, roff)
    assert np.array_equal(items, ritems)


def test_tile_lists_forced_onesweep():
    """TGSX_BINNING=onesweep forces the radix-sort binning for every view: same lists."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, paper_2412_13547_b200 as P\n"
        "from oracle import bind as B\n"
        "from tests.helpers import model_from_scene\n"
        "B.set_math(True)\n"
        "s = B.synthetic_scene(5, 20000, 400, 300)\n"
        "dm = P.DeviceModel.from_host(model_from_scene(s), P.Context(0))\n"
        "off, items = dm.stage_tile_lists(1, 400, 300)\n"
        "roff, ritems = B.tile_grid(s, 1, 400, 300)\n"
        "assert np.array_equal(off, roff) and np.array_equal(items, ritems)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, TGSX_BINNING="onesweep")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def _render_check(got, ref, label=""):
    """Colours / T within RGB_ATOL except threshold pixels, each with |T - 1e-4| evidence
    (tests/helpers.render_check)."""
    rrgb, rT, rops, _ = ref
    return render_check(got.colors, got.final_transmittance, got.blend_op_count, rrgb, rT, rops,
                        RGB_ATOL, label)


@pytest.mark.parametrize("p,ox,oy", [(1, 0, 0), (2, 0, 0), (2, 1, 1), (3, 2, 1), (4, 3, 0)])
def test_render_matches_oracle(P, ctx, p, ox, oy):
    W, H, n = 256, 200, 10000
    s, m, dm = make(P, ctx, 1, n, W, H)
    pat = P.DilationPattern(p, ox, oy, W, H)
    got = dm.render(pat, (0.1, 0.2, 0.3))
    ref = B.render(s, p, ox, oy, W, H, (0.1, 0.2, 0.3))
    _render_check(got, ref, f"p={p} o=({ox},{oy})")
    c = ctx.counters()
    assert abs(c["evals"] - ref[3]) <= max(4, int(1e-5 * ref[3]))


def test_render_empty_and_offimage(P, ctx):
    W, H = 40, 30
    s = B.synthetic_scene(1, 20, W, H)
    s.px += 1000.0  # every splat off-image: nothing binned, background everywhere
    m = model_from_scene(s)
    dm = P.DeviceModel.from_host(m, ctx)
    out = dm.render(P.DilationPattern(1, 0, 0, W, H), (0.25, 0.5, 0.75))
    assert np.all(out.colors == np.float32([0.25, 0.5, 0.75])) and np.all(out.final_transmittance == 1)
    assert out.blend_op_count == 0
    empty = P.DeviceModel.from_host(P.GaussianModel(0), ctx)
    out = empty.render(P.DilationPattern(2, 1, 0, W, H), (0.0, 0.0, 0.0))
    assert out.colors.shape == (20 * 15, 3) and np.all(out.colors == 0)


def _grad_check(g, r, label):
    for q in range(9):
        a, b = g[q], r[q]
        scale = np.abs(b).max(initial=0.0)
        fr = frac_close(a, b, GRAD_RTOL, GRAD_ATOL_REL * scale)
        assert fr >= 0.999, f"{label} comp {q}: only {fr:.5f} within tol"
        assert frac_close(a, b, 2e-2, 1e-3 * scale) == 1.0, f"{label} comp {q}: outlier"


@pytest.mark.parametrize("p,ox,oy", [(1, 0, 0), (2, 1, 0), (3, 0, 2)])
def test_backward_matches_oracle(P, ctx, p, ox, oy):
    W, H, n = 256, 256, 10000
    s, m, dm = make(P, ctx, 1, n, W, H)
    pat = P.DilationPattern(p, ox, oy, W, H)
    rng = np.random.default_rng(7)
    dl = rng.normal(size=(pat.active_count(), 3)).astype(np.float32) * 1e-4
    dl[::13] = 0.0  # skipped pixels (rasterizer.cpp:265) still record visits
    gs = dm.backward(pat, (0.0, 0.0, 0.0), dl)
    ref, scr = B.backward(s, p, ox, oy, W, H, dl, screen=True)
    _grad_check(gs.rows(), ref, f"p={p}")
    sg = dm.screen_grads()
    vis_gpu = sg[9] > 0
    vis_ref = scr["maxw"] > np.float32(1e-4)
    mism = np.nonzero(vis_gpu != vis_ref)[0]
    # visited is exact except where max blend weight sits at the 1e-4 floor
    assert np.all(np.abs(scr["maxw"][mism] - 1e-4) <= 1e-8), mism[:10]
    hm = dm.download()
    assert np.array_equal(hm.visit_count, s.visit) or len(mism) > 0


def test_chain_rule_bitexact_given_screen_sums(P, ctx):
    """With the screen-space sums from the GPU itself, the chain rule + stats reproduce the
    oracle's formula bit for bit (rasterizer.cpp:321-359)."""
    W, H, n = 128, 128, 3000
    s, m, dm = make(P, ctx, 4, n, W, H)
    pat = P.DilationPattern(1, 0, 0, W, H)
    dl = np.random.default_rng(1).normal(size=(pat.active_count(), 3)).astype(np.float32)
    gs = dm.backward(pat, (0, 0, 0), dl).rows()
    sg = dm.screen_grads().astype(np.float32)
    # restate the chain rule in float32 numpy with the oracle's evaluation order
    f = np.float32
    c = np.cos(m.params[2].astype(np.float64)).astype(f)
    sn = np.sin(m.params[2].astype(np.float64)).astype(f)
    a = np.exp((f(2) * m.params[3]).astype(np.float64)).astype(f)
    b = np.exp((f(2) * m.params[4]).astype(np.float64)).astype(f)
    m00, m01, m11 = sg[2], sg[3], sg[4]
    cs = c * sn
    amb = a - b
    rot = m00 * (f(-2) * cs * amb) + f(2) * m01 * ((c * c - sn * sn) * amb) + m11 * (f(2) * cs * amb)
    assert np.array_equal(gs[2], rot)
    lsx = f(2) * a * (m00 * c * c + f(2) * m01 * cs + m11 * sn * sn)
    assert np.array_equal(gs[3], lsx)
    assert np.array_equal(gs[0], sg[0]) and np.array_equal(gs[1], sg[1])


def test_adam_bitexact(P, ctx):
    W, H, n = 64, 64, 4000
    s, m, dm = make(P, ctx, 2, n, W, H)
    rng = np.random.default_rng(3)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)
    diag = float(np.sqrt(W * W + H * H))
    for t in range(1, 4):
        g = (rng.normal(size=(9, n)) * 10 ** rng.uniform(-6, 0, size=(9, n))).astype(np.float32)
        g[:, ::17] = 0.0
        dm.adam_step(g, t, 100, diag)
        cfg = B.adam_config(t, 100, diag)
        B.adam_step(s, g, m1, m2, cfg)
    h = dm.download()
    for i, f in enumerate(("px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb")):
        assert np.array_equal(h.params[i].view(np.uint32), getattr(s, f).view(np.uint32)), f
    d1, d2 = dm.moments()
    assert np.array_equal(d1, m1) and np.array_equal(d2, m2)


def test_fit_step_matches_oracle_sequence(P, ctx):
    """One fused fit step == render + L1 + backward + Adam (oracle), within tolerance."""
    W, H, n = 128, 96, 2000
    s, m, dm = make(P, ctx, 1, n, W, H)
    target = target_image(2, n, W, H)
    pat = P.DilationPattern(1, 0, 0, W, H)
    diag = float(np.sqrt(W * W + H * H))
    loss = dm.fit_step(pat, (0, 0, 0), target, 1, 100, diag)
    rgb, T, _, _ = B.render(s, 1, 0, 0, W, H)
    rloss, dl = B.l1_loss(rgb, 1, 0, 0, W, H, target)
    assert abs(loss - rloss) <= 1e-5 * rloss
    g, _ = B.backward(s, 1, 0, 0, W, H, dl)
    m1 = np.zeros((9, n), np.float32)
    m2 = np.zeros((9, n), np.float32)
    B.adam_step(s, g, m1, m2, B.adam_config(1, 100, diag))
    h = dm.download()
    # first Adam step moves every touched parameter by ~lr*sign(g): compare the moved params
    for i, f in enumerate(("px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb")):
        a, b = h.params[i], getattr(s, f)
        assert frac_close(a, b, 1e-6, 1e-6) >= 0.995, f


@pytest.mark.parametrize("n,bits", [(1, 8), (1000, 13), (100003, 15), (2_000_000, 32), (4096 * 3, 7)])
def test_sort_pairs_stable(P, ctx, n, bits):
    import ctypes as C
    import torch
    rng = np.random.default_rng(n)
    keys = rng.integers(0, 1 << bits, size=n, dtype=np.uint64).astype(np.uint32)
    vals = np.arange(n, dtype=np.uint32)
    dk = torch.from_numpy(keys.view(np.int32)).cuda()
    dv = torch.from_numpy(vals.view(np.int32)).cuda()
    torch.cuda.synchronize()
    ctx.check(ctx.L.tgsx_sort_pairs(ctx.h, C.c_void_p(dk.data_ptr()), C.c_void_p(dv.data_ptr()), n, bits))
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(dk.cpu().numpy().view(np.uint32), keys[order])
    assert np.array_equal(dv.cpu().numpy().view(np.uint32), vals[order])


@pytest.mark.parametrize("n", [0, 1, 7, 2048, 2049, 1_000_003])
def test_exclusive_scan(P, ctx, n):
    import ctypes as C
    import torch
    rng = np.random.default_rng(n)
    x = rng.integers(0, 40, size=max(n, 1), dtype=np.uint32)[:n]
    dx = torch.from_numpy(x.view(np.int32)).cuda() if n else torch.zeros(1, dtype=torch.int32, device="cuda")
    dy = torch.zeros_like(dx)
    tot = C.c_uint64()
    ctx.check(ctx.L.tgsx_exclusive_scan(ctx.h, C.c_void_p(dx.data_ptr()), C.c_void_p(dy.data_ptr()), n, C.byref(tot)))
    ex = np.concatenate([[0], np.cumsum(x, dtype=np.uint64)[:-1]]).astype(np.uint32) if n else x
    assert np.array_equal(dy.cpu().numpy().view(np.uint32)[:n], ex)
    assert tot.value == int(x.sum())


def test_errors_mirror_reference(P, ctx):
    W, H = 32, 32
    s = B.synthetic_scene(1, 50, W, H)
    s.rot[10] = np.nan
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    with pytest.raises(ValueError):   # std::invalid_argument (gaussian.hpp:64-68)
        dm.render(P.DilationPattern(1, 0, 0, W, H))
    s = B.synthetic_scene(1, 50, W, H)
    s.lsx[3] = -60.0
    s.lsy[3] = 60.0  # det overflows to inf -> runtime_error (gaussian.hpp:84-86)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    with pytest.raises(RuntimeError):
        dm.render(P.DilationPattern(1, 0, 0, W, H))
    dm = P.DeviceModel.from_host(model_from_scene(B.synthetic_scene(1, 50, W, H)), ctx)
    with pytest.raises(ValueError):
        dm.backward(P.DilationPattern(1, 0, 0, W, H), (0, 0, 0), np.zeros((5, 3), np.float32))
    with pytest.raises(ValueError):
        P.DilationPattern(2, 2, 0, W, H)


def test_binning_stress_random_shapes(P):
    """Random sizes / patterns / id orders with several live contexts: tile lists bit-exact vs the
    oracle on every iteration (tests/stress_binning.py)."""
    from tests import stress_binning
    assert stress_binning.main(60) == 0


def test_tile_lists_across_claim_order_refresh_and_densify(P, ctx):
    """The slab claims run in a spatial order of the blend ranks (raster.cu launch_claims) that
    is rebuilt after every depth sort and every 64 binnings while the splats move. Any order must
    give the reference's lists: checked after 70 fit steps (one refresh on moved splats), after a
    densify event (new ranks) and after the next fit steps."""
    from tests.helpers import scene_from_model
    B.set_math(True)
    W, H, n = 400, 300, 20000
    s = B.synthetic_scene(21, n, W, H)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    tgt = np.full((H, W, 3), 0.4, np.float32)
    diag = float(np.hypot(W, H))

    def check():
        host = scene_from_model(dm.download())
        off, items = dm.stage_tile_lists(1, W, H)
        roff, ritems = B.tile_grid(host, 1, W, H)
        assert np.array_equal(off, roff) and np.array_equal(items, ritems)

    for t in range(70):
        dm.fit_step(P.DilationPattern(1, 0, 0, W, H), (0.0, 0.0, 0.0), tgt, t + 1, 1000, diag)
    check()
    st = np.array(B.Pcg32(3, 1).state, np.uint64)
    rep = dm.densify(n + 2000, st, P.densify_config(tau_pos=1e-9))
    assert rep.spawned > 0
    check()
    for t in range(5):
        dm.fit_step(P.DilationPattern(2, t % 2, 0, W, H), (0.0, 0.0, 0.0), tgt, 71 + t, 1000, diag)
    check()
