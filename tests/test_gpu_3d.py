"""GPU parity of the 3-D front end against the FP64 oracle
(oracle/ewa3d.c, pinned by formula KATs, finite differences and the reference's 2-D render in
tests/test_oracle3d.py). Everything behind the 2-D record is the 2-D path's kernels.

Tolerances (written here, FP32 on the GPU vs FP64 projection in the oracle):
  records            |gpu - ref| <= 2e-5 |ref| + 2e-5 (means, inverse covariance, alpha, colour)
  blend order        identical except adjacent swaps of rows whose depths agree to 1e-6
  colours / T        <= 1e-4 abs on >= 99.9 % of pixels (box-test / order flips at float ties)
  gradients          per Gaussian, |gpu - ref| <= 2e-3 max|ref| on >= 99.5 % of Gaussians
  chain rule only    (oracle chain on the GPU's own screen sums) <= 1e-3 max|ref| per Gaussian
  Adam               bit-exact given equal gradients
"""
import numpy as np
import pytest

from oracle import bind as B

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def S():
    from paper_2412_13547_b200 import scene3d as S
    return S


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def camera(S, W=256, H=192):
    return S.Camera.look_at((0.3, -0.2, -0.5), (0.0, 0.0, 4.5), (0, -1, 0), 60.0, W, H)


def scene(S, ctx, seed=1, n=6000, W=256, H=192):
    cam = camera(S, W, H)
    m = S.GaussianModel3D.synthetic(seed, n, cam)
    dm = S.DeviceModel3D.from_host(m, ctx)
    return cam, m, dm


@pytest.mark.parametrize("lowpass", [1, 2])
def test_records_and_blend_order(S, ctx, lowpass):
    cam, m, dm = scene(S, ctx)
    got = dm.stage_prepare(cam, lowpass)
    ref = B.prepare3d(m.params, cam, lowpass)
    assert len(got["orig"]) == len(ref["orig"]) == m.size()
    mism = np.nonzero(got["orig"] != ref["orig"])[0]
    # the only allowed differences: neighbours whose depths agree to float rounding
    for i in mism:
        assert abs(float(ref["depth"][i]) - float(got["depth"][i])) <= 1e-6 * abs(float(ref["depth"][i]))
    assert len(mism) <= 0.01 * m.size()
    gi = np.argsort(got["orig"])
    ri = np.argsort(ref["orig"])
    for k in ("mx", "my", "i00", "i01", "i11", "alpha", "c0", "c1", "c2", "rx", "ry"):
        a, b = got[k][gi], ref[k][ri]
        np.testing.assert_allclose(a, b, rtol=2e-5, atol=2e-5 * float(np.abs(b).max()), err_msg=k)


def test_culling_behind_camera(S, ctx):
    cam = camera(S, 64, 48)
    m = S.GaussianModel3D.synthetic(2, 300, cam)
    p = m.params.copy()
    # move 50 Gaussians behind the camera centre
    fwd = np.asarray(cam.R)[2]
    p[0:3, :50] = (cam.center[:, None] - 2.0 * fwd[:, None]).astype(np.float32)
    dm = S.DeviceModel3D.from_host(S.GaussianModel3D(p), ctx)
    rec = dm.stage_prepare(cam, 1)
    assert len(rec["orig"]) == 250 and rec["orig"].min() >= 50
    dl = np.random.default_rng(0).normal(size=(cam.width * cam.height, 3)).astype(np.float32)
    g = dm.backward(cam, None, (0, 0, 0), dl)
    assert np.all(g[:, :50] == 0)


@pytest.mark.parametrize("p,ox,oy", [(1, 0, 0), (2, 1, 0)])
def test_render_parity(S, ctx, p, ox, oy):
    cam, m, dm = scene(S, ctx, seed=3)
    pat = cam.pattern(p, ox, oy)
    out = dm.render(cam, pat, (0.1, 0.2, 0.3))
    rgb, T, ops, _ = B.render3d(m.params, cam, p, ox, oy, (0.1, 0.2, 0.3))
    err = np.abs(out.colors - rgb).max(axis=1)
    assert np.mean(err <= 1e-4) >= 0.999, float(err.max())
    assert np.mean(np.abs(out.final_transmittance - T) <= 1e-4) >= 0.999
    assert abs(int(out.blend_op_count) - int(ops)) <= 1e-4 * ops


def test_backward_parity(S, ctx):
    cam, m, dm = scene(S, ctx, seed=4)
    pat = cam.pattern(1)
    dl = np.random.default_rng(1).normal(size=(pat.active_count(), 3)).astype(np.float32) * 1e-3
    g, scr = dm.backward(cam, pat, (0, 0, 0), dl, screen=True)
    gr, sr, touched = B.backward3d(m.params, cam, 1, 0, 0, dl)
    # visited set: identical except Gaussians at the visibility threshold
    vis_g = scr[9] > 0
    assert np.mean(vis_g == touched) >= 0.999
    # full-path gradients
    scale = np.abs(gr).max(axis=0) + 1e-30
    ok = np.all(np.abs(g - gr) <= 2e-3 * scale, axis=0)
    assert np.mean(ok[touched]) >= 0.995, np.mean(ok[touched])
    # chain rule alone: the oracle's FP64 chain on the GPU's own screen sums
    bump = 0.3
    idx = np.nonzero(vis_g)[0][:400]
    for i in idx:
        want = B.chain3d(m.params[:, i].astype(np.float64), cam, bump, scr[:9, i].astype(np.float64))
        s = np.abs(want).max() + 1e-30
        np.testing.assert_allclose(g[:, i], want, rtol=0, atol=1e-3 * s, err_msg=f"row {i}")


def test_adam3d_bitexact(S, ctx):
    cam, m, dm = scene(S, ctx, seed=5, n=2000)
    rng = np.random.default_rng(2)
    p = m.params.copy()
    mom1 = np.zeros_like(p)
    mom2 = np.zeros_like(p)
    for step in (1, 2, 3):
        g = (rng.normal(size=p.shape) * 10.0 ** rng.uniform(-6, 0, size=p.shape)).astype(np.float32)
        dm.adam_step(g, step, 100, 3.0)
        B.adam3d_step(p, g, mom1, mom2, B.adam3d_config(step, 100, 3.0))
    got = dm.download().params
    assert np.array_equal(got.view(np.uint32), p.view(np.uint32))
    m1, m2 = dm.moments()
    assert np.array_equal(m1.view(np.uint32), mom1.view(np.uint32))
    assert np.array_equal(m2.view(np.uint32), mom2.view(np.uint32))


def test_fit_step_equals_backward_plus_adam(S, ctx):
    """One fused fit step == render -> host L1 gradient -> backward3d -> Adam (bit-exact: every
    stage is deterministic, no atomics in the gradient path)."""
    cam, m, dm = scene(S, ctx, seed=6, n=3000, W=128, H=96)
    tgt = np.random.default_rng(3).uniform(0, 1, (cam.height, cam.width, 3)).astype(np.float32)
    pat = cam.pattern(1)
    c = dm.render(cam, pat).colors.reshape(cam.height, cam.width, 3)
    sc = np.float32(1.0 / (3.0 * pat.active_count()))
    d = c - tgt
    dl = (np.sign(d) * sc).astype(np.float32).reshape(-1, 3)
    g = dm.backward(cam, pat, (0, 0, 0), dl, update_stats=False)
    dm2 = S.DeviceModel3D.from_host(m, ctx)
    loss = dm2.fit_step(cam, pat, (0, 0, 0), tgt, 1, 100, 3.0)
    assert loss == pytest.approx(float(np.abs(d).mean()), rel=1e-4)
    dm.adam_step(g, 1, 100, 3.0)
    assert np.array_equal(dm.download().params.view(np.uint32), dm2.download().params.view(np.uint32))
    pos, col, vis = dm2.stats()
    assert vis.max() == 1 and np.count_nonzero(vis) > 0.5 * m.size()


def test_fit_converges_to_target(S, ctx):
    """Fitting a perturbed copy of a scene to renders of the original lowers the loss."""
    cam, m, dm_true = scene(S, ctx, seed=7, n=4000, W=128, H=96)
    tgt = dm_true.render(cam).colors.reshape(cam.height, cam.width, 3).copy()
    p = m.params.copy()
    rng = np.random.default_rng(4)
    p[11:14] += rng.normal(0, 0.3, (3, p.shape[1])).astype(np.float32)
    p[0:3] += rng.normal(0, 0.003, (3, p.shape[1])).astype(np.float32)
    dm = S.DeviceModel3D.from_host(S.GaussianModel3D(p), ctx)
    losses = [dm.fit_step(cam, None, (0, 0, 0), tgt, it, 200, 3.0) for it in range(1, 61)]
    assert losses[-1] < 0.5 * losses[0], (losses[0], losses[-1])


def test_errors(S, ctx):
    cam, m, dm = scene(S, ctx, seed=8, n=100, W=64, H=48)
    with pytest.raises(ValueError):
        dm.render(cam, S.Camera(cam.R, cam.t, cam.fx, cam.fy, cam.cx, cam.cy, 32, 48).pattern())
    p = m.params.copy()
    p[20, 5] = np.nan
    bad = S.DeviceModel3D.from_host(S.GaussianModel3D(p), ctx)
    with pytest.raises(ValueError):
        bad.render(cam)
    p = m.params.copy()
    p[3:7, 9] = 0
    bad = S.DeviceModel3D.from_host(S.GaussianModel3D(p), ctx)
    with pytest.raises(ValueError):
        bad.render(cam)
    bad_cam = S.Camera(cam.R, cam.t, -1.0, cam.fy, cam.cx, cam.cy, 64, 48)
    with pytest.raises(ValueError):
        dm.render(bad_cam)


def test_batched_views_equal_mean_of_per_view_gradients(S, ctx):
    """Batched multi-camera step (view_accumulate3d x V + apply_step3d, driven through
    dist.ViewShardedFit as one rank) == the mean of the per-view backward3d gradients (summed in
    view order) followed by the oracle's Adam: bit-exact; statistics = summed increments."""
    from paper_2412_13547_b200 import dist as D
    W, H = 96, 72
    cams = [S.Camera.look_at((0.4 * np.cos(a), 0.3 * np.sin(a), -0.5), (0.0, 0.0, 4.5), (0, -1, 0), 60.0, W, H)
            for a in np.linspace(0, 2 * np.pi, 4, endpoint=False)]
    m = S.GaussianModel3D.synthetic(9, 3000, cams[0])
    rng = np.random.default_rng(5)
    targets = [rng.uniform(0, 1, (H, W, 3)).astype(np.float32) for _ in cams]
    ref = S.DeviceModel3D.from_host(m, ctx)
    total = np.zeros((59, m.size()), np.float32)
    visits = np.zeros(m.size(), np.int64)
    for cam, tgt in zip(cams, targets):
        pat = cam.pattern(1)
        c = ref.render(cam, pat).colors.reshape(H, W, 3)
        dl = (np.sign(c - tgt) * np.float32(1.0 / (3.0 * pat.active_count()))).astype(np.float32).reshape(-1, 3)
        g, scr = ref.backward(cam, pat, (0, 0, 0), dl, update_stats=False, screen=True)
        total = (total + g).astype(np.float32)
        visits += scr[9] > 0
    mean = (total / np.float32(len(cams))).astype(np.float32)
    p = m.params.copy()
    mom1, mom2 = np.zeros_like(p), np.zeros_like(p)
    B.adam3d_step(p, mean, mom1, mom2, B.adam3d_config(1, 100, 3.0))
    dm = S.DeviceModel3D.from_host(m, ctx)
    fit = D.ViewShardedFit(dm, 0, 1)
    losses = fit.step([(cam, cam.pattern(1), t) for cam, t in zip(cams, targets)], (0, 0, 0), 1, 100, 3.0)
    assert len(losses) == 4 and all(np.isfinite(losses))
    assert np.array_equal(dm.download().params.view(np.uint32), p.view(np.uint32))
    _, _, vis = dm.stats()
    assert np.array_equal(vis, visits)
    ptr, count = dm.step_buffer()
    assert ptr != 0 and count % D.STEP3D_ROWS == 0 and count // D.STEP3D_ROWS >= m.size()
