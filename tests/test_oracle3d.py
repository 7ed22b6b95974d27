"""Pins the 3-D front-end oracle (oracle/ewa3d.c).

The reference has no 3-D code, tests or vectors, so parity is unpinned at the reference for this
row. The FP64 restatement is pinned instead by
  * known-answer values that follow from the formulas (SH basis on the axes, on-axis / off-axis
    EWA projection, near-plane culling),
  * central finite differences of or3d_project against or3d_chain (the check the reference's own
    FP64 instantiation exists for), including the clamped-Jacobian and
    clamped-colour branches,
  * equivalence with the reference's compiled 2-D render (oracle/_ref) for 3-D Gaussians at the
    principal point, whose EWA projection is exactly a 2-D Gaussian of the reference's model.
"""
import math

import numpy as np
import pytest

from oracle import bind as B
from paper_2412_13547_b200.scene3d import Camera, GaussianModel3D

C0 = 0.28209479177387814
C1 = 0.4886025119029199


def cam_identity(W=100, H=100, f=100.0):
    return Camera(np.eye(3), np.zeros(3), f, f, W / 2, H / 2, W, H, 0.2)


def theta(mu=(0, 0, 5), q=(1, 0, 0, 0), ls=(math.log(0.1),) * 3, rop=0.0, sh=None):
    t = np.zeros(59)
    t[0:3] = mu
    t[3:7] = q
    t[7:10] = ls
    t[10] = rop
    if sh is not None:
        t[11:] = np.asarray(sh, np.float64).reshape(48)
    return t


def random_rotation(rng):
    q = rng.normal(size=4)
    q /= np.linalg.norm(q)
    w, x, y, z = q
    return np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                     [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                     [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])


def test_sh_basis_known_answers():
    b, _ = B.sh_basis((0.0, 0.0, 1.0))
    want = np.zeros(16)
    want[0] = C0
    want[2] = C1
    want[6] = 2 * 0.31539156525252005
    want[12] = 2 * 0.3731763325901154
    np.testing.assert_allclose(b, want, rtol=0, atol=1e-15)
    b, _ = B.sh_basis((1.0, 0.0, 0.0))
    assert b[3] == pytest.approx(-C1)
    assert b[8] == pytest.approx(0.5462742152960396)
    assert b[15] == pytest.approx(-0.5900435899266435)


def test_sh_basis_gradient_fd():
    rng = np.random.default_rng(3)
    for _ in range(20):
        d = rng.normal(size=3)
        _, db = B.sh_basis(d)
        for j in range(3):
            e = np.zeros(3)
            e[j] = 1e-6
            fd = (B.sh_basis(d + e)[0] - B.sh_basis(d - e)[0]) / 2e-6
            np.testing.assert_allclose(db[:, j], fd, rtol=1e-6, atol=1e-8)


def test_projection_on_axis():
    cam = cam_identity()
    sh = np.zeros((16, 3))
    sh[0] = 1.0
    rc, o = B.project3d(theta(sh=sh, rop=0.5), cam, 0.3)
    assert rc == 1
    # u = fx x/z + cx, Σ2 = (f/z)^2 s^2 I = 400 * 0.01 = 4, plus the low-pass bump 0.3
    np.testing.assert_allclose(o[:5], [50, 50, 4.3, 0.0, 4.3], rtol=1e-12, atol=1e-12)
    assert o[5] == pytest.approx(1 / (1 + math.exp(-0.5)), rel=1e-14)
    np.testing.assert_allclose(o[6:9], 0.5 + C0, rtol=1e-14)
    assert o[9] == pytest.approx(5.0)
    np.testing.assert_allclose(o[10:12], 3 * math.sqrt(4.3), rtol=1e-14)


def test_projection_off_axis_and_clamp():
    cam = cam_identity()
    # x/z = 0.2 inside the 1.3 tan(fov/2) = 0.65 clamp: J02 = -fx x / z^2 = -4
    rc, o = B.project3d(theta(mu=(1, 0, 5)), cam, 0.3)
    assert rc == 1
    assert o[0] == pytest.approx(70.0)
    assert o[2] == pytest.approx(0.01 * (400 + 16) + 0.3, rel=1e-12)
    # x/z = 1.0 beyond the clamp: the Jacobian uses x/z = 0.65 (J02 = -fx 0.65 / z = -13)
    rc, o = B.project3d(theta(mu=(5, 0, 5)), cam, 0.3)
    assert rc == 1
    assert o[0] == pytest.approx(150.0)
    assert o[2] == pytest.approx(0.01 * (400 + 169) + 0.3, rel=1e-12)


def test_near_plane_and_invalid():
    cam = cam_identity()
    assert B.project3d(theta(mu=(0, 0, 0.1)), cam, 0.3)[0] == 0
    assert B.project3d(theta(mu=(0, 0, -3)), cam, 0.3)[0] == 0
    t = theta()
    t[20] = np.nan
    assert B.project3d(t, cam, 0.3)[0] == -1
    assert B.project3d(theta(q=(0, 0, 0, 0)), cam, 0.3)[0] == -1


def _objective(th, cam, bump, w):
    rc, o = B.project3d(th, cam, bump)
    assert rc == 1
    # the screen sums' symmetric convention: dL = m00 dS00 + 2 m01 dS01 + m11 dS11
    return (w[0] * o[0] + w[1] * o[1] + w[2] * o[2] + 2 * w[3] * o[3] + w[4] * o[4] + w[5] * o[5]
            + w[6] * o[6] + w[7] * o[7] + w[8] * o[8])


@pytest.mark.parametrize("case", ["generic", "clamped_x", "clamped_y", "clamped_colour", "lowpass2"])
def test_chain_matches_finite_differences(case):
    rng = np.random.default_rng({"generic": 1, "clamped_x": 2, "clamped_y": 3, "clamped_colour": 4,
                                 "lowpass2": 5}[case])
    for trial in range(8):
        R = random_rotation(rng)
        eye = rng.normal(size=3)
        cam = Camera(R, -R @ eye, 120.0, 110.0, 64.0, 48.0, 128, 96, 0.2)
        pc = np.array([rng.uniform(-0.3, 0.3), rng.uniform(-0.3, 0.3), 1.0]) * rng.uniform(2, 5)
        if case == "clamped_x":
            pc[0] = pc[2] * rng.choice([-1, 1]) * rng.uniform(0.7, 1.5)
        if case == "clamped_y":
            pc[1] = pc[2] * rng.choice([-1, 1]) * rng.uniform(0.6, 1.2)
        mu = R.T @ (pc - cam.t)
        sh = rng.uniform(-0.5, 0.5, (16, 3))
        if case == "clamped_colour":
            sh[0] = [-8.0, 0.4, -8.0]
        th = theta(mu=mu, q=rng.normal(size=4), ls=rng.uniform(-3, -1, 3), rop=rng.uniform(-2, 2), sh=sh)
        bump = 0.3 + 0.5 * (2 - 1) if case == "lowpass2" else 0.3
        w = rng.normal(size=9)
        g = B.chain3d(th, cam, bump, w)
        fd = np.zeros(59)
        for k in range(59):
            h = 1e-6 * max(1.0, abs(th[k]))
            tp, tm = th.copy(), th.copy()
            tp[k] += h
            tm[k] -= h
            fd[k] = (_objective(tp, cam, bump, w) - _objective(tm, cam, bump, w)) / (2 * h)
        scale = np.abs(fd).max()
        np.testing.assert_allclose(g, fd, rtol=2e-5, atol=2e-7 * scale, err_msg=f"{case} trial {trial}")
        if case == "clamped_colour":
            assert np.all(g[11:][0::3] == 0) and np.all(g[11:][2::3] == 0)  # r, b clamped at 0


def _principal_point_scene(rng, n, cam):
    """3-D Gaussians on the optical axis (u, v) = (cx, cy), rotated about it: their EWA
    projection is exactly the reference's 2-D Gaussian (gaussian.hpp:63-78)."""
    params = np.zeros((59, n), np.float64)
    z = rng.uniform(2, 8, n)
    params[2] = z
    rot = rng.uniform(-math.pi, math.pi, n)
    params[3] = np.cos(rot / 2)
    params[6] = np.sin(rot / 2)
    l2 = rng.uniform(0.5, 2.5, (2, n))  # 2-D log-scales in pixels
    params[7:9] = l2 + np.log(z / cam.fx)[None]
    params[9] = np.log(0.05)
    params[10] = rng.uniform(-2, 2, n)
    raw_c = rng.uniform(-2, 2, (3, n))
    params[11:14] = (1 / (1 + np.exp(-raw_c)) - 0.5) / C0
    s = B.Scene.empty(n)
    s.px[:] = cam.cx
    s.py[:] = cam.cy
    s.rot[:] = rot
    s.lsx[:], s.lsy[:] = l2
    s.rop[:] = params[10]
    s.cr[:], s.cg[:], s.cb[:] = raw_c
    s.depth[:] = z
    s.id[:] = np.arange(n)
    s.next_id = n
    return params.astype(np.float32), s


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("p", [1, 2])
def test_principal_point_render_equals_reference_2d(p):
    rng = np.random.default_rng(11 + p)
    cam = cam_identity(64, 48, 90.0)
    params, scene = _principal_point_scene(rng, 40, cam)
    rgb3, T3, ops3, _ = B.render3d(params, cam, p, 0, 0)
    rgb2, T2, ops2, _ = B.render(scene, p, 0, 0, cam.width, cam.height, impl="ref_native")
    assert ops3 == ops2
    np.testing.assert_allclose(rgb3, rgb2, atol=2e-5)
    np.testing.assert_allclose(T3, T2, atol=2e-5)


def test_synthetic_scene_projects_into_image():
    cam = Camera.look_at((0.5, -0.2, -1.0), (0.0, 0.0, 4.0), (0, -1, 0), 60.0, 160, 90)
    m = GaussianModel3D.synthetic(7, 500, cam)
    rec = B.prepare3d(m.params, cam, 1)
    assert len(rec["orig"]) == 500  # all in front of the camera
    assert np.all((rec["mx"] >= 0) & (rec["mx"] <= cam.width))
    assert np.all((rec["my"] >= 0) & (rec["my"] <= cam.height))
    assert np.all(np.diff(rec["depth"]) >= 0)


def test_adam3d_first_step_moves_by_lr():
    # the first Adam step moves each component by ~lr * sign(g)
    cfg = B.adam3d_config(1, 100, 2.0)
    n = 3
    p = np.zeros((59, n), np.float32)
    g = np.ones((59, n), np.float32)
    m = np.zeros_like(p)
    v = np.zeros_like(p)
    B.adam3d_step(p, g, m, v, cfg)
    assert p[0, 0] == pytest.approx(-1.6e-4 * 2.0 * 0.01 ** (1 / 100), rel=1e-5)  # decayed schedule
    assert p[3, 0] == pytest.approx(-1e-3, rel=1e-5)
    assert p[7, 0] == pytest.approx(-5e-3, rel=1e-5)
    assert p[10, 0] == pytest.approx(-5e-2, rel=1e-5)
    assert p[11, 0] == pytest.approx(-2.5e-3, rel=1e-5)
    assert p[20, 0] == pytest.approx(-2.5e-3 / 20, rel=1e-5)


# ---------------------------------------------------------------- 3-D densify (SPEC examples)
def _dstate(n, seed=0, pos=1e-2, visits=10):
    rng = np.random.default_rng(seed)
    P = rng.normal(size=(59, n)).astype(np.float32)
    P[3] = 1.0 + np.abs(P[3])
    P[10] = 1.0  # opacity 0.73: above both floors
    return {"params": P, "m1": np.zeros((59, n), np.float32), "m2": np.zeros((59, n), np.float32),
            "pos_acc": rng.uniform(0.5, 1.0, n).astype(np.float32) * pos,
            "col_acc": np.zeros(n, np.float32), "visit": np.full(n, visits, np.int32),
            "visit_evt": np.zeros(n, np.int32), "visit_aud": np.zeros(n, np.int32),
            "ids": np.arange(n, dtype=np.uint64), "tau_v": np.full(n, 5.0), "next_id": n}


def test_densify3d_spec_examples():
    """SPEC.md:330-347 examples on the 3-D restatement: budget 0 -> unchanged; 10 candidates,
    budget 4 -> the 4 highest averaged position norms spawn; one candidate -> one child inside
    the parent's 1-sigma ellipsoid at half scale; all below the prune floor -> empty."""
    B.set_math(True)
    cfg = B.densify_config(2e-4)
    s = _dstate(10)
    out, (sp, pr, nc, _) = B.densify3d_event(s, cfg, 10, B.Pcg32(1, 1))
    assert (sp, pr, nc) == (0, 0, 10) and np.array_equal(out["params"], s["params"])
    out, (sp, _, _, _) = B.densify3d_event(s, cfg, 14, B.Pcg32(1, 1))
    top = np.argsort(-(s["pos_acc"] / 10.0), kind="stable")[:4]
    assert sp == 4 and out["params"].shape[1] == 14
    assert np.array_equal(np.sort(np.nonzero(np.isin(np.arange(10), top))[0]),
                          np.sort([int(np.nonzero((out["params"][11:, 10 + j][:, None] == s["params"][11:]).all(0))[0][0])
                                   for j in range(4)]))
    one = _dstate(1, seed=3)
    out, (sp, _, _, _) = B.densify3d_event(one, cfg, 100, B.Pcg32(2, 1))
    assert sp == 1
    th, ch = one["params"][:, 0].astype(np.float64), out["params"][:, 1].astype(np.float64)
    w, x, y, z = th[3:7] / np.linalg.norm(th[3:7])
    R = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                  [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                  [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
    d = R.T @ (ch[:3] - th[:3]) / np.exp(th[7:10])
    assert np.linalg.norm(d) <= 1.0 + 1e-6
    assert np.allclose(ch[7:10], th[7:10] - np.log(2.0), atol=1e-6)
    assert abs(1.0 / (1.0 + np.exp(-ch[10])) - 0.1) < 1e-6 and out["ids"][1] == 1 and out["next_id"] == 2
    low = _dstate(5)
    low["params"][10] = -8.0
    out, (_, pr, _, _) = B.densify3d_event(low, cfg, 100, B.Pcg32(1, 1))
    assert pr == 5 and out["params"].shape[1] == 0


def test_visit_audit3d_spec_examples():
    """v = 10, tau 8 -> 8; v = 3, tau 8 -> 4; v = 0, tau 1 -> 1."""
    s = _dstate(3)
    s["visit"] = np.array([10, 3, 0], np.int32)
    s["tau_v"] = np.array([8.0, 8.0, 1.0])
    tv, va = B.visit_audit3d(s)
    assert list(tv) == [8.0, 4.0, 1.0] and list(va) == [10, 3, 0]
