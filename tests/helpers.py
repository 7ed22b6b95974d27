"""Shared test helpers: build the same scene for the oracle (oracle.bind.Scene) and for the
product (paper_2412_13547_b200.GaussianModel)."""
import numpy as np

from oracle import bind as B

FIELDS = ("px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb", "depth")


def model_from_scene(s: "B.Scene"):
    from paper_2412_13547_b200 import GaussianModel
    m = GaussianModel(s.n)
    for i, f in enumerate(FIELDS):
        m.params[i] = getattr(s, f)
    m.id = np.ascontiguousarray(s.id, np.uint64).copy()
    m.set_next_id(max(int(s.next_id), int(s.id.max()) + 1 if s.n else 0))
    s.ensure_stats()
    m.pos_grad_norm_accum = s.pos_acc.copy()
    m.color_grad_norm_accum = s.col_acc.copy()
    m.accum_count = s.accum.copy()
    m.visit_count = s.visit.copy()
    m.window_visit_count = s.window.copy()
    m.visit_thresholds = s.tau_v.copy()
    return m


def scene_from_model(m) -> "B.Scene":
    s = B.Scene.empty(m.size())
    for i, f in enumerate(FIELDS):
        setattr(s, f, m.params[i].copy())
    s.id = m.id.copy()
    s.next_id = m.next_id()
    s.pos_acc = m.pos_grad_norm_accum.copy()
    s.col_acc = m.color_grad_norm_accum.copy()
    s.accum = m.accum_count.copy()
    s.visit = m.visit_count.copy()
    s.window = m.window_visit_count.copy()
    s.tau_v = m.visit_thresholds.copy()
    return s


def target_image(seed, n, W, H, p=1, bg=(0, 0, 0)):
    """Loss target: the oracle render of the seed-2 synthetic scene at every pixel (W*H*3)."""
    t = B.synthetic_scene(seed, n, W, H)
    rgb, _, _, _ = B.render(t, 1, 0, 0, W, H, bg)
    return rgb.reshape(H, W, 3)


T_TERM = 1e-4          # rasterizer.cpp:129 termination threshold
# A pixel is a "threshold pixel" when one side's final T sits within this relative distance of
# 1e-4: the two sides took the termination branch (rasterizer.cpp:129) on opposite sides of the
# threshold after T values that differ by a few ulp of drift (fast exp2 vs expf, FMA).
T_EVIDENCE_REL = 2e-5


def render_check(rgb, T, ops, rrgb, rT, rops, atol=1e-5, label=""):
    """SURVEY.md §8c render parity: colours / T within `atol` abs at every pixel EXCEPT threshold
    pixels, each of which must carry |T - 1e-4| evidence (on the GPU side or the reference side)
    and may move only by the colour of what lies behind T ~ 1e-4. Returns the list of threshold
    pixels (rank, gpu T, ref T, max colour diff) so callers can report them."""
    rgb = np.asarray(rgb, np.float64).reshape(-1, 3)
    rrgb = np.asarray(rrgb, np.float64).reshape(-1, 3)
    T = np.asarray(T, np.float64).ravel()
    rT = np.asarray(rT, np.float64).ravel()
    d = np.abs(rgb - rrgb).max(axis=1)
    dT = np.abs(T - rT)
    bad = np.nonzero((d > atol) | (dT > atol))[0]
    ev = np.minimum(np.abs(T[bad] - T_TERM), np.abs(rT[bad] - T_TERM))
    unexplained = bad[ev > T_EVIDENCE_REL * T_TERM]
    assert unexplained.size == 0, (
        f"{label}: {unexplained.size} pixels off without threshold evidence; first "
        + str([(int(r), float(T[r]), float(rT[r]), float(d[r])) for r in unexplained[:5]]))
    # one more / fewer blend behind T ~ 1e-4 changes a colour by at most T * (|c| + |bg|) < 3e-4
    assert d.max(initial=0.0) <= 3e-4, f"{label}: max colour diff {d.max():.3g}"
    assert abs(int(ops) - int(rops)) <= max(4, 16 * bad.size, int(1e-5 * rops)), (label, ops, rops)
    return [(int(r), float(T[r]), float(rT[r]), float(d[r])) for r in bad]


def frac_close(a, b, rtol, atol):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    ok = np.abs(a - b) <= atol + rtol * np.abs(b)
    return ok.mean() if ok.size else 1.0
