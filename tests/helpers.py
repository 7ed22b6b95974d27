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


def frac_close(a, b, rtol, atol):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    ok = np.abs(a - b) <= atol + rtol * np.abs(b)
    return ok.mean() if ok.size else 1.0
