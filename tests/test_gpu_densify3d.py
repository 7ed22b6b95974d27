"""GPU densification of the 3-D model (tgsx_densify3d, csrc/densify3d.cu) against its FP64/C
restatement (oracle/ewa3d.c or3d_densify_event): the SPEC's 2-D densify event
on the 3-D parameters. No reference code exists for it (the reference densifier is 2-D and
missing), so the oracle restatement is the specification; its SPEC examples are checked in
tests/test_oracle3d.py.

Exactness written here: candidate count, colour coin, spawn / prune counts, selections (ids),
parent rows, copied child parameters, moments, statistics, tau_v and the advanced PCG32 state are
bit-exact (same float predicates: CR activation, IEEE averages, double tau_v; stable top-k). Child
means go through double cbrt / sin / cos / exp, whose last ulp may differ between CUDA and glibc:
|gpu - ref| <= 1e-6 (|ref| + parent 1-sigma extent). Every child lies inside its parent's 1-sigma
ellipsoid (Mahalanobis <= 1 + 1e-5).
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


def _cams(S, W=192, H=144):
    eyes = [(0.3, -0.2, -0.5), (-0.6, 0.1, -0.4), (0.1, 0.5, -0.6), (0.7, 0.3, -0.2)]
    return [S.Camera.look_at(e, (0.0, 0.0, 4.5), (0, -1, 0), 60.0, W, H) for e in eyes]


def _fitted(S, ctx, n=4000, steps=12, seed=3, low_opacity=40):
    cams = _cams(S)
    m = S.GaussianModel3D.synthetic(seed, n, cams[0])
    m.params[10, :low_opacity] = -7.0  # sigmoid < 0.005: pruned
    dm = S.DeviceModel3D.from_host(m, ctx)
    tgt = S.GaussianModel3D.synthetic(seed + 100, n, cams[0])
    td = S.DeviceModel3D.from_host(tgt, ctx)
    targets = [td.render(c).colors.reshape(c.height, c.width, 3) for c in cams]
    td.close()
    for it in range(steps):
        c = cams[it % len(cams)]
        dm.fit_step(c, None, (0.0, 0.0, 0.0), targets[it % len(cams)], it + 1, 100, 3.0)
    return cams, targets, dm


def _state(dm):
    n = dm.size()
    params = dm.download().params
    m1, m2 = dm.moments()
    pos, col, vis = dm.stats()
    ids, tau, ve, va, nxt = dm.densify_state()
    return {"params": params, "m1": m1, "m2": m2, "pos_acc": pos, "col_acc": col, "visit": vis,
            "visit_evt": ve, "visit_aud": va, "ids": ids, "tau_v": tau, "next_id": nxt, "n": n}


def _check_event(P, dm, budget, tau_pos, color_prob=0.2, seed=11):
    B.set_math(True)
    pre = _state(dm)
    avg = pre["pos_acc"] / np.maximum(pre["visit"] - pre["visit_evt"], 1)
    rng_ref = B.Pcg32(seed, 1)
    st = np.array(rng_ref.state, np.uint64)
    cfg = P.densify_config(tau_pos=tau_pos, color_branch_prob=color_prob)
    rep = dm.densify(budget, st, cfg)
    ocfg = B.densify_config(tau_pos)
    ocfg.color_branch_prob = color_prob
    ref, (sp, pr, nc, coin) = B.densify3d_event(pre, ocfg, budget, rng_ref)
    got = _state(dm)
    assert (rep.candidates, rep.spawned, rep.pruned, rep.color_coin) == (nc, sp, pr, coin)
    assert tuple(int(v) for v in st) == tuple(int(v) for v in rng_ref.state)
    assert got["n"] == ref["params"].shape[1] == rep.count_after
    assert got["n"] <= max(budget, pre["n"])
    for k in ("ids", "visit", "visit_evt", "visit_aud", "tau_v", "pos_acc", "col_acc", "m1", "m2"):
        assert np.array_equal(got[k], ref[k]), k
    assert got["next_id"] == ref["next_id"]
    # parameters: exact except the children's means (double transcendentals)
    n_old = pre["next_id"]
    child = got["ids"] >= n_old
    gp, rp = got["params"], ref["params"]
    assert np.array_equal(gp[:, ~child], rp[:, ~child])
    assert np.array_equal(gp[3:, child], rp[3:, child])
    if child.any():
        ext = np.exp(rp[7:10, child] + np.log(2.0)).max(axis=0)  # parent 1-sigma extent
        assert np.all(np.abs(gp[:3, child] - rp[:3, child]) <= 1e-6 * (np.abs(rp[:3, child]) + ext))
        # every child inside its parent's 1-sigma ellipsoid; the parent is the pre-event row whose
        # SH coefficients the child copied (unique for random synthetic scenes)
        cp = gp[:, child]
        sh_rows = {pre["params"][11:, r].tobytes(): r for r in range(pre["n"])}
        for c in range(cp.shape[1]):
            th = pre["params"][:, sh_rows[cp[11:, c].tobytes()]]
            q = th[3:7] / np.linalg.norm(th[3:7].astype(np.float64))
            w, x, y, z = q
            Rm = np.array([[1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y)],
                           [2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x)],
                           [2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)]])
            d = Rm.T @ (cp[:3, c].astype(np.float64) - th[:3].astype(np.float64))
            maha = np.sqrt(np.sum((d / np.exp(th[7:10].astype(np.float64))) ** 2))
            assert maha <= 1.0 + 1e-5
            assert np.array_equal(cp[3:7, c], th[3:7]) and np.array_equal(cp[11:, c], th[11:])
    return rep, pre, avg


def test_densify3d_under_and_over_budget(P, S, ctx):
    cams, targets, dm = _fitted(S, ctx)
    pre = _state(dm)
    avg = pre["pos_acc"] / np.maximum(pre["visit"] - pre["visit_evt"], 1)
    tau = float(np.quantile(avg[avg > 0], 0.5))
    # budget above the candidate count: every candidate spawns
    rep, _, _ = _check_event(P, dm, pre["n"] + 10 ** 6, tau, seed=5)
    assert rep.spawned == rep.candidates > 0 and rep.pruned == 40
    # the fit continues on the grown model (stats accumulate from the event mark)
    for it in range(8):
        dm.fit_step(cams[it % 4], None, (0.0, 0.0, 0.0), targets[it % 4], 20 + it, 100, 3.0)
    n1 = dm.size()
    rep2, pre2, _ = _check_event(P, dm, n1 + 25, tau * 0.5, seed=6)  # over budget: top-25
    assert rep2.candidates > 25 and rep2.spawned == 25
    assert dm.size() <= n1 + 25


def test_densify3d_color_branch_and_zero_budget(P, S, ctx):
    cams, targets, dm = _fitted(S, ctx, seed=4, low_opacity=0)
    pre = _state(dm)
    rep, _, _ = _check_event(P, dm, pre["n"], 1e9, color_prob=1.0, seed=7)  # no room: nothing spawns
    assert rep.spawned == 0 and rep.color_coin == 1
    for it in range(6):
        dm.fit_step(cams[it % 4], None, (0.0, 0.0, 0.0), targets[it % 4], 30 + it, 100, 3.0)
    pre = _state(dm)
    cavg = pre["col_acc"] / np.maximum(pre["visit"] - pre["visit_evt"], 1)
    # position gate closed (tau huge): only the colour branch (coin always on) selects
    tau_c = float(np.quantile(cavg[cavg > 0], 0.7))
    rep, _, _ = _check_event(P, dm, pre["n"] + 10 ** 6, tau_c / 0.01, color_prob=1.0, seed=8)
    assert rep.candidates > 0 and rep.spawned == rep.candidates


def test_visit_audit3d(P, S, ctx):
    cams, targets, dm = _fitted(S, ctx, seed=5, steps=6)
    pre = _state(dm)
    dm.visit_audit()
    tv, va = B.visit_audit3d(pre)
    _, tau, _, vaud, _ = dm.densify_state()
    assert np.array_equal(tau, tv) and np.array_equal(vaud, va)
    assert np.all(tau >= 1.0) and np.all(tau <= pre["tau_v"])


def test_batched_step_after_densify(P, S, ctx):
    """The packed [62][n] step buffer follows the new count: a batched multi-camera step right
    after a densify event runs on the grown model and leaves it finite."""
    cams, targets, dm = _fitted(S, ctx, seed=6)
    pre = _state(dm)
    avg = pre["pos_acc"] / np.maximum(pre["visit"] - pre["visit_evt"], 1)
    st = np.array(B.Pcg32(9, 1).state, np.uint64)
    dm.densify(pre["n"] + 10 ** 6, st, P.densify_config(tau_pos=float(np.quantile(avg[avg > 0], 0.3))))
    n = dm.size()
    assert n > pre["n"] - 40
    losses = [dm.view_accumulate(c, None, (0.0, 0.0, 0.0), t) for c, t in zip(cams[:2], targets[:2])]
    dm.apply_step(2, 50, 100, 3.0)
    assert all(np.isfinite(losses)) and np.all(np.isfinite(dm.download().params))


def test_densify3d_error_paths(P, S, ctx):
    """tgsx_densify3d refuses a model with a batched step in progress (TGSX_ESTATE) and bad
    arguments (TGSX_EINVAL); Trainer3D rejects an inconsistent schedule."""
    cams = _cams(S)
    m = S.GaussianModel3D.synthetic(9, 500, cams[0])
    dm = S.DeviceModel3D.from_host(m, ctx)
    tgt = np.full((cams[0].height, cams[0].width, 3), 0.3, np.float32)
    dm.view_accumulate(cams[0], None, (0.0, 0.0, 0.0), tgt)
    st = np.array(B.Pcg32(1, 1).state, np.uint64)
    with pytest.raises(Exception):
        dm.densify(1000, st, P.densify_config())
    dm.apply_step(1, 1, 10, 3.0)
    rep = dm.densify(1000, st, P.densify_config())  # allowed again once the step is applied
    assert rep.count_after == dm.size()
    bad = P.train_config(total_iters=100, warmup_iters=50, densify_until=20)  # warmup > densify_until
    with pytest.raises(Exception):
        S.Trainer3D(dm, cams, 3.0, bad)
