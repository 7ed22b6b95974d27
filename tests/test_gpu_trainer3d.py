"""The 3-D fit loop (tgsx_trainer3d_*: the SPEC schedule over a set of cameras with tgsx_densify3d
at every densify event) against the same schedule restated over the FP64 3-D oracle
(tests/oracle_trainer3d.py). GPU and oracle gradients agree to the 3-D front end's tolerance
(2e-3 of the largest per Gaussian, tests/test_gpu_3d.py), so the trajectories are compared
statistically: identical event cadence, budget compliance at every event, event
counts within 3 %, early losses within 1 %, final losses within 5 %, and the fit makes progress."""
import numpy as np
import pytest

from oracle import bind as B
from tests.oracle_trainer3d import oracle_train3d

pytestmark = pytest.mark.gpu


def test_trainer3d_matches_oracle_schedule():
    import paper_2412_13547_b200 as P
    from paper_2412_13547_b200 import scene3d as S
    B.set_math(True)
    W, H, n = 64, 48, 400
    eyes = [(0.3, -0.2, -0.5), (-0.5, 0.1, -0.4), (0.1, 0.4, -0.6)]
    cams = [S.Camera.look_at(e, (0.0, 0.0, 4.5), (0, -1, 0), 60.0, W, H) for e in eyes]
    m = S.GaussianModel3D.synthetic(1, n, cams[0])
    tgt_model = S.GaussianModel3D.synthetic(2, 2 * n, cams[0])
    targets = [B.render3d(tgt_model.params, c, 1, 0, 0)[0].reshape(H, W, 3).astype(np.float32) for c in cams]
    cfg = P.train_config(total_iters=300, warmup_iters=40, densify_interval=20, densify_until=220,
                         batch_final_iters=20, batch_size=3, dilation_p=2, n_views=6, m_final=900.0, seed=5)
    ctx = P.Context(0)
    dm = S.DeviceModel3D.from_host(m, ctx)
    # tau_pos at the scale of this scene's averaged screen-space position norms
    cfg.densify.tau_pos = 1e-6
    tr = S.Trainer3D(dm, cams, 3.0, cfg)
    tr.set_targets(targets)
    events, losses = [], []
    for t in range(1, 301):
        rep = tr.step()
        if rep.densified:
            events.append((t, rep.budget, rep.count, rep.spawned, rep.pruned))
            assert rep.count <= rep.budget  # budget compliance
        if t % 50 == 0:
            losses.extend(tr.losses(50).tolist())
    ost, olosses, oevents = oracle_train3d(m.params, cams, targets, cfg, 3.0, 300)
    losses = np.array(losses)
    assert len(events) == len(oevents) == (220 - 40) // 20
    assert sum(e[3] for e in events) > 0, "no Gaussian spawned: tau_pos too high for the scene"
    for (t, Bt, cnt, sp, pr), (ot, oB, ocnt, osp, opr) in zip(events, oevents):
        assert t == ot and abs(Bt - oB) <= max(2, 0.03 * oB) and abs(cnt - ocnt) <= max(4, 0.03 * ocnt)
        assert ocnt <= oB
    assert np.allclose(losses[:40], olosses[:40], rtol=1e-2)
    assert abs(losses[-20:].mean() - olosses[-20:].mean()) <= 0.05 * olosses[-20:].mean()
    assert losses[-30:].mean() < losses[:30].mean()
    assert dm.size() == events[-1][2] or dm.size() >= n
