"""The GPU fit loop (libtgsx trainer: schedule, budget controller, densify cadence, random
post-densify dilation, batched finale) against the same schedule restated over the CPU oracle
(tests/oracle_trainer.py). Trajectories are compared event by event: per-iteration FP32
differences are tiny, so losses and densify decisions agree early on; later the two runs may
drift by a few spawned Gaussians, which is checked statistically. Budget compliance
(acceptance #8) is checked at every densify event."""
import math

import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import model_from_scene
from tests.oracle_trainer import oracle_train

pytestmark = pytest.mark.gpu


def test_trainer_matches_oracle_schedule():
    import paper_2412_13547_b200 as P
    B.set_math(True)
    W, H, n = 64, 48, 300
    s = B.synthetic_scene(1, n, W, H)
    base = B.render(B.synthetic_scene(2, 600, W, H), 1, 0, 0, W, H)[0].reshape(H, W, 3)
    rng = np.random.default_rng(0)
    targets = [np.clip(base + rng.normal(0, 0.02, base.shape), 0, 1).astype(np.float32) for _ in range(4)]
    cfg = P.train_config(total_iters=400, warmup_iters=60, densify_interval=20, densify_until=300,
                         batch_final_iters=20, batch_size=4, dilation_p=2, n_views=4,
                         m_final=700.0, seed=7)
    cfg.densify.tau_pos = 2e-5
    ctx = P.Context(0)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    tr = P.Trainer(dm, W, H, cfg)
    tr.set_targets(targets)
    events, losses = [], []
    for t in range(1, 401):
        rep = tr.step()
        if rep.densified:
            events.append((t, rep.budget, rep.count, rep.spawned, rep.pruned))
            assert rep.count <= rep.budget  # budget compliance
        if t % 50 == 0:
            losses.extend(tr.losses(50).tolist())
    os_, olosses, oevents = oracle_train(s, targets, cfg, W, H, 400)
    losses = np.array(losses)
    assert len(events) == len(oevents) == (300 - 60) // 20
    # early events identical (same budget, same spawn / prune counts)
    for e, o in zip(events[:3], oevents[:3]):
        assert e == o, (e, o)
    for (t, Bt, cnt, sp, pr), (ot, oB, ocnt, osp, opr) in zip(events, oevents):
        assert t == ot and abs(Bt - oB) <= max(2, 0.02 * oB) and abs(cnt - ocnt) <= max(3, 0.03 * ocnt)
        assert ocnt <= oB
    assert np.allclose(losses[:100], olosses[:100], rtol=2e-3)
    assert abs(losses[-20:].mean() - olosses[-20:].mean()) <= 0.03 * olosses[-20:].mean()
    assert losses[-50:].mean() < losses[:50].mean()  # the fit makes progress
    st = tr.budget_state()
    assert 0.1 <= st["alpha"] <= 2.0


def _run_trainer(P, s, targets, cfg, W, H, iters, graph):
    import os
    os.environ["TGSX_TRAINER_GRAPH"] = "1" if graph else "0"
    try:
        ctx = P.Context(0)
        dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
        tr = P.Trainer(dm, W, H, cfg)
    finally:
        os.environ.pop("TGSX_TRAINER_GRAPH", None)
    tr.set_targets([t.data_ptr() for t in targets])
    reps = [tr.step() for _ in range(iters)]
    losses = tr.losses(iters)
    params = dm.download().params
    stats = ctx.graph_stats()
    tr.close()
    return [(r.densified, r.count, r.spawned, r.pruned, r.dilated) for r in reps], losses, params, stats


def test_trainer_graph_replay_matches_eager():
    """The trainer replays its warm-up and post-densification steps from CUDA graphs (one per
    pattern; the view's target is staged by a node of the graph) when the targets are
    device-resident: the trajectory over three round-robined targets — reports, per-iteration
    losses, final parameters — is bit-identical to the all-eager loop, dense SSIM iterations and
    the batched finale included."""
    import torch
    import paper_2412_13547_b200 as P
    B.set_math(True)
    W, H, n = 128, 96, 2000
    s = B.synthetic_scene(3, n, W, H)
    targets = [torch.from_numpy(np.ascontiguousarray(
        B.render(B.synthetic_scene(sd, 3000, W, H), 1, 0, 0, W, H)[0].reshape(H, W, 3), dtype=np.float32)).cuda()
        for sd in (4, 5, 6)]
    cfg = P.train_config(total_iters=200, warmup_iters=60, densify_interval=20, densify_until=120,
                         batch_final_iters=20, batch_size=4, dilation_p=2, n_views=50,
                         m_final=3000.0, seed=11)
    cfg.densify.tau_pos = 2e-5
    eager = _run_trainer(P, s, targets, cfg, W, H, 200, graph=False)
    graph = _run_trainer(P, s, targets, cfg, W, H, 200, graph=True)
    assert eager[0] == graph[0]
    assert any(r[0] for r in graph[0]) and any(not r[4] for r in graph[0])  # events, dense steps
    assert np.array_equal(eager[1], graph[1])
    assert np.array_equal(eager[2], graph[2])
    captures, replays, _ = graph[3]
    assert eager[3][1] == 0 and replays > 80 and captures <= 16
