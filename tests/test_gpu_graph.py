"""CUDA-graph replay of the fused fit step (tgsx_fit_graph_step): the
model after N graph-replayed steps is bit-identical to the model after N eager tgsx_fit_step
calls (parameters, Adam moments, densify statistics, last loss) — including dilated fits that
cycle the p x p offsets (one graph per offset), pinned host targets, and steps whose device-side
capacity guard faults (re-run eagerly in order)."""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def torch():
    import torch
    return torch


def _fit(P, torch, ctx, n, W, H, p, steps, graph, pinned=False):
    dm = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, n, W, H), ctx)
    tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(2, n, W, H), ctx)
    tgt = tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3).astype(np.float32)
    tm.close()
    diag = float(np.hypot(W, H))
    if pinned:
        t_buf = torch.from_numpy(tgt).pin_memory()
        loss = torch.zeros(1).pin_memory()
    else:
        t_buf = torch.from_numpy(tgt).cuda()
        loss = torch.zeros(1, device="cuda")
    torch.cuda.synchronize()
    losses = []
    for it in range(steps):
        ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
        pat = P.DilationPattern(p, ox, oy, W, H)
        if graph:
            dm.fit_graph_step(pat, (0.0, 0.0, 0.0), t_buf.data_ptr(), it + 1, 1000, diag, loss.data_ptr())
        else:
            losses.append(dm.fit_step(pat, (0.0, 0.0, 0.0), tgt, it + 1, 1000, diag))
    ctx.synchronize()
    out = dm.download()
    m1, m2 = dm.moments()
    last = float(loss.cpu()[0]) if graph else losses[-1]
    dm.close()
    return out, m1, m2, last


def _same(a, b):
    ma, m1a, m2a, la = a
    mb, m1b, m2b, lb = b
    assert np.array_equal(ma.params.view(np.uint32), mb.params.view(np.uint32))
    assert np.array_equal(m1a.view(np.uint32), m1b.view(np.uint32))
    assert np.array_equal(m2a.view(np.uint32), m2b.view(np.uint32))
    for f in ("pos_grad_norm_accum", "color_grad_norm_accum", "accum_count", "visit_count",
              "window_visit_count"):
        assert np.array_equal(getattr(ma, f), getattr(mb, f)), f
    assert np.float32(la) == np.float32(lb)


@pytest.mark.parametrize("n,W,H,p,steps", [(10_000, 256, 256, 1, 12), (40_000, 640, 480, 2, 14),
                                           (30_000, 512, 384, 3, 11)])
def test_graph_steps_match_eager(P, torch, n, W, H, p, steps):
    ctx = P.Context(0)
    eager = _fit(P, torch, ctx, n, W, H, p, steps, graph=False)
    g = _fit(P, torch, ctx, n, W, H, p, steps, graph=True)
    _same(eager, g)
    caps, replays, reruns = ctx.graph_stats()
    assert caps == p * p and replays == steps - p * p and reruns == 0
    ctx.close()


def test_graph_pinned_host_target(P, torch):
    ctx = P.Context(0)
    eager = _fit(P, torch, ctx, 10_000, 256, 256, 1, 8, graph=False)
    g = _fit(P, torch, ctx, 10_000, 256, 256, 1, 8, graph=True, pinned=True)
    _same(eager, g)
    assert ctx.graph_stats()[1] == 7
    ctx.close()


def test_graph_fault_reruns_eagerly(P, torch, monkeypatch):
    """A negative pair slack makes every replay exceed the capture-time capacity: the backward's
    device guard faults, the sticky word no-ops that step and its successor, and both are re-run
    eagerly in order — the final model is still bit-identical to the eager fit."""
    ctx = P.Context(0)
    eager = _fit(P, torch, ctx, 10_000, 256, 256, 1, 9, graph=False)
    monkeypatch.setenv("TGSX_GRAPH_PAIR_SLACK", "-1")
    g = _fit(P, torch, ctx, 10_000, 256, 256, 1, 9, graph=True)
    _same(eager, g)
    caps, replays, reruns = ctx.graph_stats()
    assert reruns > 0 and replays > 0
    ctx.close()


def test_graph_then_eager_entry_points_flush(P, torch):
    """An eager entry point after graph steps first verifies them (graph_flush): a render right
    after replayed steps sees the model those steps produced."""
    ctx = P.Context(0)
    W = H = 256
    dm = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, 10_000, W, H), ctx)
    tgt = torch.full((H, W, 3), 0.25, device="cuda")
    torch.cuda.synchronize()
    pat = P.DilationPattern(1, 0, 0, W, H)
    for it in range(6):
        dm.fit_graph_step(pat, (0.0, 0.0, 0.0), tgt.data_ptr(), it + 1, 1000, 362.0)
    img = dm.render(pat, (0.0, 0.0, 0.0)).colors
    ref = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, 10_000, W, H), ctx)
    host_t = np.full((H, W, 3), 0.25, np.float32)
    for it in range(6):
        ref.fit_step(pat, (0.0, 0.0, 0.0), host_t, it + 1, 1000, 362.0)
    assert np.array_equal(img, ref.render(pat, (0.0, 0.0, 0.0)).colors)
    dm.close()
    ref.close()
    ctx.close()


@pytest.mark.parametrize("p,steps,W,H", [(1, 9, 384, 256), (2, 13, 384, 256), (2, 9, 250, 131),
                                          (3, 14, 250, 131)])
def test_graph_per_replay_targets_and_losses(P, torch, p, steps, W, H):
    """A fit over several device targets with a new loss destination every step (the trainer's
    loss ring): after the second distinct target the graphs stage the target through a copy node
    whose source is set per replay, and the loss-copy node gets each step's destination — one
    graph per pattern, every loss and the final model bit-identical to eager steps. Widths not
    divisible by 4 take the staging kernel's scalar path (dilated views stage active rows)."""
    ctx = P.Context(0)
    n = 20_000
    diag = float(np.hypot(W, H))
    tgts = []
    for s in (2, 3, 4):
        tm = P.DeviceModel.from_host(P.GaussianModel.synthetic(s, n, W, H), ctx)
        tgts.append(tm.render(P.DilationPattern(1, 0, 0, W, H)).colors.reshape(H, W, 3).astype(np.float32))
        tm.close()
    dev = [torch.from_numpy(t).cuda() for t in tgts]
    ring = torch.zeros(steps, device="cuda")
    torch.cuda.synchronize()
    runs = []
    for graph in (False, True):
        dm = P.DeviceModel.from_host(P.GaussianModel.synthetic(1, n, W, H), ctx)
        losses = []
        for it in range(steps):
            ox, oy = (it % (p * p)) % p, (it % (p * p)) // p
            pat = P.DilationPattern(p, ox, oy, W, H)
            if graph:
                dm.fit_graph_step(pat, (0.0, 0.0, 0.0), dev[it % 3].data_ptr(), it + 1, 1000, diag,
                                  ring[it:it + 1].data_ptr())
            else:
                losses.append(dm.fit_step(pat, (0.0, 0.0, 0.0), tgts[it % 3], it + 1, 1000, diag))
        ctx.synchronize()
        out = dm.download()
        m1, m2 = dm.moments()
        runs.append((out, m1, m2, losses if not graph else ring.cpu().numpy().tolist()))
        dm.close()
    (ea, e1, e2, el), (ga, g1, g2, gl) = runs
    _same((ea, e1, e2, el[-1]), (ga, g1, g2, gl[-1]))
    assert np.array_equal(np.float32(el), np.float32(gl))
    caps, replays, reruns = ctx.graph_stats()
    assert caps == 1 + p * p and replays == steps - caps and reruns == 0
    ctx.close()
