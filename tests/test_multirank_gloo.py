"""Multi-rank view sharding on CPU (gloo, world_size 2): the host-side logic of the batched
step (view assignment, step-buffer layout, all-reduce, mean + stats application) reproduces the
single-process batched step exactly. Per-view increments come from the CPU oracle here; on the
GPU the same buffer is produced by tgsx_view_accumulate and reduced over NCCL
(paper_2412_13547_b200/dist.py)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import bind as B
from paper_2412_13547_b200 import dist as D

W, H, N, VIEWS = 48, 40, 300, 4


def _targets():
    rng = np.random.default_rng(1)
    base = B.render(B.synthetic_scene(2, N, W, H), 1, 0, 0, W, H)[0].reshape(H, W, 3)
    return [(base + rng.normal(0, 0.02, base.shape)).astype(np.float32) for _ in range(VIEWS)]


def view_increment(s, v, target):
    """One view's [12][n] step-buffer increment (layout of dist.STEP_ROWS)."""
    p = 2
    ox, oy = (v % 4) % 2, (v % 4) // 2   # the batch's views = the p^2 cycled offsets
    rgb = B.render(s, p, ox, oy, W, H)[0]
    _, dl = B.l1_loss(rgb, p, ox, oy, W, H, target)
    t = s.copy().ensure_stats()
    t.pos_acc[:] = 0
    t.col_acc[:] = 0
    t.visit[:] = 0
    g, _ = B.backward(t, p, ox, oy, W, H, dl)
    buf = np.zeros((D.STEP_ROWS, s.n), np.float32)
    buf[D.ROW_GRADS] = g
    buf[D.ROW_POS_NORM] = t.pos_acc
    buf[D.ROW_COL_NORM] = t.col_acc
    buf[D.ROW_VISITS] = t.visit
    return buf


def apply(s, buf, nviews, m1, m2, step):
    s.ensure_stats()
    grads = (buf[D.ROW_GRADS] / np.float32(nviews)).astype(np.float32)
    B.adam_step(s, grads, m1, m2, B.adam_config(step, 100, math.hypot(W, H)))
    vis = buf[D.ROW_VISITS].astype(np.int64)
    s.pos_acc += buf[D.ROW_POS_NORM]
    s.col_acc += buf[D.ROW_COL_NORM]
    s.accum += vis.astype(np.int32)
    s.visit += vis
    s.window += vis


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    s = B.synthetic_scene(1, N, W, H).ensure_stats()
    targets = _targets()
    m1 = np.zeros((9, N), np.float32)
    m2 = np.zeros((9, N), np.float32)
    for step in (1, 2):
        buf = np.zeros((D.STEP_ROWS, N), np.float32)
        for v in D.views_for_rank(VIEWS, rank, world):
            buf += view_increment(s, v, targets[v])
        t = torch.from_numpy(buf)
        dist.all_reduce(t)
        apply(s, t.numpy(), VIEWS, m1, m2, step)
    out[rank] = (s.px.copy(), s.rop.copy(), s.pos_acc.copy(), s.visit.copy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_views_for_rank():
    assert D.views_for_rank(8, 0, 1) == list(range(8))
    assert D.views_for_rank(8, 1, 4) == [1, 5]
    assert sorted(sum((D.views_for_rank(8, r, 3) for r in range(3)), [])) == list(range(8))
    with pytest.raises(ValueError):
        D.views_for_rank(8, 2, 2)


def test_two_rank_gloo_matches_single_process():
    B.set_math(True)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    # single process reference of the same two batched steps
    s = B.synthetic_scene(1, N, W, H).ensure_stats()
    targets = _targets()
    m1 = np.zeros((9, N), np.float32)
    m2 = np.zeros((9, N), np.float32)
    for step in (1, 2):
        buf = sum(view_increment(s, v, targets[v]) for v in range(VIEWS))
        apply(s, buf, VIEWS, m1, m2, step)
    r0, r1 = out[0], out[1]
    for a, b in zip(r0, r1):
        assert np.array_equal(a, b)            # ranks stay bit-identical
    # ring/gloo summation order differs from the sequential sum only at ulp level
    assert np.allclose(r0[0], s.px, rtol=0, atol=1e-4)
    assert np.allclose(r0[2], s.pos_acc, rtol=1e-5, atol=1e-9)
    assert np.array_equal(r0[3], s.visit)
