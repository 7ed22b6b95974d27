"""Multi-rank view sharding on CPU (gloo, world_size 2): the PRODUCT's host-side logic of the
batched step — paper_2412_13547_b200.dist.ViewShardedFit.step: view assignment, the canonical
row-order step (step_layout) on ranks, the all-reduce of the step buffer, apply over the global
view count — reproduces the single-process batched step exactly.

The model behind ViewShardedFit is a host test double with the DeviceModel step protocol whose
per-view increments come from the CPU oracle. Like the device model (csrc/capi.cu physical row
order), it keeps its rows — and the step buffer — in blend order after a fused view and in
logical order otherwise, and applies the buffer to its PHYSICAL rows: a rank with no view of a
step that skipped the canonical-order step would apply blend-ordered sums to logically ordered
rows and diverge (dist.py), which the world > views case below checks."""
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

W, H, N = 48, 40, 300


def _targets(views):
    rng = np.random.default_rng(1)
    base = B.render(B.synthetic_scene(2, N, W, H), 1, 0, 0, W, H)[0].reshape(H, W, 3)
    return [(base + rng.normal(0, 0.02, base.shape)).astype(np.float32) for _ in range(views)]


def view_increment(s, v, target):
    """One view's [n][12] step-buffer increment (layout of dist.STEP_ROWS), logical order."""
    p = 2
    ox, oy = (v % 4) % 2, (v % 4) // 2   # the batch's views = the p^2 cycled offsets
    rgb = B.render(s, p, ox, oy, W, H)[0]
    _, dl = B.l1_loss(rgb, p, ox, oy, W, H, target)
    t = s.copy().ensure_stats()
    t.pos_acc[:] = 0
    t.col_acc[:] = 0
    t.visit[:] = 0
    g, _ = B.backward(t, p, ox, oy, W, H, dl)
    buf = np.zeros((s.n, D.STEP_ROWS), np.float32)
    buf[:, D.ROW_GRADS] = g.T
    buf[:, D.ROW_POS_NORM] = t.pos_acc
    buf[:, D.ROW_COL_NORM] = t.col_acc
    buf[:, D.ROW_VISITS] = t.visit
    return buf


def apply(s, buf, nviews, m1, m2, step):
    """apply_step on a LOGICAL-order buffer [n][12]."""
    s.ensure_stats()
    grads = (buf[:, D.ROW_GRADS].T / np.float32(nviews)).astype(np.float32)
    B.adam_step(s, np.ascontiguousarray(grads), m1, m2, B.adam_config(step, 100, math.hypot(W, H)))
    vis = buf[:, D.ROW_VISITS].astype(np.int64)
    s.pos_acc += buf[:, D.ROW_POS_NORM]
    s.col_acc += buf[:, D.ROW_COL_NORM]
    s.accum += vis.astype(np.int32)
    s.visit += vis
    s.window += vis


class OracleStepModel:
    """DeviceModel step protocol over the oracle, with the device model's physical row order."""

    def __init__(self, s):
        self.s = s
        self.perm = B.sorted_order(s).astype(np.int64)   # blend rank -> logical index
        self.blend = False
        self.buf = torch.zeros((s.n, D.STEP_ROWS), dtype=torch.float32)
        self.m1 = np.zeros((9, s.n), np.float32)
        self.m2 = np.zeros((9, s.n), np.float32)

    def _to_blend(self):  # permute_model: rows and step buffer move together
        if not self.blend:
            self.buf.copy_(self.buf[torch.from_numpy(self.perm)])
            self.blend = True

    def view_accumulate(self, pattern, background, target):
        self._to_blend()
        inc = view_increment(self.s, pattern, target)
        self.buf += torch.from_numpy(inc[self.perm])
        return 0.0

    def step_layout(self):
        self._to_blend()

    def step_tensor(self):
        return self.buf.view(-1)

    def apply_step(self, nviews, step, total_steps, diag):
        phys = self.buf.numpy()
        logical = np.empty_like(phys)
        if self.blend:
            logical[self.perm] = phys
        else:
            logical[:] = phys
        apply(self.s, logical, nviews, self.m1, self.m2, step)
        self.buf.zero_()


def _worker(rank, world, port, views, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    B.set_math(True)
    model = OracleStepModel(B.synthetic_scene(1, N, W, H).ensure_stats())
    fit = D.ViewShardedFit(model, rank, world, comm="torch")
    targets = _targets(views)
    for step in (1, 2):
        fit.step([(v, targets[v]) for v in range(views)], (0, 0, 0), step, 100, math.hypot(W, H))
    s = model.s
    out[rank] = (s.px.copy(), s.rop.copy(), s.pos_acc.copy(), s.visit.copy())
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def test_views_for_rank():
    assert D.views_for_rank(8, 0, 1) == list(range(8))
    assert D.views_for_rank(8, 1, 4) == [1, 5]
    assert D.views_for_rank(1, 1, 2) == []
    assert sorted(sum((D.views_for_rank(8, r, 3) for r in range(3)), [])) == list(range(8))
    with pytest.raises(ValueError):
        D.views_for_rank(8, 2, 2)


@pytest.mark.parametrize("views", [4, 3, 1])
def test_two_rank_gloo_matches_single_process(views):
    """views=1: rank 1 renders nothing and must still apply the reduced sums to the right rows."""
    B.set_math(True)
    ctx = mp.get_context("spawn")
    mgr = ctx.Manager()
    out = mgr.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, views, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    # single process reference of the same two batched steps (logical order throughout)
    s = B.synthetic_scene(1, N, W, H).ensure_stats()
    targets = _targets(views)
    m1 = np.zeros((9, N), np.float32)
    m2 = np.zeros((9, N), np.float32)
    for step in (1, 2):
        buf = sum(view_increment(s, v, targets[v]) for v in range(views))
        apply(s, buf, views, m1, m2, step)
    r0, r1 = out[0], out[1]
    for a, b in zip(r0, r1):
        assert np.array_equal(a, b)            # ranks stay bit-identical
    # ring/gloo summation order differs from the sequential sum only at ulp level
    assert np.allclose(r0[0], s.px, rtol=0, atol=1e-4)
    assert np.allclose(r0[1], s.rop, rtol=0, atol=1e-4)
    assert np.allclose(r0[2], s.pos_acc, rtol=1e-5, atol=1e-9)
    assert np.array_equal(r0[3], s.visit)
