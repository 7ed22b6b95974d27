"""In-library NCCL view sharding on one B200: a 1-rank communicator attached to
the context, the pipelined batched step (chain(b) -> all-reduce(b) -> Adam(b) over Gaussian
buckets) and the canonical row order of ranks without a view.

Multi-rank runs need several GPUs (the 8-GPU scaling run); here the same code paths run with
nranks = 1 and the cross-rank arithmetic is emulated on one GPU with two model replicas, which
is exactly what the all-reduce computes (tests/test_multirank_gloo.py covers the host-side
logic with 2 processes)."""
import math

import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import model_from_scene, target_image

pytestmark = pytest.mark.gpu

W, H, N = 160, 120, 6000


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    c = P.Context(0)
    c.comm_init(P.Context.comm_unique_id(), 1, 0)
    yield c
    c.comm_destroy()


def _views(P, k):
    t = target_image(2, N, W, H)
    rng = np.random.default_rng(0)
    out = []
    for v in range(k):
        ox, oy = P.next_offsets(2, v)
        out.append((P.DilationPattern(2, ox, oy, W, H), (t + rng.normal(0, 0.02, t.shape)).astype(np.float32)))
    return out


def _same(a, b):
    ha, hb = a.download(), b.download()
    return (np.array_equal(ha.params.view(np.uint32), hb.params.view(np.uint32)) and
            np.array_equal(ha.visit_count, hb.visit_count) and
            np.array_equal(ha.pos_grad_norm_accum.view(np.uint32), hb.pos_grad_norm_accum.view(np.uint32)))


@pytest.mark.parametrize("buckets", [1, 3, 8])
def test_batched_step_with_comm_equals_accumulate_apply(P, ctx, buckets):
    """tgsx_batched_step (1-rank NCCL all-reduce, bucketed pipeline) == view_accumulate x V +
    apply_step, bit for bit, over two steps."""
    assert ctx.comm_size() == 1
    s = B.synthetic_scene(1, N, W, H)
    a = P.DeviceModel.from_host(model_from_scene(s), ctx)
    plain_ctx = P.Context(0)
    b = P.DeviceModel.from_host(model_from_scene(s), plain_ctx)
    views = _views(P, 4)
    diag = math.hypot(W, H)
    for step in (1, 2):
        la = a.batched_step(views, (0, 0, 0), 4, step, 100, diag, buckets=buckets)
        lb = [b.view_accumulate(p, (0, 0, 0), t) for p, t in views]
        b.apply_step(4, step, 100, diag)
        assert la == lb
    assert _same(a, b)


def test_zero_view_rank_uses_canonical_rows(P, ctx):
    """Two replicas emulate two ranks: rank A renders every view of the step, rank B none (its
    rows in logical order after a download). B brings its rows to the canonical order
    (step_layout), receives A's sums (the all-reduce), applies: both replicas stay identical."""
    import torch
    s = B.synthetic_scene(3, N, W, H)
    a = P.DeviceModel.from_host(model_from_scene(s), ctx)
    b = P.DeviceModel.from_host(model_from_scene(s), ctx)
    views = _views(P, 2)
    diag = math.hypot(W, H)
    for step in (1, 2):
        for p, t in views:
            a.view_accumulate(p, (0, 0, 0), t)
        b.download()          # logical row order on B
        b.step_layout()       # what ViewShardedFit / tgsx_batched_step do on a rank with no view
        from paper_2412_13547_b200 import dist as D
        ta = D.step_buffer_tensor(a, 0)
        tb = D.step_buffer_tensor(b, 0)
        ctx.synchronize()
        tb += ta              # the all-reduce (sum over ranks; B's own buffer is zero)
        torch.cuda.synchronize()
        a.apply_step(2, step, 100, diag)
        b.apply_step(2, step, 100, diag)
    assert _same(a, b)


def test_zero_view_batched_step(P, ctx):
    """tgsx_batched_step with n_views = 0 (a rank with no view): layout + all-reduce + Adam of a
    zero buffer leaves the parameters unchanged (zero gradient -> zero Adam move on fresh moments)."""
    s = B.synthetic_scene(4, 2000, W, H)
    a = P.DeviceModel.from_host(model_from_scene(s), ctx)
    a.batched_step([], (0, 0, 0), 4, 1, 100, math.hypot(W, H))
    h = a.download()
    assert np.array_equal(h.params[0], s.px) and np.array_equal(h.visit_count, np.zeros(2000))


def test_pipeline_timeline_orders_buckets(P, ctx):
    """Profiled batched step: per bucket the all-reduce starts after its chain ends, Adam after its
    all-reduce ends; chain(b+1) is queued before Adam(b) waits (the overlap the pipeline exists
    for)."""
    s = B.synthetic_scene(5, 200_000, 640, 480)
    a = P.DeviceModel.from_host(model_from_scene(s), ctx)
    t = target_image(2, 2000, 640, 480)
    views = [(P.DilationPattern(2, 0, 0, 640, 480), t), (P.DilationPattern(2, 1, 1, 640, 480), t)]
    ctx.profile(True)
    a.batched_step(views, (0, 0, 0), 2, 1, 100, 800.0, buckets=4)
    tl = ctx.pipeline_timeline()
    ctx.profile(False)
    assert tl.shape == (4, 6)
    for b in range(4):
        cs, ce, ars, are, ads, ade = tl[b]
        assert cs <= ce <= ars + 1e-3 and ars <= are <= ads + 1e-3 and ads <= ade
        if b + 1 < 4:
            assert tl[b + 1][0] >= ce - 1e-3     # chains in order on the compute stream
    print("\npipeline timeline (ms):\n", np.array2string(tl, precision=4))
