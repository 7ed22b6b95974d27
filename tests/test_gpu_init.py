"""Initializer on the device: the grid-hash kNN equals the reference
KdTree2<float>::knn (kdtree.hpp:30-38) exactly — order, ties and duplicates included — and
kdtree_upsample / init_model meet the SPEC's examples."""
import numpy as np
import pytest

from oracle import bind as B

pytestmark = pytest.mark.gpu

IMPL = "ref_native" if B.ref_available() else "brute"


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def _sets():
    rng = np.random.default_rng(21)
    g = np.stack(np.meshgrid(np.arange(40), np.arange(30)), -1).reshape(-1, 2).astype(np.float32)
    centers = rng.uniform(0, 1000, (12, 2))
    clustered = np.concatenate([c + rng.normal(0, 0.5, (300, 2)) for c in centers]).astype(np.float32)
    line = np.stack([np.arange(500) * 0.25, np.full(500, 3.0)], 1).astype(np.float32)
    dup = np.concatenate([g[:200], g[:200], g[100:300]])
    return {"random": rng.uniform(0, 1920, (20000, 2)).astype(np.float32),
            "grid_ties": g * np.float32(1.3),
            "clustered": clustered,
            "collinear": line,
            "duplicates": dup,
            "pair": np.array([[5, 5], [6, 7]], np.float32),
            "single": np.array([[1, 1]], np.float32)}


@pytest.mark.parametrize("name", list(_sets()))
@pytest.mark.parametrize("k", [1, 3, 8])
def test_knn_matches_reference_kdtree(P, ctx, name, k):
    xy = _sets()[name]
    idx, d2 = P.knn(ctx, xy, k)
    want = B.knn(xy, k, IMPL) if len(xy) <= 5000 or IMPL != "brute" else None
    if want is None:
        pytest.skip("reference KD-tree not built")
    assert np.array_equal(idx, want)
    ok = idx != 0xFFFFFFFF
    j = np.where(ok, idx, 0).astype(np.int64)
    dx = (xy[:, None, 0] - xy[j, 0]).astype(np.float32)
    dy = (xy[:, None, 1] - xy[j, 1]).astype(np.float32)
    ref_d2 = (dx * dx).astype(np.float32) + (dy * dy).astype(np.float32)
    assert np.array_equal(d2[ok], ref_d2[ok])
    assert np.all(np.isinf(d2[~ok]))


def test_knn_large(P, ctx):
    """200k points at bench scale (a 1920x1080 seed cloud), against the reference KD-tree."""
    if IMPL == "brute":
        pytest.skip("reference KD-tree not built")
    xy = np.random.default_rng(5).uniform(0, [1920, 1080], (200000, 2)).astype(np.float32)
    idx, _ = P.knn(ctx, xy, 3)
    assert np.array_equal(idx, B.knn(xy, 3, IMPL))


def test_upsample_two_points(P, ctx):
    xy = np.array([[1, 2], [4, 8]], np.float32)
    rgb = np.array([[0, 0, 1], [1, 0.5, 0]], np.float32)
    oxy, orgb = P.kdtree_upsample(ctx, xy, rgb, 1)
    assert oxy.shape == (3, 2)
    assert np.array_equal(oxy[2], [2.5, 5.0]) and np.array_equal(orgb[2], [0.5, 0.25, 0.5])
    oxy0, orgb0 = P.kdtree_upsample(ctx, xy, rgb, 0)
    assert np.array_equal(oxy0, xy) and np.array_equal(orgb0, rgb)
    one, _ = P.kdtree_upsample(ctx, xy[:1], rgb[:1], 3)
    assert np.array_equal(one, xy[:1])  # < 2 points: unchanged


def test_upsample_random_bruteforce(P, ctx):
    """SPEC example: every inserted point is the midpoint of some input pair that are
    (mutual or one-way) nearest neighbours (O(n^2) oracle); count at most doubles; superset."""
    rng = np.random.default_rng(7)
    xy = rng.uniform(0, 100, (100, 2)).astype(np.float32)
    rgb = rng.uniform(0, 1, (100, 3)).astype(np.float32)
    oxy, orgb = P.kdtree_upsample(ctx, xy, rgb, 1)
    assert np.array_equal(oxy[:100], xy) and np.array_equal(orgb[:100], rgb)
    assert 100 < len(oxy) <= 200
    nn = B.knn(xy, 1, "brute")[:, 0]
    pairs = sorted({(min(i, int(j)), max(i, int(j))) for i, j in enumerate(nn)})
    mids = np.array([(xy[a] + xy[b]) * np.float32(0.5) for a, b in pairs], np.float32)
    cols = np.array([(rgb[a] + rgb[b]) * np.float32(0.5) for a, b in pairs], np.float32)
    assert np.array_equal(oxy[100:], mids) and np.array_equal(orgb[100:], cols)


def test_upsample_dedupes_and_rounds(P, ctx):
    # duplicate input points: their midpoint is an existing position and is skipped
    xy = np.array([[0, 0], [0, 0], [5, 5]], np.float32)
    oxy, _ = P.kdtree_upsample(ctx, xy, np.zeros((3, 3), np.float32), 1)
    assert np.array_equal(oxy, np.array([[0, 0], [0, 0], [5, 5], [2.5, 2.5]], np.float32))
    rng = np.random.default_rng(8)
    pts = rng.uniform(0, 50, (64, 2)).astype(np.float32)
    cur = pts
    for r in range(1, 4):
        nxt, _ = P.kdtree_upsample(ctx, pts, np.zeros((64, 3), np.float32), r)
        assert len(cur) < len(nxt) <= 2 * len(cur) and np.array_equal(nxt[:len(cur)], cur)
        assert len({tuple(p) for p in nxt.tolist()}) == len(nxt)
        cur = nxt
    with pytest.raises(Exception):
        P.kdtree_upsample(ctx, pts, np.zeros((64, 3), np.float32), 1, capacity=65)


def test_init_model_grid_spacing(P, ctx):
    """SPEC example: a regular grid with spacing s gives every interior Gaussian scale s
    (within 1e-6); every scale equals the mean 3-NN distance of the reference KD-tree."""
    s = 2.5
    g = np.stack(np.meshgrid(np.arange(20), np.arange(15)), -1).reshape(-1, 2).astype(np.float32) * np.float32(s)
    rgb = np.random.default_rng(3).uniform(0, 1, (len(g), 3)).astype(np.float32)
    dm = P.DeviceModel(ctx, 1)
    P.init_model(dm, g, rgb, 80, 60, seed=1)
    m = dm.download()
    assert m.size() == len(g)
    scale = np.exp(m.row("lsx").astype(np.float64))
    assert np.array_equal(m.row("lsx"), m.row("lsy"))
    gx, gy = g[:, 0] / s, g[:, 1] / s
    interior = (gx > 0) & (gx < 19) & (gy > 0) & (gy < 14)
    assert np.allclose(scale[interior], s, rtol=1e-6)
    # the mean in double of sqrt of the float dist2 (dx*dx + dy*dy, unfused float)
    nn = B.knn(g, 3, IMPL).astype(np.int64)
    dx = (g[:, None, 0] - g[nn, 0]).astype(np.float32)
    dy = (g[:, None, 1] - g[nn, 1]).astype(np.float32)
    d2 = (dx * dx).astype(np.float32) + (dy * dy).astype(np.float32)
    d = (np.sqrt(d2[:, 0].astype(np.float64)) + np.sqrt(d2[:, 1].astype(np.float64))
         + np.sqrt(d2[:, 2].astype(np.float64))) / 3.0
    assert np.array_equal(m.row("lsx"), np.log(d).astype(np.float32))
    # activated opacity 0.1, rotation 0, activated colour = sampled colour
    assert np.allclose(1 / (1 + np.exp(-m.row("rop").astype(np.float64))), 0.1, rtol=1e-6)
    assert np.all(m.row("rot") == 0)
    col = 1 / (1 + np.exp(-np.stack([m.row("cr"), m.row("cg"), m.row("cb")], 1).astype(np.float64)))
    assert np.allclose(col, np.clip(rgb, 1e-4, 1 - 1e-4), atol=1e-6)
    assert len(np.unique(m.row("depth"))) == len(g)
    assert np.array_equal(m.id, np.arange(len(g), dtype=np.uint64))


def test_init_model_single_point_and_render(P, ctx):
    dm = P.DeviceModel(ctx, 1)
    P.init_model(dm, np.array([[10, 20]], np.float32), np.array([[0.2, 0.4, 0.6]], np.float32), 64, 48)
    m = dm.download()
    assert m.size() == 1 and m.row("px")[0] == 10 and m.row("py")[0] == 20
    assert m.row("lsx")[0] == np.float32(np.log(np.hypot(64, 48) / 16))
    with pytest.raises(Exception):
        P.init_model(dm, np.zeros((0, 2), np.float32), np.zeros((0, 3), np.float32), 64, 48)
    # seed -> upsample -> init -> render: non-degenerate, finite
    img = np.random.default_rng(2).uniform(0, 1, (48, 64, 3)).astype(np.float32)
    xy, rgb = P.sample_seed_points(img, 300, seed=2)
    xy, rgb = P.kdtree_upsample(ctx, xy, rgb, 1)
    P.init_model(dm, xy, rgb, 64, 48, seed=2)
    out = dm.render(P.DilationPattern(1, 0, 0, 64, 48))
    assert np.isfinite(out.colors).all() and (out.final_transmittance < 1).any()
