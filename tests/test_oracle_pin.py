"""Pins the CPU oracle (oracle/tgs_oracle.c) to the reference (CPU, no GPU needed).

1. Against the committed golden fixtures (tests/golden/c1_small.npz, generated from the
   UNMODIFIED reference compiled into oracle/_ref by tests/golden/make_golden.py): bit-exact in
   both transcendental modes (CR interposer and glibc libm).
2. Against oracle/_ref itself on random / edge-case scenes when it is built (this container).
3. The reference's fp64 backward against central finite differences.
"""
import os

import numpy as np
import pytest

from oracle import bind as B

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def scene_from(d, prefix="scene_"):
    n = d[prefix + "px"].shape[0]
    s = B.Scene.empty(n)
    for f in B.ALL_FIELDS:
        setattr(s, f, np.array(d[prefix + f], np.float32))
    s.id = np.arange(n, dtype=np.uint64)
    s.next_id = n
    return s


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(GOLD, "c1_small.npz"))


@pytest.mark.parametrize("kind", ["cr", "native"])
def test_oracle_matches_golden(gold, kind):
    B.set_math(kind == "cr")
    s = scene_from(gold)
    W, H = int(gold["W"]), int(gold["H"])
    for tag, (p, ox, oy) in (("p1", (1, 0, 0)), ("p2", (2, 1, 0))):
        rgb, T, ops, _ = B.render(s, p, ox, oy, W, H, (0.1, 0.2, 0.3))
        assert np.array_equal(rgb, gold[f"{kind}_{tag}_rgb"])
        assert np.array_equal(T, gold[f"{kind}_{tag}_T"])
        assert ops == int(gold[f"{kind}_{tag}_ops"])
        s2 = s.copy().ensure_stats()
        g, _ = B.backward(s2, p, ox, oy, W, H, gold[f"{kind}_{tag}_dLdC"], (0.1, 0.2, 0.3))
        assert np.array_equal(g, gold[f"{kind}_{tag}_grads"])
        assert np.array_equal(s2.pos_acc, gold[f"{kind}_{tag}_pos_acc"])
        assert np.array_equal(s2.col_acc, gold[f"{kind}_{tag}_col_acc"])
        assert np.array_equal(s2.visit, gold[f"{kind}_{tag}_visit"])
    off, items = B.tile_grid(s, 1, W, H)
    assert np.array_equal(off, gold[f"{kind}_tiles_offsets"])
    assert np.array_equal(items, gold[f"{kind}_tiles_items"])
    prep = B.prepare(s, 1)
    for k, v in prep.items():
        assert np.array_equal(v, gold[f"{kind}_prep_{k}"]), k
    assert np.array_equal(B.sorted_order(s), gold["sorted_order"])
    B.set_math(True)


def test_golden_modes_differ_only_by_libm(gold):
    """The CR and native builds share all arithmetic; any difference is glibc rounding."""
    a, b = gold["cr_prep_alpha"], gold["native_prep_alpha"]
    assert np.abs(a - b).max() <= 2 ** -23
    assert np.array_equal(gold["cr_tiles_offsets"], gold["native_tiles_offsets"])


needs_ref = pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built (needs /root/reference)")


def _edge_scenes():
    yield "basic", B.synthetic_scene(3, 800, 77, 53), 77, 53
    s = B.synthetic_scene(4, 400, 64, 64)
    s.depth = np.round(s.depth * 4).astype(np.float32) / 4  # depth ties -> id order
    s.rop[::5] = 11.9                                       # near-opaque splats (sigma ~ 1)
    s.lsx[::7] = -6.0                                       # tiny splats
    yield "ties_opaque_tiny", s, 64, 64
    s = B.synthetic_scene(5, 300, 40, 33)
    s.px[::3] += 35.0                                       # partly off-image
    s.py[::4] -= 30.0
    yield "offimage", s, 40, 33
    yield "empty", B.synthetic_scene(6, 0, 17, 9), 17, 9
    yield "single_pixel", B.synthetic_scene(8, 20, 1, 1), 1, 1


@needs_ref
@pytest.mark.parametrize("cr", [True, False])
def test_oracle_vs_reference_edge_cases(cr):
    B.set_math(cr)
    impl = "ref_cr" if cr else "ref_native"
    rng = np.random.default_rng(0)
    for name, s, W, H in _edge_scenes():
        for p, ox, oy, lp in ((1, 0, 0, 0), (2, 1, 1, 0), (3, 2, 0, 0), (4, 1, 3, 0), (2, 0, 1, 1)):
            if ox >= W or oy >= H:
                continue
            a = B.render(s, p, ox, oy, W, H, (0.3, 0.0, 0.7), lowpass_p=lp)
            b = B.render(s, p, ox, oy, W, H, (0.3, 0.0, 0.7), lowpass_p=lp, impl=impl, threads=3)
            assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and a[2] == b[2], name
            dl = rng.normal(size=a[0].shape).astype(np.float32)
            dl[::3] = 0.0
            s1, s2 = s.copy().ensure_stats(), s.copy().ensure_stats()
            ga, _ = B.backward(s1, p, ox, oy, W, H, dl, (0.3, 0.0, 0.7), lowpass_p=lp)
            gb, _ = B.backward(s2, p, ox, oy, W, H, dl, (0.3, 0.0, 0.7), lowpass_p=lp, impl=impl, threads=2)
            assert np.array_equal(ga, gb), name
            assert np.array_equal(s1.pos_acc, s2.pos_acc) and np.array_equal(s1.visit, s2.visit)
    B.set_math(True)


@needs_ref
def test_oracle_errors_match_reference():
    s = B.synthetic_scene(1, 30, 16, 16)
    s.rot[4] = np.inf
    for impl in ("oracle", "ref_native"):
        with pytest.raises(B.OracleError) as e:
            B.render(s, 1, 0, 0, 16, 16, impl=impl)
        assert e.value.code == 1
    s = B.synthetic_scene(1, 30, 16, 16)
    s.lsx[2], s.lsy[2] = -60.0, 60.0
    for impl in ("oracle", "ref_native"):
        with pytest.raises(B.OracleError) as e:
            B.render(s, 1, 0, 0, 16, 16, impl=impl)
        assert e.value.code == 2
    with pytest.raises(B.OracleError):
        B.backward(B.synthetic_scene(1, 5, 8, 8), 1, 0, 0, 8, 8, np.zeros((3, 3), np.float32),
                   impl="ref_native")


@needs_ref
def test_reference_fp64_gradients_match_finite_differences():
    """SPEC.md:671 acceptance #1 (fp64 mode): backward vs central differences <= 1e-6 rel."""
    d = np.load(os.path.join(GOLD, "fd64.npz"))
    eps = 1e-6
    for i in range(5):
        s = scene_from(d, f"s{i}_").astype(np.float64)
        for p in (1, 2):
            dl = d[f"s{i}_p{p}_dLdC"]
            g = d[f"s{i}_p{p}_grads"]

            def loss(sc):
                rgb, _, _, _ = B.render(sc, p, 0, 0, 8, 8, (0.2, 0.3, 0.4), impl="ref_native", dtype=np.float64)
                return float((rgb * dl).sum())

            for q, f in enumerate(B.PARAM_FIELDS):
                for k in range(s.n):
                    sp, sm = s.copy(), s.copy()
                    getattr(sp, f)[k] += eps
                    getattr(sm, f)[k] -= eps
                    fd = (loss(sp) - loss(sm)) / (2 * eps)
                    assert abs(fd - g[q, k]) <= 1e-6 * max(1.0, abs(fd)) + 1e-7, (i, p, f, k)


def _knn_sets():
    rng = np.random.default_rng(11)
    g = np.stack(np.meshgrid(np.arange(12), np.arange(9)), -1).reshape(-1, 2).astype(np.float32)
    dup = np.concatenate([g[:20], g[:20], rng.uniform(0, 12, (30, 2)).astype(np.float32)])
    return {"random": rng.uniform(0, 500, (700, 2)).astype(np.float32),
            "grid_ties": g * np.float32(0.7),
            "duplicates": dup,
            "tiny": np.array([[1, 2], [3, 4]], np.float32)}


@needs_ref
@pytest.mark.parametrize("name", ["random", "grid_ties", "duplicates", "tiny"])
@pytest.mark.parametrize("k", [1, 3, 5])
def test_knn_restatement_matches_reference_kdtree(name, k):
    """The brute-force (dist2, index) restatement equals KdTree2<float>::knn (kdtree.hpp:30-38)
    exactly, ties and duplicate points included (SPEC: KD-tree queries agree with brute force)."""
    xy = _knn_sets()[name]
    assert np.array_equal(B.knn(xy, k, "brute"), B.knn(xy, k, "ref_native"))
