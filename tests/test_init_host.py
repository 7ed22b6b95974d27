"""Initializer host-side operations on CPU: sample_seed_points' KATs and
the seed-point file format. These entry points of libtgsx do no device work."""
import numpy as np
import pytest

import paper_2412_13547_b200 as P


def test_single_point_in_bounds():
    img = np.random.default_rng(0).uniform(0, 1, (7, 9, 3)).astype(np.float32)
    xy, rgb = P.sample_seed_points(img, 1, seed=5)
    assert xy.shape == (1, 2)
    assert 0 <= xy[0, 0] < 9 and 0 <= xy[0, 1] < 7
    px, py = int(xy[0, 0]), int(xy[0, 1])
    assert np.array_equal(rgb[0], img[py, px])


def test_deterministic_and_in_bounds():
    img = np.random.default_rng(1).uniform(0, 1, (40, 50, 3)).astype(np.float32)
    a = P.sample_seed_points(img, 500, seed=9)
    b = P.sample_seed_points(img, 500, seed=9)
    c = P.sample_seed_points(img, 500, seed=10)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    assert not np.array_equal(a[0], c[0])
    xy = a[0]
    assert (xy[:, 0] >= 0).all() and (xy[:, 0] < 50).all() and (xy[:, 1] >= 0).all() and (xy[:, 1] < 40).all()


def test_count_limits():
    img = np.zeros((4, 5, 3), np.float32)
    P.sample_seed_points(img, 20)  # count == W*H is allowed
    with pytest.raises(ValueError):
        P.sample_seed_points(img, 21)
    with pytest.raises(ValueError):
        P.sample_seed_points(img, 0)


def test_constant_image_importance_is_uniform():
    """Zero gradient everywhere: the importance half is uniform too (mean and quartiles of a
    uniform distribution over 10^4 draws)."""
    img = np.full((160, 160, 3), 0.4, np.float32)
    xy, rgb = P.sample_seed_points(img, 20000, seed=3)
    imp = xy[10000:]
    for ax in range(2):
        q = np.quantile(imp[:, ax], [0.25, 0.5, 0.75])
        assert np.allclose(q, [40, 80, 120], atol=3)
    assert np.all(rgb == np.float32(0.4))


def test_sharp_edge_attracts_importance_samples():
    """SPEC example: ≥ 60 % of the importance half within 2 px of a sharp vertical edge."""
    img = np.zeros((160, 160, 3), np.float32)
    img[:, 80:] = 1.0
    xy, _ = P.sample_seed_points(img, 20000, seed=4)
    imp = xy[10000:]
    near = np.abs(imp[:, 0] - 80.0) <= 2.0
    assert near.mean() >= 0.6
    uni = xy[:10000]
    assert np.abs(uni[:, 0] - 80.0).mean() > 20  # the uniform half is not drawn to the edge


def test_seed_point_file(tmp_path):
    p = tmp_path / "seeds.txt"
    p.write_text("1.5 2.5 0.1 0.2 0.3\n4 5 1 0 0.5\n")
    xy, rgb = P.load_seed_points(str(p))
    assert np.array_equal(xy, np.array([[1.5, 2.5], [4, 5]], np.float32))
    assert np.array_equal(rgb, np.array([[0.1, 0.2, 0.3], [1, 0, 0.5]], np.float32))
    p.write_text("1 2 3\n")
    with pytest.raises(ValueError):
        P.load_seed_points(str(p))
