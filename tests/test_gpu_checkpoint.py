"""TGS1 checkpoint: save -> load -> save is byte-identical (model, moments,
training state), the resumed fit continues exactly like the uninterrupted one, a truncated or
corrupt file is rejected, and an empty model is a 24-byte header + sections."""
import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import model_from_scene

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_2412_13547_b200 as P
    return P


@pytest.fixture(scope="module")
def ctx(P):
    return P.Context(0)


def _trainer(P, dm, W, H):
    cfg = P.train_config(total_iters=200, warmup_iters=20, densify_interval=10, densify_until=120,
                         batch_final_iters=10, batch_size=2, dilation_p=2, n_views=2, m_final=1600.0, seed=3)
    cfg.densify.tau_pos = 2e-5
    return P.Trainer(dm, W, H, cfg)


def test_round_trip_and_resume(P, ctx, tmp_path):
    W, H, n = 64, 48, 1000
    s = B.synthetic_scene(1, n, W, H)
    targets = [B.render(B.synthetic_scene(2, 800, W, H), 1, 0, 0, W, H)[0].reshape(H, W, 3)] * 2
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    tr = _trainer(P, dm, W, H)
    tr.set_targets(targets)
    for _ in range(45):  # through two densify events
        tr.step()
    a = str(tmp_path / "a.tgs")
    dm.save_checkpoint(a, tr)
    # restore into a fresh model + trainer, save again: identical bytes
    dm2 = P.DeviceModel.from_host(P.GaussianModel(0), ctx)
    tr2 = _trainer(P, dm2, W, H)
    tr2.set_targets(targets)
    dm2.load_checkpoint(a, tr2)
    b = str(tmp_path / "b.tgs")
    dm2.save_checkpoint(b, tr2)
    assert open(a, "rb").read() == open(b, "rb").read()
    # both continue identically (same losses, same model)
    for _ in range(30):
        r1, r2 = tr.step(), tr2.step()
        assert (r1.count, r1.budget, r1.densified) == (r2.count, r2.budget, r2.densified)
    assert np.array_equal(tr.losses(30), tr2.losses(30))
    h1, h2 = dm.download(), dm2.download()
    assert np.array_equal(h1.params, h2.params) and np.array_equal(h1.id, h2.id)


def test_corrupt_truncated_and_empty(P, ctx, tmp_path):
    W, H = 32, 32
    s = B.synthetic_scene(3, 200, W, H)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    path = tmp_path / "m.tgs"
    dm.save_checkpoint(str(path))
    data = path.read_bytes()
    assert data[:4] == b"TGS1" and int.from_bytes(data[8:16], "little") == 200
    assert len(data) == 24 + 156 * 200 + 4
    bad = tmp_path / "bad.tgs"
    for blob in (data[:-7], data[:30], b"TGS2" + data[4:], data + b"\0"):
        bad.write_bytes(blob)
        with pytest.raises(RuntimeError):
            dm.load_checkpoint(str(bad))
    empty = P.DeviceModel.from_host(P.GaussianModel(0), ctx)
    e = tmp_path / "e.tgs"
    empty.save_checkpoint(str(e))
    assert len(e.read_bytes()) == 24 + 4
    dm.load_checkpoint(str(e))
    assert dm.size() == 0
    dm.load_checkpoint(str(path))
    assert dm.size() == 200 and np.array_equal(dm.download().params[0], s.px)


def test_load_is_atomic(P, ctx, tmp_path):
    """A checkpoint whose trainer section is corrupt or truncated (or that has trailing bytes)
    is rejected BEFORE the caller's model or trainer changes (the load validates the whole file
    first)."""
    W, H, n = 64, 48, 600
    src = P.DeviceModel.from_host(model_from_scene(B.synthetic_scene(1, n, W, H)), ctx)
    targets = [B.render(B.synthetic_scene(2, 500, W, H), 1, 0, 0, W, H)[0].reshape(H, W, 3)] * 2
    tr = _trainer(P, src, W, H)
    tr.set_targets(targets)
    for _ in range(25):
        tr.step()
    path = tmp_path / "t.tgs"
    src.save_checkpoint(str(path), tr)
    data = path.read_bytes()
    model_end = 24 + 156 * src.size() + 4
    keep = B.synthetic_scene(5, 300, W, H)
    dst = P.DeviceModel.from_host(model_from_scene(keep), ctx)
    tr2 = _trainer(P, dst, W, H)
    tr2.set_targets(targets)
    tr2.step()
    before = tr2.losses(1).copy()
    px_before = dst.download().params[0].copy()
    for blob in (data[:model_end + 20], data[:-3], data + b"\x01\x02"):
        bad = tmp_path / "bad.tgs"
        bad.write_bytes(blob)
        with pytest.raises(RuntimeError):
            dst.load_checkpoint(str(bad), tr2)
        assert dst.size() == 300 and np.array_equal(dst.download().params[0], px_before)
        assert np.array_equal(tr2.losses(1), before)
    dst.load_checkpoint(str(path), tr2)
    assert dst.size() == src.size()
