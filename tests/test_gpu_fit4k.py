"""A full Turbo-GS fit at 4K (north_star: "a full 4K synthetic-scene Turbo-GS fit matching
reference quality within tolerance"; SPEC.md:572-580 schedule, SPEC.md:675/678 acceptance):
the GPU trainer (warm-up -> densify every 20 iterations under the convergence-aware budget ->
post-densify random dilation with dense L1 + SSIM iterations -> batched-view finale) against the
same schedule over the CPU reference (tests/oracle_trainer.py, render / backward by the
unmodified reference in oracle/_ref on all host threads). Reduced Gaussian count (30K) so the
CPU side finishes in about a minute; the view is the full 3840x2160.

Tolerances (FP32 order differences grow along a 160-iteration trajectory, so the comparison is
statistical; the reference run adopts the GPU run's RNG state so both draw the same coins): first
densify event at the same iteration and budget with its count within 1 %; every event within 3 %
of the reference's count and budget; budget compliance at every event on both sides; the last
20 losses within 3 %; final PSNR against the clean scene within 0.05 dB of the reference's."""
import math
import os

import numpy as np
import pytest

from oracle import bind as B
from tests.helpers import model_from_scene
from tests.oracle_trainer import oracle_train

pytestmark = pytest.mark.gpu

W, H, N = 3840, 2160, 30_000


def _psnr(rgb, clean):
    mse = float(np.mean((rgb.reshape(-1, 3).astype(np.float64) - clean.reshape(-1, 3)) ** 2))
    return 10.0 * math.log10(1.0 / mse)


@pytest.mark.skipif(not B.ref_available(), reason="oracle/_ref not built")
def test_4k_fit_matches_reference_schedule():
    import paper_2412_13547_b200 as P
    B.set_math(True)
    threads = os.cpu_count() or 8
    s = B.synthetic_scene(1, N, W, H)
    clean = B.render(B.synthetic_scene(2, 2 * N, W, H), 1, 0, 0, W, H, impl="ref_cr", threads=threads)[0]
    clean = clean.reshape(H, W, 3)
    rng = np.random.default_rng(0)
    targets = [np.clip(clean + rng.normal(0, 0.02, clean.shape), 0, 1).astype(np.float32) for _ in range(2)]
    iters = 160
    cfg = P.train_config(total_iters=iters, warmup_iters=40, densify_interval=20, densify_until=120,
                         batch_final_iters=16, batch_size=4, dilation_p=2, n_views=2,
                         m_final=1.5 * N, seed=7)
    # SPEC's tau_pos = 2e-4 is calibrated for NDC-scale gradients; the per-pixel normalised L1 at
    # 4K gives mean position-gradient norms near 5e-8..2e-7 (~90th percentile after warm-up)
    cfg.densify.tau_pos = 1.2e-7
    cfg.ssim_weight = 0.2

    ctx = P.Context(0)
    dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
    tr = P.Trainer(dm, W, H, cfg)
    tr.set_targets(targets)
    events, rng_sync, chunks = [], {}, []
    for t in range(1, iters + 1):
        rng_sync[t] = tr.rng_state()
        rep = tr.step()
        if rep.densified:
            events.append((t, rep.budget, rep.count, rep.spawned, rep.pruned))
            assert rep.count <= rep.budget  # budget compliance (acceptance #8)
        if t % 20 == 0:  # the trainer keeps a ring of recent losses
            chunks.append(tr.losses(20))
    losses = np.concatenate(chunks)
    gpu_model = dm.download()

    # the reference run adopts the GPU run's PCG32 state at every iteration: spawning draws child
    # positions from it, so a few Gaussians' difference at one event would otherwise shift the
    # stream and flip every later coin — with the same draws the runs stay comparable
    os_, olosses, oevents = oracle_train(s, targets, cfg, W, H, iters, impl="ref_cr", threads=threads,
                                         rng_sync=rng_sync)
    assert len(events) == len(oevents) == (120 - 40) // 20
    # first event: same iteration and budget, spawn count within 1 % (borderline threshold
    # decisions flip under FP32 summation-order differences accumulated over 60 iterations)
    assert events[0][:2] == oevents[0][:2] and abs(events[0][2] - oevents[0][2]) <= 0.01 * oevents[0][2]
    assert sum(e[3] for e in events) > 0  # densification did real work
    for (t, Bt, cnt, sp, pr), (ot, oB, ocnt, osp, opr) in zip(events, oevents):
        assert t == ot and cnt <= Bt and ocnt <= oB
        assert abs(Bt - oB) <= max(2, 0.03 * oB) and abs(cnt - ocnt) <= max(3, 0.03 * ocnt), (events, oevents)
    assert np.allclose(losses[:40], olosses[:40], rtol=2e-3)
    assert abs(losses[-20:].mean() - olosses[-20:].mean()) <= 0.03 * olosses[-20:].mean()
    assert losses[-20:].mean() < losses[:20].mean()  # the fit makes progress

    # quality: both final models rendered by the same (reference) renderer at full resolution
    from tests.helpers import scene_from_model
    gs = scene_from_model(gpu_model)
    p_gpu = _psnr(B.render(gs, 1, 0, 0, W, H, impl="ref_cr", threads=threads)[0], clean)
    p_ref = _psnr(B.render(os_, 1, 0, 0, W, H, impl="ref_cr", threads=threads)[0], clean)
    p_init = _psnr(B.render(s, 1, 0, 0, W, H, impl="ref_cr", threads=threads)[0], clean)
    print(f"4K fit: PSNR init {p_init:.3f} dB, GPU {p_gpu:.3f} dB, reference schedule {p_ref:.3f} dB; "
          f"events GPU {events} ref {oevents}")
    assert p_gpu > p_init + 0.5
    assert abs(p_gpu - p_ref) <= 0.05
    dm.close()
    ctx.close()
