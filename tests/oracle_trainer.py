"""TEST INFRASTRUCTURE — the fit-loop schedule restated over the CPU oracle,
mirroring paper_2412_13547_b200/csrc/trainer.cpp step for step (same RNG draw order, same
budget feeding, same Adam step numbering) so trajectories can be compared with the GPU trainer."""
import math

import numpy as np

from oracle import bind as B


def oracle_train(s, targets, cfg, W, H, iters, on_iter=None, impl="oracle", threads=1, rng_sync=None):
    """impl="ref_cr": render / backward by the unmodified reference compiled in oracle/_ref (CR
    libm build, bit-exact with the restatement) on `threads` host threads — for large views.
    rng_sync: {iteration t: (state, inc)} PCG32 state adopted at the start of iteration t (the
    state another run of the schedule had there), so both runs draw the same coins / jitter even
    after their spawn counts differ by a few Gaussians."""
    s = s.copy().ensure_stats()
    kw = {"impl": impl, "threads": threads}
    n0 = s.n
    rng = B.Pcg32(cfg.seed, 1)
    m_final = cfg.m_final if cfg.m_final > 0 else 1.5 * n0
    budget = B.Budget(float(n0), float(m_final))
    dcfg = B.densify_config(cfg.densify.tau_pos)
    m1 = np.zeros((9, n0), np.float32)
    m2 = np.zeros((9, n0), np.float32)
    diag = math.hypot(W, H)
    bg = tuple(cfg.background)
    p = cfg.dilation_p
    adam_t = 0
    final_start = cfg.total_iters - cfg.batch_final_iters
    losses, events = [], []
    for t in range(1, iters + 1):
        if rng_sync and t in rng_sync:
            rng.set_state(rng_sync[t])
        if t > final_start and cfg.batch_size > 1:
            gsum = np.zeros((9, s.n), np.float32)
            loss0 = None
            for b in range(cfg.batch_size):
                idx = ((t - 1) * cfg.batch_size + b) % (p * p)
                ox, oy = idx % p, idx // p
                tg = targets[((t - 1) * cfg.batch_size + b) % len(targets)]
                rgb = B.render(s, p, ox, oy, W, H, bg, **kw)[0]
                loss, dl = B.l1_loss(rgb, p, ox, oy, W, H, tg)
                loss0 = loss if loss0 is None else loss0
                g, _ = B.backward(s, p, ox, oy, W, H, dl, bg, **kw)
                gsum += g
            adam_t += 1
            B.adam_step(s, (gsum / np.float32(cfg.batch_size)).astype(np.float32), m1, m2,
                        B.adam_config(adam_t, cfg.total_iters, diag))
            loss = loss0
        else:
            dilate = True
            if t > cfg.densify_until:
                dilate = rng.uniform() < float(np.float32(cfg.post_densify_dilation_prob))
            pp = p if dilate else 1
            idx = (t - 1) % (pp * pp)
            ox, oy = idx % pp, idx // pp
            rgb = B.render(s, pp, ox, oy, W, H, bg, **kw)[0]
            # compute_loss: dense iterations add the SSIM term
            loss, dl = B.loss(rgb, pp, ox, oy, W, H, targets[(t - 1) % len(targets)],
                              float(np.float32(cfg.ssim_weight)) if pp == 1 else 0.0)
            g, _ = B.backward(s, pp, ox, oy, W, H, dl, bg, **kw)
            adam_t += 1
            B.adam_step(s, g, m1, m2, B.adam_config(adam_t, cfg.total_iters, diag))
        losses.append(loss)
        if loss > 0:
            budget.record_loss(t, float(np.float32(loss)))
        if cfg.warmup_iters < t <= cfg.densify_until and t % cfg.densify_interval == 0:
            budget.update(t)
            Bt = budget.budget_at(B.budget_t_norm(t, cfg.warmup_iters, cfg.densify_until))
            s, sp, pr, nc, (m1, m2) = B.densify_event(s, s.n + max(0, Bt - s.n) + 8, dcfg, Bt, rng, m1, m2)
            events.append((t, Bt, s.n, sp, pr))
        if cfg.n_views > 0 and t % cfg.n_views == 0:
            B.visit_audit(s)
        if on_iter:
            on_iter(t, s)
    return s, np.array(losses), events
