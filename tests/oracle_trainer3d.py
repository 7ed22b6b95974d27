"""TEST INFRASTRUCTURE — the 3-D fit loop (tgsx_trainer3d_*, csrc/trainer.cpp) restated over the
FP64 3-D oracle (oracle/ewa3d.c render / backward / Adam / densify3d), step for step: same view
and offset order, same RNG draw order, same budget feeding, same statistics (screen-space
position norm, SH-DC colour-gradient norm, visits), same Adam step numbering."""
import numpy as np

from oracle import bind as B


def oracle_train3d(params, cams, targets, cfg, extent, iters):
    n0 = params.shape[1]
    st = {"params": np.ascontiguousarray(params, np.float32).copy(), "m1": np.zeros((59, n0), np.float32),
          "m2": np.zeros((59, n0), np.float32), "pos_acc": np.zeros(n0, np.float32),
          "col_acc": np.zeros(n0, np.float32), "visit": np.zeros(n0, np.int32), "visit_evt": np.zeros(n0, np.int32),
          "visit_aud": np.zeros(n0, np.int32), "ids": np.arange(n0, dtype=np.uint64), "tau_v": np.full(n0, 5.0),
          "next_id": n0}
    rng = B.Pcg32(cfg.seed, 1)
    m_final = cfg.m_final if cfg.m_final > 0 else 1.5 * n0
    budget = B.Budget(float(n0), float(m_final))
    dcfg = B.densify_config(cfg.densify.tau_pos)
    dcfg.color_branch_prob = cfg.densify.color_branch_prob
    bg = tuple(cfg.background)
    p, nv = cfg.dilation_p, len(cams)
    final_start = cfg.total_iters - cfg.batch_final_iters
    adam_t = 0
    losses, events = [], []

    def view(cam, tg, pp, ox, oy, lam):
        W, H = cam.width, cam.height
        rgb = B.render3d(st["params"], cam, pp, ox, oy, bg)[0]
        loss, dl = B.loss(rgb, pp, ox, oy, W, H, tg, lam)
        g, scr, _ = B.backward3d(st["params"], cam, pp, ox, oy, dl, bg)
        vis = scr[9] > 0
        pn = np.sqrt(scr[0] * scr[0] + scr[1] * scr[1]).astype(np.float32)
        cn = np.sqrt(np.sum(g[11:14].astype(np.float32) ** 2, axis=0)).astype(np.float32)
        return loss, g, vis, pn, cn

    for t in range(1, iters + 1):
        if t > final_start and cfg.batch_size > 1:
            gsum = np.zeros_like(st["params"])
            loss0 = None
            for b in range(cfg.batch_size):
                k = (t - 1) * cfg.batch_size + b
                idx = k % (p * p)
                loss, g, vis, pn, cn = view(cams[k % nv], targets[k % nv], p, idx % p, idx // p, 0.0)
                loss0 = loss if loss0 is None else loss0
                gsum += g
                st["pos_acc"][vis] += pn[vis]
                st["col_acc"][vis] += cn[vis]
                st["visit"][vis] += 1
            adam_t += 1
            g = np.ascontiguousarray((gsum / np.float32(cfg.batch_size)).astype(np.float32))
            B.adam3d_step(st["params"], g, st["m1"], st["m2"], B.adam3d_config(adam_t, cfg.total_iters, extent))
            loss = loss0
        else:
            dilate = True
            if t > cfg.densify_until:
                dilate = rng.uniform() < float(np.float32(cfg.post_densify_dilation_prob))
            pp = p if dilate else 1
            idx = ((t - 1) // nv) % (pp * pp)
            lam = float(np.float32(cfg.ssim_weight)) if pp == 1 else 0.0
            loss, g, vis, pn, cn = view(cams[(t - 1) % nv], targets[(t - 1) % nv], pp, idx % pp, idx // pp, lam)
            st["pos_acc"][vis] += pn[vis]
            st["col_acc"][vis] += cn[vis]
            st["visit"][vis] += 1
            adam_t += 1
            B.adam3d_step(st["params"], np.ascontiguousarray(g), st["m1"], st["m2"],
                          B.adam3d_config(adam_t, cfg.total_iters, extent))
        losses.append(loss)
        if loss > 0:
            budget.record_loss(t, float(np.float32(loss)))
        if cfg.warmup_iters < t <= cfg.densify_until and t % cfg.densify_interval == 0:
            budget.update(t)
            Bt = budget.budget_at(B.budget_t_norm(t, cfg.warmup_iters, cfg.densify_until))
            st, (sp, pr, _, _) = B.densify3d_event(st, dcfg, Bt, rng)
            events.append((t, Bt, st["params"].shape[1], sp, pr))
        if cfg.n_views > 0 and t % cfg.n_views == 0:
            st["tau_v"], st["visit_aud"] = B.visit_audit3d(st)
    return st, np.array(losses), events
