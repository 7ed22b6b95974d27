"""Debug: GPU trainer vs reference schedule at 4K — stats before the second densify event."""
import os, sys, math
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import bind as B
from tests.helpers import model_from_scene, scene_from_model
from tests.oracle_trainer import oracle_train
import paper_2412_13547_b200 as P

B.set_math(True)
W, H, N = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
threads = os.cpu_count()
s = B.synthetic_scene(1, N, W, H)
clean = B.render(B.synthetic_scene(2, 2 * N, W, H), 1, 0, 0, W, H, impl="ref_cr", threads=threads)[0].reshape(H, W, 3)
rng = np.random.default_rng(0)
targets = [np.clip(clean + rng.normal(0, 0.02, clean.shape), 0, 1).astype(np.float32) for _ in range(2)]
cfg = P.train_config(total_iters=160, warmup_iters=40, densify_interval=20, densify_until=120,
                     batch_final_iters=16, batch_size=4, dilation_p=2, n_views=2, m_final=1.5 * N, seed=7)
cfg.densify.tau_pos = float(sys.argv[4]) if len(sys.argv) > 4 else 1.2e-7
snaps = {}
def on_iter(t, st):
    if t in (59, 60, 61, 79):
        snaps[t] = st.copy()
    if t == 79:
        raise StopIteration
try:
    oracle_train(s, targets, cfg, W, H, 79, on_iter=on_iter, impl="ref_cr", threads=threads)
except StopIteration:
    pass
ctx = P.Context(0)
dm = P.DeviceModel.from_host(model_from_scene(s), ctx)
tr = P.Trainer(dm, W, H, cfg)
tr.set_targets(targets)
gs = {}
for t in range(1, 80):
    rep = tr.step()
    if rep.densified:
        print("gpu event", t, rep.budget, rep.count, rep.spawned, rep.pruned)
    if t in (59, 60, 61, 79):
        gs[t] = dm.download()
def summ(name, m):
    d = {}
    for f in ("pos_acc", "col_acc", "accum", "visit", "window", "tau_v"):
        pass
    return d
for t in (59, 60, 61, 79):
    o = snaps[t]; g = gs[t]
    print("t", t, "n", o.n, g.size())
    for of, gf in (("pos_acc", "pos_grad_norm_accum"), ("col_acc", "color_grad_norm_accum"), ("accum", "accum_count"),
                   ("visit", "visit_count"), ("window", "window_visit_count"), ("tau_v", "visit_thresholds")):
        a = np.asarray(getattr(o, of), np.float64); b = np.asarray(getattr(g, gf), np.float64)
        k = min(len(a), len(b))
        print(f"  {of:8s} oracle mean {a.mean():.4g} p50 {np.percentile(a,50):.4g} p99 {np.percentile(a,99):.4g} | gpu mean {b.mean():.4g} p50 {np.percentile(b,50):.4g} p99 {np.percentile(b,99):.4g} | equal {np.mean(a[:k]==b[:k]):.4f}")
    po = np.stack([getattr(o, f) for f in ("px", "py", "rot", "lsx", "lsy", "rop", "cr", "cg", "cb", "depth")]); pg = np.asarray(g.params)
    k = min(po.shape[1], pg.shape[1])
    print("  params max abs diff per row", np.abs(po[:, :k] - pg[:, :k]).max(axis=1))
    print("  ids equal", np.array_equal(np.asarray(o.id)[:k], np.asarray(g.id)[:k]))
