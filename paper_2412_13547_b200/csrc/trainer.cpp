// The Turbo-GS fit loop (train(); trainer.cpp is missing from the reference so
// the schedule is the SPEC's) as native host orchestration over the device-resident fit path:
//
//   1..warmup                 dilated (p) with cycled offsets, optimise only
//   warmup..densify_until     + every densify_interval: budget update -> B(t_norm) -> densify
//                             (select / top-k cap / spawn / prune / reset) on the device
//   densify_until..final      no densification; dilated with probability
//                             post_densify_dilation_prob (one coin per iteration), else dense
//   last batch_final_iters    batch_size renders with distinct cycled offsets accumulated on the
//                             device, one Adam step on the mean
//   every n_views iterations  visit audit
// Targets are round-robined (multi-image fitting). RNG draw order per SPEC.md:604:
// offset coin -> colour coin -> spawn jitter (the last two inside tgsx_densify). Per-iteration
// losses stay on the device and are fed to the budget controller in order at each densify event
// (the controller only reads them there), so the loop never waits on a loss readback.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/tgsx.h"
#include "host_state.h"
#include <cuda_runtime.h>

struct tgsx_trainer {
    tgsx_ctx* ctx = nullptr;
    tgsx_model* m = nullptr;
    tgsx_train_config cfg{};
    int32_t W = 0, H = 0;
    tgsx_budget* budget = nullptr;
    uint64_t rng[2] = {0, 0};
    int64_t t = 0;                   // last completed iteration (1-based)
    int64_t adam_step = 0;
    int64_t n_init = 0;
    float* d_losses = nullptr;       // device ring of per-iteration losses
    int64_t ring = 0;
    int64_t fed = 0;                 // iterations already fed to the budget controller
    std::vector<float> h_losses;
    float* h_pinned = nullptr;
    double last_budget = 0;
    bool use_graph = true;           // TGSX_TRAINER_GRAPH=0: every step eager (A/B)
};

// The same schedule over a set of cameras of a 3-D model (tgsx_trainer3d_*).
struct tgsx_trainer3d {
    tgsx_ctx* ctx = nullptr;
    tgsx_model3d* m = nullptr;
    tgsx_train_config cfg{};
    std::vector<tgsx_camera> cams;
    double extent = 1.0;
    tgsx_budget* budget = nullptr;
    uint64_t rng[2] = {0, 0};
    int64_t t = 0;
    int64_t adam_step = 0;
    int64_t n_init = 0;
    float* d_losses = nullptr;
    int64_t ring = 0;
    int64_t fed = 0;
    float* h_pinned = nullptr;
    double last_budget = 0;
};

namespace {

template <typename TR>
int32_t feed_losses(TR* tr) {
    const int64_t pending = tr->t - tr->fed;
    if (pending <= 0) return TGSX_OK;
    // graph-replayed steps are verified first (a faulted one is re-run and rewrites its loss)
    if (int32_t rc = tgsx_synchronize(tr->ctx)) return rc;
    if (cudaMemcpyAsync(tr->h_pinned, tr->d_losses, sizeof(float) * tr->ring, cudaMemcpyDeviceToHost,
                        (cudaStream_t)tgsx_get_stream(tr->ctx)) != cudaSuccess)
        return TGSX_ECUDA;
    if (cudaStreamSynchronize((cudaStream_t)tgsx_get_stream(tr->ctx)) != cudaSuccess) return TGSX_ECUDA;
    for (int64_t it = tr->fed + 1; it <= tr->t; ++it) {
        const float l = tr->h_pinned[(it - 1) % tr->ring];
        if (l > 0.f) tgsx_budget_record_loss(tr->budget, it, (double)l);
    }
    tr->fed = tr->t;
    return TGSX_OK;
}

}  // namespace

extern "C" {

void tgsx_train_config_default(tgsx_train_config* c) {
    std::memset(c, 0, sizeof(*c));
    c->total_iters = 10000;       // SPEC.md:543 (paper scale)
    c->warmup_iters = 300;
    c->densify_interval = 20;
    c->densify_until = 3000;
    c->batch_final_iters = 50;
    c->batch_size = 4;
    c->dilation_p = 2;
    c->post_densify_dilation_prob = 0.5f;
    c->ssim_weight = 0.2f;                 // SPEC.md DESIGN DECISIONS (dense iterations only)
    c->n_views = 1;
    c->m_final = 0;               // 0 => 1.5 x initial count
    c->seed = 1;
    c->background[0] = c->background[1] = c->background[2] = 0.f;
    tgsx_densify_config_default(&c->densify);
}

int32_t tgsx_trainer_create(tgsx_ctx* ctx, tgsx_model* m, const tgsx_train_config* cfg,
                            int32_t width, int32_t height, tgsx_trainer** out) {
    if (!ctx || !m || !cfg || !out || width < 1 || height < 1) return TGSX_EINVAL;
    if (cfg->dilation_p < 1 || cfg->batch_size < 1 || cfg->densify_interval < 1) return TGSX_EINVAL;
    if (!(cfg->ssim_weight >= 0.f && cfg->ssim_weight <= 1.f)) return TGSX_EINVAL;
    if (!(cfg->warmup_iters <= cfg->densify_until && cfg->densify_until <= cfg->total_iters))
        return TGSX_EINVAL;  // SPEC.md:552 invariants
    tgsx_trainer* tr = new (std::nothrow) tgsx_trainer();
    if (!tr) return TGSX_ENOMEM;
    tr->ctx = ctx;
    tr->m = m;
    tr->cfg = *cfg;
    tr->W = width;
    tr->H = height;
    tr->n_init = tgsx_model_size(m);
    const double mf = cfg->m_final > 0 ? cfg->m_final : 1.5 * (double)tr->n_init;
    tgsx_budget_create((double)tr->n_init, mf, &tr->budget);
    // the budget never exceeds the adaptive maximum 1.5 M: reserve it up front so
    // densify events allocate nothing
    if (cfg->densify_until > cfg->warmup_iters) {
        const int32_t rc = tgsx_model_reserve(ctx, m, (int64_t)std::ceil(1.5 * mf) + 1024);
        if (rc) {
            tgsx_budget_destroy(tr->budget);
            delete tr;
            return rc;
        }
    }
    tgsx_pcg32_init(tr->rng, cfg->seed, 1);
    if (const char* e = std::getenv("TGSX_TRAINER_GRAPH")) tr->use_graph = std::strcmp(e, "0") != 0;
    tr->ring = std::max<int64_t>(cfg->densify_interval, 1) * 4 + 64;
    if (cudaMalloc(&tr->d_losses, sizeof(float) * tr->ring) != cudaSuccess ||
        cudaMallocHost(&tr->h_pinned, sizeof(float) * tr->ring) != cudaSuccess) {
        delete tr;
        return TGSX_ECUDA;
    }
    cudaMemset(tr->d_losses, 0, sizeof(float) * tr->ring);
    *out = tr;
    return TGSX_OK;
}

void tgsx_trainer_destroy(tgsx_trainer* tr) {
    if (!tr) return;
    if (tr->budget) tgsx_budget_destroy(tr->budget);
    if (tr->d_losses) cudaFree(tr->d_losses);
    if (tr->h_pinned) cudaFreeHost(tr->h_pinned);
    delete tr;
}

// One iteration. targets: n_targets device or host pointers to full-resolution W*H*3 RGB.
int32_t tgsx_trainer_step(tgsx_trainer* tr, const float* const* targets, int64_t n_targets,
                          tgsx_train_report* rep) {
    if (!tr || !targets || n_targets < 1) return TGSX_EINVAL;
    const tgsx_train_config& c = tr->cfg;
    const int64_t t = tr->t + 1;
    const float* bg = c.background;
    tgsx_train_report r{};
    r.iteration = t;
    const int64_t final_start = c.total_iters - c.batch_final_iters;
    float* dloss = tr->d_losses + (t - 1) % tr->ring;
    int32_t rc = TGSX_OK;
    const int p = c.dilation_p;
    if (t > final_start && c.batch_size > 1) {
        // batched finale: batch_size renders with distinct cycled offsets, mean, one Adam step
        for (int32_t b = 0; b < c.batch_size; ++b) {
            const int64_t idx = ((t - 1) * c.batch_size + b) % ((int64_t)p * p);
            tgsx_pattern pat{p, (int32_t)(idx % p), (int32_t)(idx / p), tr->W, tr->H};
            const float* tg = targets[((t - 1) * c.batch_size + b) % n_targets];
            if ((rc = tgsx_view_accumulate(tr->ctx, tr->m, &pat, bg, tg, b == 0 ? dloss : nullptr)))
                return rc;
        }
        tgsx_adam_args a{++tr->adam_step, c.total_iters, std::hypot((double)tr->W, (double)tr->H)};
        if ((rc = tgsx_apply_step(tr->ctx, tr->m, c.batch_size, &a))) return rc;
        r.dilated = 1;
    } else {
        int dilate = 1;
        if (t > c.densify_until) {  // offset coin (SPEC.md:604 draw order)
            dilate = tgsx_pcg32_uniform(tr->rng) < (double)c.post_densify_dilation_prob;
        }
        const int pp = dilate ? p : 1;
        const int64_t idx = (t - 1) % ((int64_t)pp * pp);  // next_offsets (dilation.hpp:60-64)
        tgsx_pattern pat{pp, (int32_t)(idx % pp), (int32_t)(idx / pp), tr->W, tr->H};
        tgsx_adam_args a{++tr->adam_step, c.total_iters, std::hypot((double)tr->W, (double)tr->H)};
        // compute_loss: dense iterations add the SSIM term
        if ((rc = tgsx_set_ssim_weight(tr->ctx, pp == 1 ? c.ssim_weight : 0.f))) return rc;
        // While the model keeps its size (warm-up, and after the densification window) the step
        // is replayed from a CUDA graph, one per pattern (graph.cpp stages the view's target by a
        // node of the graph): the host only launches it. Inside the window every event resizes
        // the model and would force p^2 + 1 recaptures per event, so those steps run eagerly.
        const bool steady = t <= c.warmup_iters || t > c.densify_until;
        if (steady && (int64_t)p * p + 1 <= 12 && tr->use_graph)
            rc = tgsx_fit_graph_step(tr->ctx, tr->m, &pat, bg, targets[(t - 1) % n_targets], &a, dloss);
        else
            rc = tgsx_fit_step(tr->ctx, tr->m, &pat, bg, targets[(t - 1) % n_targets], &a, dloss);
        tgsx_set_ssim_weight(tr->ctx, 0.f);
        if (rc) return rc;
        r.dilated = dilate;
    }
    tr->t = t;
    // drain the device loss ring before it wraps (one small readback every ring/2 iterations)
    if (tr->t - tr->fed >= tr->ring / 2 && (rc = feed_losses(tr))) return rc;
    // densification phase (SPEC.md:575(3))
    if (t > c.warmup_iters && t <= c.densify_until && t % c.densify_interval == 0) {
        if ((rc = feed_losses(tr))) return rc;
        tgsx_budget_update(tr->budget, t);
        const double tn = tgsx_budget_t_norm(t, c.warmup_iters, c.densify_until);
        const int64_t B = tgsx_budget_at(tr->budget, tn);
        tgsx_densify_report dr{};
        if ((rc = tgsx_densify(tr->ctx, tr->m, &c.densify, B, tr->rng, &dr))) return rc;
        r.densified = 1;
        r.budget = B;
        r.spawned = dr.spawned;
        r.pruned = dr.pruned;
        tr->last_budget = (double)B;
    }
    if (c.n_views > 0 && t % c.n_views == 0) {
        if ((rc = tgsx_visit_audit(tr->ctx, tr->m))) return rc;
    }
    r.count = tgsx_model_size(tr->m);
    r.budget = r.budget ? r.budget : (int64_t)tr->last_budget;
    if (rep) *rep = r;
    return TGSX_OK;
}

// Per-iteration losses of the last min(ring, t) iterations (oldest first) + budget state.
int32_t tgsx_trainer_losses(tgsx_trainer* tr, float* out, int64_t max_out, int64_t* out_n) {
    if (!tr) return TGSX_EINVAL;
    if (feed_losses(tr)) return TGSX_ECUDA;
    const int64_t n = std::min<int64_t>(std::min<int64_t>(tr->t, tr->ring), max_out);
    for (int64_t k = 0; k < n; ++k) {
        const int64_t it = tr->t - n + 1 + k;
        out[k] = tr->h_pinned[(it - 1) % tr->ring];
    }
    if (out_n) *out_n = n;
    return TGSX_OK;
}

const tgsx_budget* tgsx_trainer_budget(const tgsx_trainer* tr) { return tr ? tr->budget : nullptr; }
int32_t tgsx_trainer_rng(const tgsx_trainer* tr, uint64_t out_state[2]) {
    if (!tr || !out_state) return TGSX_EINVAL;
    out_state[0] = tr->rng[0];
    out_state[1] = tr->rng[1];
    return TGSX_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- 3-D trainer
extern "C" {

int32_t tgsx_trainer3d_create(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_train_config* cfg,
                              const tgsx_camera* cams, int32_t n_cams, double scene_extent,
                              tgsx_trainer3d** out) {
    if (!ctx || !m || !cfg || !cams || n_cams < 1 || !out || !(scene_extent > 0)) return TGSX_EINVAL;
    if (cfg->dilation_p < 1 || cfg->batch_size < 1 || cfg->densify_interval < 1) return TGSX_EINVAL;
    if (!(cfg->ssim_weight >= 0.f && cfg->ssim_weight <= 1.f)) return TGSX_EINVAL;
    if (!(cfg->warmup_iters <= cfg->densify_until && cfg->densify_until <= cfg->total_iters)) return TGSX_EINVAL;
    for (int32_t v = 0; v < n_cams; ++v)
        if (cams[v].width < 1 || cams[v].height < 1) return TGSX_EINVAL;
    tgsx_trainer3d* tr = new (std::nothrow) tgsx_trainer3d();
    if (!tr) return TGSX_ENOMEM;
    tr->ctx = ctx;
    tr->m = m;
    tr->cfg = *cfg;
    tr->cams.assign(cams, cams + n_cams);
    tr->extent = scene_extent;
    tr->n_init = tgsx_model3d_size(m);
    const double mf = cfg->m_final > 0 ? cfg->m_final : 1.5 * (double)tr->n_init;
    tgsx_budget_create((double)tr->n_init, mf, &tr->budget);
    if (cfg->densify_until > cfg->warmup_iters) {
        const int32_t rc = tgsx_model3d_reserve(ctx, m, (int64_t)std::ceil(1.5 * mf) + 1024);
        if (rc) {
            tgsx_budget_destroy(tr->budget);
            delete tr;
            return rc;
        }
    }
    tgsx_pcg32_init(tr->rng, cfg->seed, 1);
    tr->ring = std::max<int64_t>(cfg->densify_interval, 1) * 4 + 64;
    if (cudaMalloc(&tr->d_losses, sizeof(float) * tr->ring) != cudaSuccess ||
        cudaMallocHost(&tr->h_pinned, sizeof(float) * tr->ring) != cudaSuccess) {
        tgsx_trainer3d_destroy(tr);
        return TGSX_ECUDA;
    }
    cudaMemset(tr->d_losses, 0, sizeof(float) * tr->ring);
    *out = tr;
    return TGSX_OK;
}

void tgsx_trainer3d_destroy(tgsx_trainer3d* tr) {
    if (!tr) return;
    if (tr->budget) tgsx_budget_destroy(tr->budget);
    if (tr->d_losses) cudaFree(tr->d_losses);
    if (tr->h_pinned) cudaFreeHost(tr->h_pinned);
    delete tr;
}

int32_t tgsx_trainer3d_step(tgsx_trainer3d* tr, const float* const* targets, int64_t n_targets,
                            tgsx_train_report* rep) {
    if (!tr || !targets || n_targets != (int64_t)tr->cams.size()) return TGSX_EINVAL;
    const tgsx_train_config& c = tr->cfg;
    const int64_t t = tr->t + 1;
    const int64_t nv = (int64_t)tr->cams.size();
    const float* bg = c.background;
    tgsx_train_report r{};
    r.iteration = t;
    const int64_t final_start = c.total_iters - c.batch_final_iters;
    float* dloss = tr->d_losses + (t - 1) % tr->ring;
    int32_t rc = TGSX_OK;
    const int p = c.dilation_p;
    if (t > final_start && c.batch_size > 1) {
        // batched finale: batch_size distinct cameras (cycled offsets), mean, one Adam step
        for (int32_t b = 0; b < c.batch_size; ++b) {
            const int64_t k = (t - 1) * c.batch_size + b;
            const tgsx_camera& cam = tr->cams[k % nv];
            const int64_t idx = k % ((int64_t)p * p);
            tgsx_pattern pat{p, (int32_t)(idx % p), (int32_t)(idx / p), cam.width, cam.height};
            if ((rc = tgsx_view_accumulate3d(tr->ctx, tr->m, &cam, &pat, bg, targets[k % nv], b == 0 ? dloss : nullptr)))
                return rc;
        }
        tgsx_adam3d_args a{++tr->adam_step, c.total_iters, tr->extent};
        if ((rc = tgsx_apply_step3d(tr->ctx, tr->m, c.batch_size, &a))) return rc;
        r.dilated = 1;
    } else {
        int dilate = 1;
        if (t > c.densify_until) dilate = tgsx_pcg32_uniform(tr->rng) < (double)c.post_densify_dilation_prob;
        const int pp = dilate ? p : 1;
        const tgsx_camera& cam = tr->cams[(t - 1) % nv];
        const int64_t idx = ((t - 1) / nv) % ((int64_t)pp * pp);  // offsets cycle per pass over the cameras
        tgsx_pattern pat{pp, (int32_t)(idx % pp), (int32_t)(idx / pp), cam.width, cam.height};
        tgsx_adam3d_args a{++tr->adam_step, c.total_iters, tr->extent};
        if ((rc = tgsx_set_ssim_weight(tr->ctx, pp == 1 ? c.ssim_weight : 0.f))) return rc;
        rc = tgsx_fit_step3d(tr->ctx, tr->m, &cam, &pat, bg, targets[(t - 1) % nv], &a, dloss);
        tgsx_set_ssim_weight(tr->ctx, 0.f);
        if (rc) return rc;
        r.dilated = dilate;
    }
    tr->t = t;
    if (tr->t - tr->fed >= tr->ring / 2 && (rc = feed_losses(tr))) return rc;
    if (t > c.warmup_iters && t <= c.densify_until && t % c.densify_interval == 0) {
        if ((rc = feed_losses(tr))) return rc;
        tgsx_budget_update(tr->budget, t);
        const double tn = tgsx_budget_t_norm(t, c.warmup_iters, c.densify_until);
        const int64_t B = tgsx_budget_at(tr->budget, tn);
        tgsx_densify_report dr{};
        if ((rc = tgsx_densify3d(tr->ctx, tr->m, &c.densify, B, tr->rng, &dr))) return rc;
        r.densified = 1;
        r.budget = B;
        r.spawned = dr.spawned;
        r.pruned = dr.pruned;
        tr->last_budget = (double)B;
    }
    if (c.n_views > 0 && t % c.n_views == 0) {
        if ((rc = tgsx_visit_audit3d(tr->ctx, tr->m))) return rc;
    }
    r.count = tgsx_model3d_size(tr->m);
    r.budget = r.budget ? r.budget : (int64_t)tr->last_budget;
    if (rep) *rep = r;
    return TGSX_OK;
}

int32_t tgsx_trainer3d_losses(tgsx_trainer3d* tr, float* out, int64_t max_out, int64_t* out_n) {
    if (!tr) return TGSX_EINVAL;
    if (feed_losses(tr)) return TGSX_ECUDA;
    const int64_t n = std::min<int64_t>(std::min<int64_t>(tr->t, tr->ring), max_out);
    for (int64_t k = 0; k < n; ++k) {
        const int64_t it = tr->t - n + 1 + k;
        out[k] = tr->h_pinned[(it - 1) % tr->ring];
    }
    if (out_n) *out_n = n;
    return TGSX_OK;
}

}  // extern "C"

// ---------------------------------------------------------------- checkpoint state
namespace tgsx {

void trainer_write(const tgsx_trainer* tr, ByteWriter& w) {
    w.put(tr->t);
    w.put(tr->adam_step);
    w.put(tr->n_init);
    w.put(tr->fed);
    w.put(tr->rng[0]);
    w.put(tr->rng[1]);
    w.put(tr->last_budget);
    // the device loss ring (losses not yet fed to the controller)
    std::vector<float> ring((size_t)tr->ring);
    cudaStream_t s = (cudaStream_t)tgsx_get_stream(tr->ctx);
    cudaMemcpyAsync(ring.data(), tr->d_losses, sizeof(float) * ring.size(), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    w.put(tr->ring);
    w.bytes(ring.data(), ring.size() * sizeof(float));
    budget_write(tr->budget, w);
}

TrainerState::~TrainerState() {
    if (budget) tgsx_budget_destroy(budget);
}

int32_t trainer_parse(const tgsx_trainer* tr, ByteReader& r, TrainerState& st) {
    if (!(r.get(st.t) && r.get(st.adam_step) && r.get(st.n_init) && r.get(st.fed) && r.get(st.rng[0]) &&
          r.get(st.rng[1]) && r.get(st.last_budget) && r.get(st.ring)))
        return TGSX_ERUNTIME;
    if (st.ring != tr->ring) return TGSX_ERUNTIME;  // trainer created with another densify interval
    st.losses.resize((size_t)st.ring);
    if (!r.bytes(st.losses.data(), st.losses.size() * sizeof(float))) return TGSX_ERUNTIME;
    st.budget = budget_clone(tr->budget);
    return budget_read(st.budget, r) ? TGSX_OK : TGSX_ERUNTIME;
}

int32_t trainer_commit(tgsx_trainer* tr, const TrainerState& st) {
    cudaStream_t s = (cudaStream_t)tgsx_get_stream(tr->ctx);
    if (cudaMemcpyAsync(tr->d_losses, st.losses.data(), sizeof(float) * st.losses.size(), cudaMemcpyHostToDevice, s) ||
        cudaStreamSynchronize(s))
        return TGSX_ECUDA;
    std::memcpy(tr->h_pinned, st.losses.data(), sizeof(float) * st.losses.size());
    tr->t = st.t;
    tr->adam_step = st.adam_step;
    tr->n_init = st.n_init;
    tr->fed = st.fed;
    tr->rng[0] = st.rng[0];
    tr->rng[1] = st.rng[1];
    tr->last_budget = st.last_budget;
    budget_assign(tr->budget, st.budget);
    return TGSX_OK;
}

}  // namespace tgsx
