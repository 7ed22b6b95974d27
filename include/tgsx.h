/* tgsx — B200-native (sm_100a) Turbo-GS fit hot path, C ABI.
 *
 * This is the drop-in boundary for the reference's hot path. The reference
 * (a C++20 static library, /root/reference/proj/core) exposes the path as C++ templates; a
 * maintainer binds this ABI from C++ through the shim in paper_2412_13547_b200/shim/
 * (re-implements tgs::render<float> / tgs::backward<float> with the exact reference
 * signatures) or from any FFI (ctypes stub in INTEGRATION.md).
 *
 * Conventions
 *  - Every function returns int32 status: TGSX_OK or an error code; the message is available
 *    from tgsx_last_error(ctx). Error codes mirror the reference's exception types:
 *      TGSX_EINVAL   <-> std::invalid_argument (rasterizer.cpp:222-224, dilation.hpp:18-22,
 *                        gaussian.hpp:64-68)
 *      TGSX_ERUNTIME <-> std::runtime_error     (gaussian.hpp:84-86, degenerate covariance)
 *  - Pointer arguments documented "host or device" are resolved through CUDA unified virtual
 *    addressing: pass host memory (pinned for async copies) or device memory.
 *  - All work is enqueued on the context's stream; functions that return data to host memory
 *    synchronize that stream before returning. One context per host thread; a model may be
 *    used by one context at a time (the reference is likewise not re-entrant on one model,
 *    model.hpp:150-151).
 *  - Arrays are in MODEL (creation/index) order unless stated; "rank" arrays (per active
 *    pixel) follow the reference's dense rank (dilation.hpp:32, rasterizer.hpp:21-26).
 */
#ifndef TGSX_H
#define TGSX_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGSX_VERSION_MAJOR 0
#define TGSX_VERSION_MINOR 1

enum {
    TGSX_OK = 0,
    TGSX_EINVAL = 1,
    TGSX_ERUNTIME = 2,
    TGSX_ECUDA = 3,
    TGSX_ENOMEM = 4,
    TGSX_ESTATE = 5
};

typedef struct tgsx_ctx tgsx_ctx;
typedef struct tgsx_model tgsx_model;
typedef struct tgsx_budget tgsx_budget;

/* DilationPattern (dilation.hpp:14-56): pixel (x,y) active iff x%p==ox && y%p==oy. */
typedef struct {
    int32_t p, ox, oy, width, height;
} tgsx_pattern;

/* Host-side scene in model order: the SoA view of GaussianModel<float> (model.hpp:45-152,
 * Gaussian2D gaussian.hpp:35-44, DensifyStats model.hpp:17-40). Stats / tau_v pointers may be
 * NULL on upload (zeros / tau_v = 5.0) and are skipped on download when NULL. */
typedef struct {
    int64_t n;
    float *px, *py, *rot, *lsx, *lsy, *rop, *cr, *cg, *cb, *depth;
    uint64_t* id;
    uint64_t next_id;
    float *pos_acc, *col_acc;
    int32_t* accum;
    int64_t *visit, *window;
    double* tau_v;
} tgsx_host_scene;

/* ---------------------------------------------------------------- context */
int32_t tgsx_create(int32_t device, tgsx_ctx** out);
void tgsx_destroy(tgsx_ctx* ctx);
/* Replaces the context's stream (a cudaStream_t; NULL = the context's own stream). */
int32_t tgsx_set_stream(tgsx_ctx* ctx, void* stream);
void* tgsx_get_stream(tgsx_ctx* ctx);
const char* tgsx_last_error(const tgsx_ctx* ctx);
int32_t tgsx_synchronize(tgsx_ctx* ctx);
/* Page-locked host memory (cudaHostAlloc) for staging buffers a host caller reuses across calls:
 * copies from / to it run at full PCIe speed. */
int32_t tgsx_host_alloc(size_t bytes, void** out);
void tgsx_host_free(void* p);
/* Counters of this library's kernel launches on ctx (for the bench's gpu_launches claim). */
uint64_t tgsx_launch_count(const tgsx_ctx* ctx);
/* Live per-stage timing: CUDA events recorded on the context stream around each stage
 * (0 depth sort, 1 preprocess, 2 scan, 3 duplicate, 4 radix sort, 5 ranges, 6 blend forward,
 * 7 blend backward, 8 chain+stats+Adam, 9 loss reduce, 10 densify). Enabling resets totals. */
int32_t tgsx_profile(tgsx_ctx* ctx, int32_t enable);
/* Accumulated milliseconds and launch counts per stage (n entries). */
int32_t tgsx_profile_read(tgsx_ctx* ctx, double* ms, int64_t* counts, int32_t n);

/* ---------------------------------------------------------------- model (device SoA) */
/* Replaces GaussianModel<float> storage: params, ids, DensifyStats, tau_v (model.hpp:140-151)
 * plus Adam moments live in HBM for the model's lifetime. */
int32_t tgsx_model_create(tgsx_ctx* ctx, int64_t capacity, tgsx_model** out);
void tgsx_model_destroy(tgsx_model* m);
/* Grows the model's capacity (contents kept) and the context's per-Gaussian workspace to at
 * least `capacity` Gaussians, so densification up to that size allocates nothing (the
 * trainer reserves its maximal budget up front). */
int32_t tgsx_model_reserve(tgsx_ctx* ctx, tgsx_model* m, int64_t capacity);
int64_t tgsx_model_size(const tgsx_model* m);
uint64_t tgsx_model_next_id(const tgsx_model* m);
/* Upload replaces the whole model (moments zeroed, Adam step counter kept). */
int32_t tgsx_model_upload(tgsx_ctx* ctx, tgsx_model* m, const tgsx_host_scene* host);
/* Download copies params, ids, stats, tau_v into caller arrays sized >= tgsx_model_size. */
int32_t tgsx_model_download(tgsx_ctx* ctx, tgsx_model* m, tgsx_host_scene* host);
/* Adam moments, component-major [9][n] float, host or device destination. */
int32_t tgsx_model_download_moments(tgsx_ctx* ctx, tgsx_model* m, float* m1, float* m2);
int32_t tgsx_model_upload_moments(tgsx_ctx* ctx, tgsx_model* m, const float* m1, const float* m2);

/* ---------------------------------------------------------------- the reference's ops */
/* tgs::render<float> (rasterizer.hpp:58-60, rasterizer.cpp:144-184). out_rgb [P*3] and out_T
 * [P] by dense rank (host or device, may be NULL); *out_blend_ops (host, may be NULL).
 * lowpass_p = RenderOptions::lowpass_p (rasterizer.hpp:48-53; 0 = pattern p). */
int32_t tgsx_render(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                    int32_t lowpass_p, float* out_rgb, float* out_T, uint64_t* out_blend_ops);

/* tgs::backward<float> (rasterizer.hpp:66-69, rasterizer.cpp:218-361). dLdC [P*3] by rank
 * (host or device); dLdC_count = number of RGB entries, must equal the pattern's active count
 * (TGSX_EINVAL otherwise, rasterizer.cpp:222-224). out_grads component-major [9][n] (pos x, pos y, rot, ls x, ls y,
 * raw_opacity, r, g, b), host or device, may be NULL. Updates the model's DensifyStats in
 * place when update_stats != 0, like the reference (rasterizer.cpp:350-358). */
int32_t tgsx_backward(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                      int32_t lowpass_p, const float* dLdC, int64_t dLdC_count,
                      float* out_grads, int32_t update_stats);

/* ---------------------------------------------------------------- fit step (fused path) */
typedef struct {
    int64_t step;         /* 1-based Adam step t (bias correction) */
    int64_t total_steps;  /* position-LR decay horizon */
    double image_diagonal;
} tgsx_adam_args;

/* Adam + clamp_parameters (gaussian.hpp:105-116) with explicit
 * gradients [9][n] (host or device). */
int32_t tgsx_adam_step(tgsx_ctx* ctx, tgsx_model* m, const float* grads,
                       const tgsx_adam_args* a);

/* compute_loss (loss.cpp is missing from the reference): for a dense pattern
 * (p = 1) L = (1 - w) L1 + w (1 - SSIM) with the 11x11 Gaussian-window SSIM, for a dilated one
 * L1 over the active pixels. rgb: colours by rank (active_count x 3), target: full-resolution
 * W*H*3 (host or device). Writes the loss and dL/dC by rank (host or device, may be NULL).
 * EINVAL on a bad pattern or w outside [0, 1]. */
int32_t tgsx_loss(tgsx_ctx* ctx, const tgsx_pattern* pat, const float* rgb, const float* target,
                  float ssim_weight, float* out_loss, float* out_dLdC);
/* lambda_ssim of the fused fit views below on dense patterns (default 0: L1 only; the trainer
 * uses its config's value, SPEC.md DESIGN DECISIONS 0.2). */
int32_t tgsx_set_ssim_weight(tgsx_ctx* ctx, float ssim_weight);
/* Binning path: 0 (default) slab binning with per-tile sorts (2-D and 3-D), falling back to the
 * onesweep paths for lists longer than a slab; 1 always the onesweep paths (2-D: key
 * duplication + radix sort; 3-D: global depth sort + rank gather + onesweep). Both give identical
 * per-tile lists (tests compare them at full size). */
int32_t tgsx_set_binning(tgsx_ctx* ctx, int32_t mode);

/* One fused fit iteration on one view: render -> loss (L1 over active pixels; plus the SSIM
 * term on dense views when tgsx_set_ssim_weight > 0)
 * -> backward -> densify stats -> Adam. target: full-resolution W*H*3 float RGB, host or
 * device. A host target is copied on the context's copy stream into one of two staging
 * buffers, overlapping the previous call's kernels; the caller may reuse a pinned target
 * buffer after the next tgsx_synchronize (pageable buffers are consumed before returning).
 * *out_loss may be NULL, device, pinned host (written in stream order: read it after
 * tgsx_synchronize) or pageable host (written before returning).
 * Equivalent to render + L1 + backward + tgsx_adam_step with the same args. */
int32_t tgsx_fit_step(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                      const float* target, const tgsx_adam_args* a, float* out_loss);
/* tgsx_fit_step replayed from a CUDA graph: the first call with a given model
 * / pattern / background / target / loss pointer runs eagerly and captures the step; later
 * calls launch the graph (one launch, no host wait) with this call's Adam arguments. The
 * binning capacities are frozen at capture and checked on the device; a step that exceeds them
 * (or raises a kernel error) and its successor are re-run eagerly, so the model sequence is
 * exactly that of tgsx_fit_step. Steps are verified one call behind: errors of a replayed step
 * are returned by a later call (this, tgsx_synchronize or any call that touches the model), and
 * target / *out_loss must be device or pinned host memory that stays unchanged until the call
 * after next returns (other targets run eagerly). Not used while profiling is enabled. */
int32_t tgsx_fit_graph_step(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                            const float* target, const tgsx_adam_args* a, float* out_loss);
/* Graph statistics: captures, replayed launches, eager re-runs after a device-side fault. */
int32_t tgsx_fit_graph_stats(const tgsx_ctx* ctx, uint64_t* out_captures, uint64_t* out_replays,
                             uint64_t* out_reruns);

/* Batched views (SPEC.md:269-277 accumulate; multi-GPU view sharding):
 * tgsx_view_accumulate adds one view's gradients and densify-stat increments into the
 * model's per-step buffer (12 floats per Gaussian: 9 gradient sums, pos-norm sum,
 * colour-norm sum, visit count; the reference accumulates stats per backward call,
 * rasterizer.cpp:350-358). The buffer (device pointer, AoS [n][12] floats = exactly 48 B per
 * Gaussian, rows in the model's physical order) may be all-reduced across ranks before
 * tgsx_apply_step divides by batch_views, applies the stats and runs Adam.
 * tgsx_step_layout brings the rows to the canonical order every rank shares (the blend
 * order); a rank that accumulated no view of the step must call it before an external
 * all-reduce (the fused views already leave the rows there). */
int32_t tgsx_view_accumulate(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat,
                             const float bg[3], const float* target, float* out_loss);
float* tgsx_step_buffer(tgsx_model* m, int64_t* out_floats);
int32_t tgsx_step_layout(tgsx_ctx* ctx, tgsx_model* m);
int32_t tgsx_apply_step(tgsx_ctx* ctx, tgsx_model* m, int32_t batch_views,
                        const tgsx_adam_args* a);

/* ------------------------------------------------ in-library NCCL (view-batch DP, §8e)
 * Replaces the reference's `accumulate` over a batch when the batch is
 * sharded across GPUs: every rank holds the full model, renders its views, and the per-Gaussian
 * step buffer is summed with ONE NCCL all-reduce over NVLink (NVLS where NCCL enables it).
 * NCCL is dlopen'ed (libnccl.so.2: inside PyTorch, torch's own NCCL).
 * tgsx_comm_unique_id: rank 0 creates the 128-byte id, the caller distributes it;
 * tgsx_comm_init: attach a communicator of nranks to the context (its device);
 * tgsx_allreduce_step: in-place sum of the step buffer over the ranks (stream-ordered);
 * tgsx_batched_step: this rank's n_views views (pats[v], targets[v]; n_views may be 0) of a
 *   step of batch_views views in total -> step buffer -> all-reduce (if a communicator is
 *   attached) -> Adam over the mean + stats, with the last view's chain kernel, the all-reduce
 *   and Adam pipelined over `buckets` Gaussian ranges (chain(b) -> all-reduce(b) -> Adam(b)).
 *   out_losses[v] (may be NULL) as tgsx_fit_step's out_loss.
 * tgsx_pipeline_timeline: with profiling enabled, the last batched step's per-bucket event
 *   times in ms (chain start/end, all-reduce start/end, Adam start/end); returns the count. */
int32_t tgsx_comm_unique_id(uint8_t out_id[128]);
int32_t tgsx_comm_init(tgsx_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank);
int32_t tgsx_comm_destroy(tgsx_ctx* ctx);
int32_t tgsx_comm_size(const tgsx_ctx* ctx);
int32_t tgsx_allreduce_step(tgsx_ctx* ctx, tgsx_model* m);
int32_t tgsx_batched_step(tgsx_ctx* ctx, tgsx_model* m, int32_t n_views, const tgsx_pattern* pats,
                          const float bg[3], const float* const* targets, int32_t batch_views,
                          const tgsx_adam_args* a, float* out_losses, int32_t buckets);
int32_t tgsx_pipeline_timeline(tgsx_ctx* ctx, float* out, int32_t max_floats);

/* ---------------------------------------------------------------- densify */
typedef struct {
    float tau_pos;              /* 2e-4 default; tau_color = 0.01 * tau_pos */
    float opacity_mask_floor;   /* 0.05 */
    float opacity_prune_floor;  /* 0.005 */
    float color_branch_prob;    /* 0.2 */
    double tau_v_init;          /* 5 */
} tgsx_densify_config;

typedef struct {
    int64_t candidates, spawned, pruned, count_after;
    int32_t color_coin;
} tgsx_densify_report;

void tgsx_densify_config_default(tgsx_densify_config* c);
/* One densify event: colour coin -> select_candidates -> cap to budget - count (top-k by
 * averaged positional norm, ties by index) -> spawn -> prune -> reset accumulators.
 * rng_state[2] = PCG32 (state, inc) (rng.hpp:10-46), advanced in place exactly as the
 * sequential draw order would. */
int32_t tgsx_densify(tgsx_ctx* ctx, tgsx_model* m, const tgsx_densify_config* c,
                     int64_t budget, uint64_t rng_state[2], tgsx_densify_report* out);
/* update_visit_thresholds. */
int32_t tgsx_visit_audit(tgsx_ctx* ctx, tgsx_model* m);

/* ---------------------------------------------------------------- budget controller */
/* BudgetController, host scalar logic. */
int32_t tgsx_budget_create(double n_init, double m_final, tgsx_budget** out);
void tgsx_budget_destroy(tgsx_budget* b);
int32_t tgsx_budget_record_loss(tgsx_budget* b, int64_t t, double loss);
void tgsx_budget_update(tgsx_budget* b, int64_t t);
int64_t tgsx_budget_at(const tgsx_budget* b, double t_norm);
/* out[5] = alpha, alpha_base, m_adaptive, ema, number of fits */
void tgsx_budget_state(const tgsx_budget* b, double* out);
double tgsx_budget_t_norm(int64_t step, int64_t warmup, int64_t densify_end);
int32_t tgsx_fit_power_exponent(const double* t, const double* y, int64_t n, double* out);

/* ---------------------------------------------------------------- fit loop */
typedef struct tgsx_trainer tgsx_trainer;

/* TrainConfig. */
typedef struct {
    int64_t total_iters, warmup_iters, densify_interval, densify_until, batch_final_iters;
    int32_t batch_size;               /* renders per step in the batched finale (4) */
    int32_t dilation_p;               /* p of the dilated phases */
    float post_densify_dilation_prob; /* 0.5 */
    int64_t n_views;                  /* visit-audit period */
    double m_final;                   /* budget M (0 => 1.5 x initial count) */
    uint64_t seed;                    /* trainer PCG32 seed (stream 1) */
    float background[3];
    tgsx_densify_config densify;
    float ssim_weight;                /* lambda_ssim of dense iterations (0.2, SPEC.md DESIGN) */
} tgsx_train_config;

typedef struct {
    int64_t iteration, count, budget, spawned, pruned;
    int32_t densified, dilated;
} tgsx_train_report;

void tgsx_train_config_default(tgsx_train_config* c);
int32_t tgsx_trainer_create(tgsx_ctx* ctx, tgsx_model* m, const tgsx_train_config* cfg,
                            int32_t width, int32_t height, tgsx_trainer** out);
void tgsx_trainer_destroy(tgsx_trainer* tr);
/* One iteration of the schedule; targets[n_targets] = full-resolution W*H*3 RGB images (host
 * or device), round-robined. */
int32_t tgsx_trainer_step(tgsx_trainer* tr, const float* const* targets, int64_t n_targets,
                          tgsx_train_report* report);
/* Losses of the most recent iterations (oldest first), up to max_out. */
int32_t tgsx_trainer_losses(tgsx_trainer* tr, float* out, int64_t max_out, int64_t* out_n);
const tgsx_budget* tgsx_trainer_budget(const tgsx_trainer* tr);
/* The trainer's PCG32 state (state, inc): offset coin -> colour coin -> spawn jitter stream
 * (SPEC.md:604), e.g. to drive a reference run of the schedule with the same draws. */
int32_t tgsx_trainer_rng(const tgsx_trainer* tr, uint64_t out_state[2]);

/* ---------------------------------------------------------------- TGS1 checkpoint */
/* "TGS1", u32 version, u64 count, u64 next_id, the parameter arrays in declared field order,
 * ids, DensifyStats, Adam moments, then (when a trainer is given) the training state: iteration,
 * Adam step, RNG, loss ring, BudgetController. Load validates magic, version and lengths:
 * a corrupt or truncated file returns TGSX_ERUNTIME (the reference's corrupt-checkpoint
 * error); a file carrying training state needs a trainer (created with the same config).
 * Round trip: saving a loaded state reproduces the file byte for byte. */
int32_t tgsx_checkpoint_save(tgsx_ctx* ctx, tgsx_model* m, const tgsx_trainer* tr, const char* path);
int32_t tgsx_checkpoint_load(tgsx_ctx* ctx, tgsx_model* m, tgsx_trainer* tr, const char* path);

/* ---------------------------------------------------------------- initializer */
/* Exact k nearest neighbours (1 <= k <= 8) of every host point xy[n][2], self excluded, in
 * ascending (dist2, index) order: KdTree2<float>::knn (kdtree.hpp:30-38) for every point, on the
 * device (uniform-grid hash). Missing neighbours (n - 1 < k) are UINT32_MAX / +inf. out_d2 may
 * be null. */
int32_t tgsx_knn(tgsx_ctx* ctx, const float* xy, int64_t n, int32_t k, uint32_t* out_idx, float* out_d2);
/* sample_seed_points: count/2 uniform points, the rest importance-sampled on the image's
 * luminance-gradient magnitude (uniform for a flat image), jittered in their pixel; colours
 * read at the point's pixel. image = host W*H*3 RGB; PCG32 (seed, stream 2). */
int32_t tgsx_seed_points(const float* image, int32_t W, int32_t H, int64_t count, uint64_t seed,
                         float* out_xy, float* out_rgb);
/* kdtree_upsample: `rounds` times, append the midpoint of every unique {i, nearest(i)} pair
 * (ascending pair order, exact-duplicate positions skipped). Outputs hold up to capacity
 * points (TGSX_EINVAL when exceeded); *out_n = the final count. */
int32_t tgsx_upsample(tgsx_ctx* ctx, const float* xy, const float* rgb, int64_t n, int32_t rounds,
                      int64_t capacity, float* out_xy, float* out_rgb, int64_t* out_n);
/* init_model: one Gaussian per point; isotropic log-scale of the mean 3-NN distance (image
 * diagonal / 16 below 4 points), opacity 0.1, rotation 0, colour logit, PCG32 (seed, stream 3)
 * depth keys. Replaces m's contents. */
int32_t tgsx_init_model(tgsx_ctx* ctx, tgsx_model* m, const float* xy, const float* rgb, int64_t n,
                        int32_t W, int32_t H, uint64_t seed);

/* ---------------------------------------------------------------- utilities */
/* Seeded synthetic scene, written into caller host arrays (n entries). */
void tgsx_synthetic_scene(uint64_t seed, int64_t n, int32_t width, int32_t height,
                          tgsx_host_scene* out);
/* PCG32 (rng.hpp:10-46) helpers. */
void tgsx_pcg32_init(uint64_t state_out[2], uint64_t seed, uint64_t stream);
double tgsx_pcg32_uniform(uint64_t state[2]);
void tgsx_pcg32_advance(uint64_t state[2], uint64_t delta);

/* ---------------------------------------------------------------- stage access (parity) */
/* Per-stage outputs for bit-exact parity checks. All write host or device
 * memory. prepare: 11 float arrays [11][n] (mean x, mean y, inv00, inv01, inv11, alpha, r, g,
 * b, rx, ry) + orig[n], in blend order (rasterizer.cpp:23-46). */
int32_t tgsx_stage_prepare(tgsx_ctx* ctx, tgsx_model* m, int32_t lowpass_p, float* out,
                           uint32_t* orig);
/* Blend order (model.hpp:106-119). */
int32_t tgsx_stage_sorted_order(tgsx_ctx* ctx, tgsx_model* m, uint32_t* perm);
/* Per-tile CSR lists (rasterizer.cpp:59-102): offsets[tiles+1]; items up to items_cap; items
 * are blend-order indices. */
int32_t tgsx_stage_tile_lists(tgsx_ctx* ctx, tgsx_model* m, int32_t lowpass_p, int32_t width,
                              int32_t height, uint32_t* offsets, uint32_t* items,
                              int64_t items_cap, int64_t* out_k);
/* Screen-space per-Gaussian sums of the last backward (rasterizer.cpp:294-319):
 * [10][n] floats (mean x, mean y, s00, s01, s11, alpha, r, g, b, visited 0/1). */
int32_t tgsx_stage_screen_grads(tgsx_ctx* ctx, tgsx_model* m, float* out);
/* Per-pixel last-contributor count and evaluation counters of the last render:
 * *out_evals = reference-equivalent pixel-splat evaluations. */
int32_t tgsx_stage_counters(tgsx_ctx* ctx, uint64_t* out_blend_ops, uint64_t* out_evals,
                            uint64_t* out_pairs);
/* Device-wide stable LSD radix sort of (u32 key, u32 value) pairs on the low key_bits bits
 * (the onesweep kernels used for binning), exposed for direct testing. Device pointers. */
int32_t tgsx_sort_pairs(tgsx_ctx* ctx, uint32_t* keys, uint32_t* vals, int64_t n,
                        int32_t key_bits);
/* Device-wide exclusive scan of u32 (single-pass decoupled look-back). Device pointers;
 * *out_total (host) may be NULL. */
int32_t tgsx_exclusive_scan(tgsx_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                            uint64_t* out_total);

/* ---------------------------------------------------------------- 3-D front end
 * SURVEY.md §8a row A3b / BASELINE.json north_star item (1): per-Gaussian EWA projection to a
 * 2-D covariance, SH-degree-3 colour and near-plane / tile-rect culling in front of the same
 * binning, blend and backward kernels as the 2-D path, and the chain rule back to the 3-D
 * parameters fused with Adam. The reference is a 2-D analog with NO 3-D code:
 * these entry points have no reference counterpart to replace; they follow the published 3DGS
 * algorithm (restated in FP64 by oracle/ewa3d.c) and reuse the 2-D conventions: the low-pass
 * bump 0.3 + 0.5 (p - 1) (dilation.hpp:67-80), 3-sigma box extents (rasterizer.cpp:40-41),
 * pixel centres at (x + 0.5, y + 0.5) (rasterizer.cpp:114), the reference's blend.
 *
 * Parameters: float[59][n] (row-major, one row per component, n columns): mean xyz (world),
 * quaternion w x y z (normalised in the forward), log-scales xyz, raw opacity (sigmoid),
 * SH coefficients sh[k][c] at row 11 + 3k + c (k = 0..15, c = r g b); colour = SH + 0.5
 * clamped at 0. Blend order: ascending camera depth, ties by row. Gaussians at depth <= znear
 * are culled. Non-finite parameters / zero quaternion -> TGSX_EINVAL. */
typedef struct tgsx_model3d tgsx_model3d;
#define TGSX_3D_PARAMS 59
/* Pinhole camera: p_cam = R p_world + t (R row-major), u = fx x/z + cx, v = fy y/z + cy in
 * pixel units of a width x height image (OpenCV axes: x right, y down, z forward). */
typedef struct {
    float R[9];
    float t[3];
    float fx, fy, cx, cy, znear;
    int32_t width, height;
} tgsx_camera;
/* 3DGS learning rates: mean 1.6e-4 * scene_extent * 0.01^(step/total) (as SPEC.md:284's
 * position schedule), rotation 1e-3, log-scale 5e-3, opacity 5e-2, SH DC 2.5e-3, SH rest
 * 2.5e-3 / 20; Adam beta (0.9, 0.999), eps 1e-15; raw opacity in [-12, 12]. */
typedef struct {
    int64_t step, total_steps;
    double scene_extent;
} tgsx_adam3d_args;

int32_t tgsx_model3d_create(tgsx_ctx* ctx, int64_t capacity, tgsx_model3d** out);
void tgsx_model3d_destroy(tgsx_model3d* m);
int64_t tgsx_model3d_size(const tgsx_model3d* m);
/* Grows the capacity (rows kept) so later densify events allocate nothing. */
int32_t tgsx_model3d_reserve(tgsx_ctx* ctx, tgsx_model3d* m, int64_t capacity);
/* params host or device float[59][n]; zeroes the Adam moments and statistics. */
int32_t tgsx_model3d_upload(tgsx_ctx* ctx, tgsx_model3d* m, const float* params, int64_t n);
/* Any pointer may be NULL. Statistics: screen-space position-gradient norm sum, SH-DC
 * colour-gradient norm sum and visit count per Gaussian (the 2-D DensifyStats analogues,
 * rasterizer.cpp:348-359). */
int32_t tgsx_model3d_download(tgsx_ctx* ctx, tgsx_model3d* m, float* params, float* pos_acc,
                              float* col_acc, int32_t* visits);
int32_t tgsx_model3d_download_moments(tgsx_ctx* ctx, tgsx_model3d* m, float* m1, float* m2);
/* render<float> (rasterizer.hpp:58-60) with the 3-D front end; camera size == pattern size. */
int32_t tgsx_render3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                      const float bg[3], int32_t lowpass_p, float* out_rgb, float* out_T,
                      uint64_t* out_blend_ops);
/* backward<float> (rasterizer.hpp:66-69) with the 3-D chain rule: out_grads float[59][n] (zero for
 * Gaussians this view does not touch), out_screen float[10][n] the merged screen-space sums
 * (d mean xy, d Sigma' 00 01 11, d alpha, d rgb, visited), both host or device, may be NULL. */
int32_t tgsx_backward3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                        const float bg[3], int32_t lowpass_p, const float* dLdC, int64_t dLdC_count,
                        float* out_grads, float* out_screen, int32_t update_stats);
/* Adam with explicit gradients float[59][n] (host or device). */
int32_t tgsx_adam3d_step(tgsx_ctx* ctx, tgsx_model3d* m, const float* grads, const tgsx_adam3d_args* a);
/* One fused fit iteration of the 3-D model on one view (tgsx_fit_step with the 3-D front end). */
int32_t tgsx_fit_step3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                        const float bg[3], const float* target, const tgsx_adam3d_args* a, float* out_loss);
/* Batched views (SPEC.md:269-277 accumulate): each view adds its 59 gradients, the
 * position / colour norms and a visit count into the model's step buffer float[62][capacity]
 * (device; all-reduce it across ranks with NCCL), then tgsx_apply_step3d applies the mean over
 * batch_views (all ranks' views), the statistics and Adam, and zeroes the buffer. */
int32_t tgsx_view_accumulate3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                               const float bg[3], const float* target, float* out_loss);
float* tgsx_step_buffer3d(tgsx_model3d* m, int64_t* out_floats);
int32_t tgsx_allreduce_step3d(tgsx_ctx* ctx, tgsx_model3d* m);  /* NCCL sum of the [62][n] buffer */
int32_t tgsx_apply_step3d(tgsx_ctx* ctx, tgsx_model3d* m, int32_t batch_views, const tgsx_adam3d_args* a);
/* Parity stage: the 64-B records (Prepared layout, raster.cu) of all n Gaussians and their
 * orderable depth keys (culled: 0xffffffff), in the order the binning produced them:
 * *out_blend_ordered = 0 -> row order (per-tile path: each tile list is sorted by (key, row)),
 * 1 -> blend order (global-sort fallback for lists longer than a slab). */
int32_t tgsx_stage_prepare3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, int32_t lowpass_p,
                             float* out_records, uint32_t* out_keys, int32_t* out_blend_ordered);

/* Densification of the 3-D model (north_star item 4 on the 3-D path). The reference has only the
 * 2-D densifier; this is the same event on the 3-D parameters, with the SPEC's
 * statistics mapped to the 3-D front end's (screen-space position-gradient norm, SH-DC colour
 * norm, visits; accum = visits since the last event, window = visits since the last audit):
 * colour coin -> select (visits > tau_v, sigmoid(opacity) >= mask floor, averaged position norm >
 * tau_pos or coin and averaged colour norm > 0.01 tau_pos) -> cap to budget - count (top-k by
 * averaged position norm, ties by index) -> spawn (child at a point uniform in the parent's
 * 1-sigma ellipsoid, log-scales - ln 2, quaternion and SH copied, opacity 0.1, 3 PCG32 draws per
 * child in parent order) -> prune (sigmoid(opacity) < prune floor, order-preserving compaction)
 * -> reset. Restated in FP64 by oracle/ewa3d.c (or3d_densify_event); no reference code exists
 * for it. Fails with TGSX_ESTATE while a batched step (tgsx_view_accumulate3d) is pending. */
int32_t tgsx_densify3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_densify_config* c, int64_t budget,
                       uint64_t rng_state[2], tgsx_densify_report* out);
/* update_visit_thresholds on the visits since the last audit. */
int32_t tgsx_visit_audit3d(tgsx_ctx* ctx, tgsx_model3d* m);
/* The SPEC fit loop (tgsx_trainer_*) over a set of cameras of a 3-D model:
 * view (t - 1) mod n_cams at iteration t; dilated warm-up with cycled offsets; densify every
 * densify_interval with the convergence-aware budget (tgsx_densify3d); after densify_until a
 * dilation coin per iteration, dense iterations with the SSIM term; the last batch_final_iters
 * iterations accumulate batch_size distinct cameras and take one Adam step on the mean; visit
 * audits every n_views iterations. Adam: tgsx_adam3d_args with scene_extent. targets[v]: the
 * full-resolution RGB of camera v (host or device), n_targets == n_cams. */
typedef struct tgsx_trainer3d tgsx_trainer3d;
int32_t tgsx_trainer3d_create(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_train_config* cfg,
                              const tgsx_camera* cams, int32_t n_cams, double scene_extent,
                              tgsx_trainer3d** out);
void tgsx_trainer3d_destroy(tgsx_trainer3d* tr);
int32_t tgsx_trainer3d_step(tgsx_trainer3d* tr, const float* const* targets, int64_t n_targets,
                            tgsx_train_report* report);
/* Per-iteration losses of the last min(ring, t) iterations, oldest first. */
int32_t tgsx_trainer3d_losses(tgsx_trainer3d* tr, float* out, int64_t max_out, int64_t* out_n);
/* Densification state per Gaussian (any pointer may be NULL): stable ids (0..n-1 at upload,
 * children numbered from next_id), tau_v, the visit count at the last event / audit. */
int32_t tgsx_model3d_download_state(tgsx_ctx* ctx, tgsx_model3d* m, uint64_t* ids, double* tau_v,
                                    int32_t* visit_evt, int32_t* visit_aud, uint64_t* next_id);

/* Diagnostics: measured FP32 throughput of this GPU (8 independent FMA chains per thread, one
 * launch of 8 CTAs x 256 threads per SM) with scalar FFMA and packed FFMA2, in TFLOP/s (FMA = 2
 * flops) — the roofline denominator of the blend kernels. */
int32_t tgsx_measure_fp32_peak(tgsx_ctx* ctx, double* out_ffma_tflops, double* out_ffma2_tflops);

#ifdef __cplusplus
}
#endif
#endif /* TGSX_H */
