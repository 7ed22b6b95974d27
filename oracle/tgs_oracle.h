/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the Turbo-GS fit hot path.
 *
 * A single-threaded C restatement of the reference algorithm, used ONLY by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg, as the checker. Nothing in the
 * product (paper_2412_13547_b200/) links or calls it.
 *
 * Pinning:
 *  - render / backward / prepare / tile grid / sorted order: restated from
 *    /root/reference/proj/core/src/rasterizer.cpp and include/tgs/*.hpp; pinned bit-for-bit
 *    against the unmodified reference compiled into oracle/_ref (tests/test_oracle_pin.py),
 *    in both transcendental modes (cr_math.h), and against committed golden fixtures
 *    (tests/golden/, generated from oracle/_ref by tests/golden/make_golden.py).
 *  - L1 loss, Adam, densify, visit audit, budget controller: the reference sources are
 *    MISSING; restated from SPEC.md prose and pinned only by the SPEC's
 *    known-answer examples and properties (tests/test_oracle_spec.py).
 */
#ifndef TGS_ORACLE_H
#define TGS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Scene in model (creation/index) order. Stats / tau_v may be NULL where unused. */
typedef struct {
    int64_t n;
    float *px, *py, *rot, *lsx, *lsy, *rop, *cr, *cg, *cb, *depth;
    uint64_t* id;
    float *pos_acc, *col_acc;
    int32_t* accum;
    int64_t *visit, *window;
    double* tau_v;
    uint64_t next_id;
} or_scene;

/* prepare_splats output (rasterizer.cpp:13-21), blend order. */
typedef struct {
    float *mx, *my, *i00, *i01, *i11, *alpha, *c0, *c1, *c2, *rx, *ry;
    uint32_t* orig;
} or_prepared;

/* Screen-space per-Gaussian sums after the tile-order merge (rasterizer.cpp:294-319). */
typedef struct {
    float *gmx, *gmy, *gs00, *gs01, *gs11, *galpha, *gc0, *gc1, *gc2, *maxw;
    uint8_t* touched;
} or_screen_grads;

typedef struct {
    uint64_t state, inc;
} or_pcg32;

typedef struct {
    double n_init, m_final, m_adaptive, alpha, alpha_base, ema;
    int has_ema;
    int64_t warmup_steps, window_size, refit_interval, ma_depth, last_refit;
    double lambda;
    /* loss log (t, ema) and fitted alpha_history values */
    int64_t log_len, log_cap;
    double *log_t, *log_ema;
    int64_t fit_len, fit_cap;
    double* fits;
} or_budget;

void or_set_math(int cr);

/* rng.hpp:10-46 */
void or_pcg32_init(or_pcg32* r, uint64_t seed, uint64_t stream);
uint32_t or_pcg32_next(or_pcg32* r);
double or_pcg32_uniform(or_pcg32* r);
void or_pcg32_advance(or_pcg32* r, uint64_t delta);

/* Synthetic generator: per Gaussian x,y,rot,lsx,lsy,rop,r,g,b,depth. */
void or_synthetic_scene(uint64_t seed, int64_t n, int W, int H, or_scene* out);

int or_sorted_order(const or_scene* s, uint32_t* perm);
int or_prepare(const or_scene* s, int lowpass_p, or_prepared* out);
int or_tile_grid(const or_prepared* sp, int64_t n, int W, int H, uint32_t* offsets,
                 uint32_t* items, int64_t items_cap, int64_t* out_k);
int or_render(const or_scene* s, int p, int ox, int oy, int W, int H, const float* bg,
              int lowpass_p, float* out_rgb, float* out_T, uint64_t* out_ops, uint64_t* out_evals);
int or_backward(or_scene* s, int p, int ox, int oy, int W, int H, const float* bg,
                const float* dLdC, int lowpass_p, float* const* grads, or_screen_grads* screen,
                int update_stats);

/* compute_loss: dense (p = 1, lam > 0) (1-lam) L1 + lam (1 - SSIM), else L1 */
double or_loss(const float* rgb, int p, int ox, int oy, int W, int H, const float* target,
               float lam, float* dLdC);
double or_l1_loss(const float* rgb, int p, int ox, int oy, int W, int H, const float* target,
                  float* dLdC);

typedef struct {
    float beta1, beta2, eps;
    float lr[9]; /* per component: pos x, pos y, rot, ls x, ls y, raw_o, r, g, b */
    float bc1, bc2; /* 1 - beta^t, computed in double and rounded */
    float ls_lo, ls_hi, raw_cap;
} or_adam_cfg;
void or_adam_config(or_adam_cfg* c, int64_t step, int64_t total_steps, double diag);
void or_adam_step(or_scene* s, float* const* grads, float* const* m, float* const* v,
                  const or_adam_cfg* c);

typedef struct {
    float tau_pos, tau_color, opacity_mask_floor, opacity_prune_floor, color_branch_prob;
    double tau_v_init;
    float child_raw_opacity; /* inverse_activate(0.1) */
} or_densify_cfg;
void or_densify_config(or_densify_cfg* c, float tau_pos);
int64_t or_select_candidates(const or_scene* s, const or_densify_cfg* c, int color_coin,
                             uint8_t* cand);
int64_t or_cap_candidates(const or_scene* s, uint8_t* cand, int64_t budget_remaining);
int64_t or_spawn(or_scene* s, int64_t capacity, const uint8_t* sel, or_pcg32* rng,
                 const or_densify_cfg* c, float* const* m, float* const* v);
int64_t or_prune(or_scene* s, const or_densify_cfg* c, float* const* m, float* const* v);
void or_reset_accumulators(or_scene* s);
void or_visit_audit(or_scene* s);
int64_t or_densify_event(or_scene* s, int64_t capacity, const or_densify_cfg* c, int64_t budget,
                         or_pcg32* rng, float* const* m, float* const* v, int64_t* out_spawned,
                         int64_t* out_pruned, int64_t* out_candidates);

void or_budget_init(or_budget* b, double n_init, double m_final);
void or_budget_free(or_budget* b);
int or_budget_record_loss(or_budget* b, int64_t t, double loss);
int or_fit_power_exponent(const double* t, const double* y, int64_t n, double* out);
void or_budget_update(or_budget* b, int64_t t);
int64_t or_budget_at(const or_budget* b, double t_norm);
double or_budget_t_norm(int64_t step, int64_t warmup, int64_t densify_end);


/* Blend stages over splats already prepared in blend order (orig = index into n_orig). */
int or_render_prepared(const or_prepared* sp, int64_t n, int p, int ox, int oy, int W, int H,
                       const float* bg, float* out_rgb, float* out_T, uint64_t* out_ops,
                       uint64_t* out_evals);
int or_backward_prepared(const or_prepared* sp, int64_t n, int64_t n_orig, int p, int ox, int oy,
                         int W, int H, const float* bg, const float* dLdC, or_screen_grads* screen);

/* ---------------- 3-D front end (ewa3d.c; SURVEY.md §8a A3b — parity unpinned at the
 * reference, which has no 3-D code; pinned by formula KATs and FP64 finite differences) */
#define OR3D_PARAMS 59
typedef struct {
    double R[9]; /* world -> camera rotation, row-major */
    double t[3];
    double fx, fy, cx, cy, znear;
    int W, H;
} or_camera;
void or3d_sh_basis(double x, double y, double z, double* b, double* db);
/* out[12]: u v s00 s01 s11 (Σ' incl. bump) alpha r g b depth rx ry; 1 visible, 0 culled, -1 invalid */
int or3d_project(const double* theta, const or_camera* cam, double bump, double* out);
/* screen[9]: d(u, v), dΣ'(00, 01, 11; symmetric convention), d alpha, d rgb -> grad[59] */
void or3d_chain(const double* theta, const or_camera* cam, double bump, const double* screen,
                double* grad);
int or3d_prepare(const float* params, int64_t n, const or_camera* cam, int lowpass_p,
                 or_prepared* out, float* depth_out, int64_t* out_visible);
int or3d_render(const float* params, int64_t n, const or_camera* cam, int p, int ox, int oy,
                const float* bg, int lowpass_p, float* out_rgb, float* out_T, uint64_t* out_ops,
                uint64_t* out_evals);
int or3d_backward(const float* params, int64_t n, const or_camera* cam, int p, int ox, int oy,
                  const float* bg, const float* dLdC, int lowpass_p, float* grads,
                  or_screen_grads* screen);
typedef struct {
    float beta1, beta2, eps;
    float lr_pos, lr_rot, lr_scale, lr_opacity, lr_dc, lr_rest;
    float bc1, bc2, raw_cap;
} or3d_adam_cfg;
void or3d_adam_config(or3d_adam_cfg* c, int64_t step, int64_t total_steps, double extent);
float or3d_lr(const or3d_adam_cfg* c, int k);
void or3d_adam_step(float* params, const float* grads, float* m, float* v, int64_t n,
                    const or3d_adam_cfg* c);
/* activate (gaussian.hpp:47-49) in float with the oracle's expf (libm or correctly rounded) */
float or_activatef(float raw);
/* Densification of the 3-D model (the 2-D densify event of SPEC.md:300-383 on the 3-D
 * parameters; the GPU counterpart is tgsx_densify3d). Arrays are capacity-strided like the
 * device model ([59][cap] params and moments); accum = visit - visit_evt. */
typedef struct {
    int64_t n, cap;
    float* params;          /* [59][cap] */
    float* m1;              /* [59][cap] */
    float* m2;              /* [59][cap] */
    float* pos_acc;
    float* col_acc;
    int32_t* visit;
    int32_t* visit_evt;
    int32_t* visit_aud;
    uint64_t* id;
    double* tau_v;
    uint64_t next_id;
} or3d_model;
int64_t or3d_densify_event(or3d_model* s, const or_densify_cfg* c, int64_t budget, or_pcg32* rng,
                           int64_t* out_spawned, int64_t* out_pruned, int64_t* out_candidates,
                           int* out_coin);
void or3d_visit_audit(or3d_model* s);

#ifdef __cplusplus
}
#endif
#endif
