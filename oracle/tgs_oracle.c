/* TEST INFRASTRUCTURE ONLY — CPU oracle (C restatement) of the Turbo-GS fit hot path.
 * See tgs_oracle.h for scope and pinning. Every function cites the reference file:line it
 * restates (paths relative to /root/reference/). Single-threaded by design: the reference's
 * results are independent of its worker count, so a serial restatement in
 * the reference's tile/merge order reproduces them bit for bit. Compiled with
 * -ffp-contract=off (proj/CMakeLists.txt:12) and written with the reference's evaluation
 * order, so every float expression rounds the same way.
 */
#include "tgs_oracle.h"

#include "cr_math.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

int or_math_cr = 1;
void or_set_math(int cr) { or_math_cr = cr ? 1 : 0; }

/* ---------------------------------------------------------------- constants */
/* rasterizer.hpp:12-19 */
#define TILE 16
static const float kTermT = (float)1e-4;   /* kTerminationTransmittance */
static const float kMinVisitW = (float)1e-4; /* kMinVisitWeight */
static const float kCullSigmas = 3.0f;
/* gaussian.hpp:14,18 */
static const double kMinScale = 1e-4;
static const double kRawCap = 12.0;

/* ---------------------------------------------------------------- PCG32 (rng.hpp:10-46) */
void or_pcg32_init(or_pcg32* r, uint64_t seed, uint64_t stream) {
    r->state = 0;
    r->inc = (stream << 1u) | 1u;
    or_pcg32_next(r);
    r->state += seed;
    or_pcg32_next(r);
}

uint32_t or_pcg32_next(or_pcg32* r) {
    uint64_t old = r->state;
    r->state = old * 6364136223846793005ULL + r->inc;
    uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
    uint32_t rot = (uint32_t)(old >> 59u);
    return (xs >> rot) | (xs << ((32u - rot) & 31u));
}

double or_pcg32_uniform(or_pcg32* r) { return or_pcg32_next(r) * 0x1p-32; }

static double uniform_in(or_pcg32* r, double lo, double hi) {
    return lo + (hi - lo) * or_pcg32_uniform(r);
}

/* LCG jump-ahead (Brown, "Random number generation with arbitrary strides"): advancing the
 * state by delta steps without drawing. Used to check the GPU spawner's per-child streams. */
void or_pcg32_advance(or_pcg32* r, uint64_t delta) {
    uint64_t cur_mult = 6364136223846793005ULL, cur_plus = r->inc;
    uint64_t acc_mult = 1u, acc_plus = 0u;
    while (delta > 0) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    r->state = acc_mult * r->state + acc_plus;
}

/* ---------------------------------------------------------------- synthetic generator */
/* SURVEY.md §8(d) / BASELINE.md §2: Pcg32(seed, stream 1); per Gaussian in order
 * x~U[0,W), y~U[0,H), rot~U[-pi,pi), log_s~U[0,1.5)^2, raw_o~U[-2,2), raw_rgb~U[-2,2)^3,
 * depth~U[0,1); ids 0..n-1; tau_v = 5. Caller owns the arrays (all length n). */
void or_synthetic_scene(uint64_t seed, int64_t n, int W, int H, or_scene* s) {
    or_pcg32 r;
    or_pcg32_init(&r, seed, 1);
    const double pi = 3.14159265358979323846;
    for (int64_t i = 0; i < n; ++i) {
        s->px[i] = (float)uniform_in(&r, 0.0, (double)W);
        s->py[i] = (float)uniform_in(&r, 0.0, (double)H);
        s->rot[i] = (float)uniform_in(&r, -pi, pi);
        s->lsx[i] = (float)uniform_in(&r, 0.0, 1.5);
        s->lsy[i] = (float)uniform_in(&r, 0.0, 1.5);
        s->rop[i] = (float)uniform_in(&r, -2.0, 2.0);
        s->cr[i] = (float)uniform_in(&r, -2.0, 2.0);
        s->cg[i] = (float)uniform_in(&r, -2.0, 2.0);
        s->cb[i] = (float)uniform_in(&r, -2.0, 2.0);
        s->depth[i] = (float)uniform_in(&r, 0.0, 1.0);
        if (s->id) s->id[i] = (uint64_t)i;
        if (s->tau_v) s->tau_v[i] = 5.0;
        if (s->pos_acc) {
            s->pos_acc[i] = 0.f;
            s->col_acc[i] = 0.f;
            s->accum[i] = 0;
            s->visit[i] = 0;
            s->window[i] = 0;
        }
    }
    s->n = n;
    s->next_id = (uint64_t)n;
}

/* ---------------------------------------------------------------- blend order */
/* GaussianModel::sorted_order, model.hpp:106-119: ascending depth_key, ties by id. */
static const or_scene* g_sort_scene;
static int cmp_order(const void* a, const void* b) {
    uint32_t i = *(const uint32_t*)a, j = *(const uint32_t*)b;
    const float di = g_sort_scene->depth[i], dj = g_sort_scene->depth[j];
    if (di != dj) return di < dj ? -1 : 1;
    const uint64_t ii = g_sort_scene->id ? g_sort_scene->id[i] : i;
    const uint64_t ij = g_sort_scene->id ? g_sort_scene->id[j] : j;
    return ii < ij ? -1 : (ii > ij ? 1 : 0);
}

int or_sorted_order(const or_scene* s, uint32_t* perm) {
    for (int64_t i = 0; i < s->n; ++i) perm[i] = (uint32_t)i;
    g_sort_scene = s;
    qsort(perm, (size_t)s->n, sizeof(uint32_t), cmp_order);
    return 0;
}

/* ---------------------------------------------------------------- preprocess */
/* covariance_from_params gaussian.hpp:63-78, apply_lowpass dilation.hpp:67-80 (bump
 * 0.3 + 0.5(p-1), dilation.hpp:60-64), invert gaussian.hpp:82-92, activate gaussian.hpp:47-49,
 * rx/ry rasterizer.cpp:40-41. Returns 0, 1 (invalid_argument: non-finite rotation/log-scale,
 * gaussian.hpp:64-68; bad p, dilation.hpp:75) or 2 (runtime_error: det<=0, gaussian.hpp:84-86). */
static float activate(float raw) { return 1.0f / (1.0f + m_expf(-raw)); }
float or_activatef(float raw) { return activate(raw); }

static int prepare_one(const or_scene* s, uint32_t idx, int lowpass_p, float* o /*11*/) {
    const float rot = s->rot[idx], lx = s->lsx[idx], ly = s->lsy[idx];
    if (!isfinite((double)rot) || !isfinite((double)lx) || !isfinite((double)ly)) return 1;
    const float c = m_cosf(rot);
    const float n = m_sinf(rot);
    const float a = m_expf(2.0f * lx);
    const float b = m_expf(2.0f * ly);
    float s00 = c * c * a + n * n * b;
    float s01 = c * n * (a - b);
    float s11 = n * n * a + c * c * b;
    if (lowpass_p < 1) return 1;
    const float bump = 0.3f + 0.5f * (float)(lowpass_p - 1);
    s00 += bump;
    s11 += bump;
    const float det = s00 * s11 - s01 * s01;
    if (!(det > 0.0f) || !isfinite((double)det)) return 2;
    o[0] = s->px[idx];
    o[1] = s->py[idx];
    o[2] = s11 / det;
    o[3] = -s01 / det;
    o[4] = s00 / det;
    o[5] = activate(s->rop[idx]);
    o[6] = activate(s->cr[idx]);
    o[7] = activate(s->cg[idx]);
    o[8] = activate(s->cb[idx]);
    o[9] = kCullSigmas * sqrtf(s00);
    o[10] = kCullSigmas * sqrtf(s11);
    return 0;
}

int or_prepare(const or_scene* s, int lowpass_p, or_prepared* out) {
    uint32_t* perm = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(s->n ? s->n : 1));
    or_sorted_order(s, perm);
    int rc = 0;
    for (int64_t r = 0; r < s->n && rc == 0; ++r) {
        float o[11];
        rc = prepare_one(s, perm[r], lowpass_p, o);
        if (rc) break;
        out->mx[r] = o[0]; out->my[r] = o[1];
        out->i00[r] = o[2]; out->i01[r] = o[3]; out->i11[r] = o[4];
        out->alpha[r] = o[5];
        out->c0[r] = o[6]; out->c1[r] = o[7]; out->c2[r] = o[8];
        out->rx[r] = o[9]; out->ry[r] = o[10];
        out->orig[r] = perm[r];
    }
    free(perm);
    return rc;
}

/* ---------------------------------------------------------------- binning */
/* pixel_span rasterizer.cpp:50-56: the bounds are computed in double on the float m±r. */
static void pixel_span(float m, float r, int limit, int* lo, int* hi) {
    *lo = (int)ceil((double)(m - r) - 0.5);
    *hi = (int)floor((double)(m + r) - 0.5);
    if (*lo < 0) *lo = 0;
    if (*hi > limit - 1) *hi = limit - 1;
}

static int tile_rect(float mx, float my, float rx, float ry, int W, int H, int* tx0, int* tx1,
                     int* ty0, int* ty1) {
    int px0, px1, py0, py1;
    pixel_span(mx, rx, W, &px0, &px1);
    pixel_span(my, ry, H, &py0, &py1);
    if (px0 > px1 || py0 > py1) return 0;
    *tx0 = px0 / TILE; *tx1 = px1 / TILE;
    *ty0 = py0 / TILE; *ty1 = py1 / TILE;
    return 1;
}

/* build_tile_grid rasterizer.cpp:67-102: count, exclusive scan, scatter in blend order. */
int or_tile_grid(const or_prepared* sp, int64_t n, int W, int H, uint32_t* offsets,
                 uint32_t* items, int64_t items_cap, int64_t* out_k) {
    const int tx = (W + TILE - 1) / TILE, ty = (H + TILE - 1) / TILE;
    const int tiles = tx * ty;
    memset(offsets, 0, sizeof(uint32_t) * (size_t)(tiles + 1));
    for (int64_t i = 0; i < n; ++i) {
        int a, b, c, d;
        if (!tile_rect(sp->mx[i], sp->my[i], sp->rx[i], sp->ry[i], W, H, &a, &b, &c, &d)) continue;
        for (int y = c; y <= d; ++y)
            for (int x = a; x <= b; ++x) ++offsets[y * tx + x + 1];
    }
    for (int t = 1; t <= tiles; ++t) offsets[t] += offsets[t - 1];
    *out_k = offsets[tiles];
    if (!items || items_cap < *out_k) return 0;
    uint32_t* cur = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)tiles);
    memcpy(cur, offsets, sizeof(uint32_t) * (size_t)tiles);
    for (int64_t i = 0; i < n; ++i) {
        int a, b, c, d;
        if (!tile_rect(sp->mx[i], sp->my[i], sp->rx[i], sp->ry[i], W, H, &a, &b, &c, &d)) continue;
        for (int y = c; y <= d; ++y)
            for (int x = a; x <= b; ++x) items[cur[y * tx + x]++] = (uint32_t)i;
    }
    free(cur);
    return 0;
}

/* ---------------------------------------------------------------- pattern helpers */
/* DilationPattern dilation.hpp:16-56 */
typedef struct {
    int p, ox, oy, W, H, cols, rows;
} pattern_t;

static int make_pattern(int p, int ox, int oy, int W, int H, pattern_t* pt) {
    if (p < 1 || ox < 0 || oy < 0 || ox >= p || oy >= p || W < 1 || H < 1) return 1;
    pt->p = p; pt->ox = ox; pt->oy = oy; pt->W = W; pt->H = H;
    pt->cols = W > ox ? (W - ox - 1) / p + 1 : 0;
    pt->rows = H > oy ? (H - oy - 1) / p + 1 : 0;
    return 0;
}

static int first_active(const pattern_t* pt, int v, int offset) {
    if (v <= offset) return offset;
    const int k = (v - offset + pt->p - 1) / pt->p;
    return offset + k * pt->p;
}

typedef struct {
    int64_t n;
    or_prepared sp;
    float* buf;
    uint32_t* orig;
    uint32_t* offsets;
    uint32_t* items;
    int64_t k;
    int tiles_x, tiles_y;
} stage_t;

static int build_stage(const or_scene* s, int lowpass_p, int W, int H, stage_t* st) {
    memset(st, 0, sizeof(*st));
    const int64_t n = s->n;
    const size_t nn = (size_t)(n ? n : 1);
    st->n = n;
    st->buf = (float*)malloc(sizeof(float) * 11 * nn);
    st->orig = (uint32_t*)malloc(sizeof(uint32_t) * nn);
    float* b = st->buf;
    or_prepared* sp = &st->sp;
    sp->mx = b; sp->my = b + nn; sp->i00 = b + 2 * nn; sp->i01 = b + 3 * nn;
    sp->i11 = b + 4 * nn; sp->alpha = b + 5 * nn; sp->c0 = b + 6 * nn; sp->c1 = b + 7 * nn;
    sp->c2 = b + 8 * nn; sp->rx = b + 9 * nn; sp->ry = b + 10 * nn; sp->orig = st->orig;
    int rc = or_prepare(s, lowpass_p, sp);
    if (rc) return rc;
    st->tiles_x = (W + TILE - 1) / TILE;
    st->tiles_y = (H + TILE - 1) / TILE;
    st->offsets = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(st->tiles_x * st->tiles_y + 1));
    or_tile_grid(sp, n, W, H, st->offsets, NULL, 0, &st->k);
    st->items = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(st->k ? st->k : 1));
    or_tile_grid(sp, n, W, H, st->offsets, st->items, st->k, &st->k);
    return 0;
}

/* Stage over splats that are already prepared and in blend order (the 3-D front end, ewa3d.c). */
static void stage_from_prepared(const or_prepared* src, int64_t n, int W, int H, stage_t* st) {
    memset(st, 0, sizeof(*st));
    const size_t nn = (size_t)(n ? n : 1);
    st->n = n;
    st->buf = (float*)malloc(sizeof(float) * 11 * nn);
    st->orig = (uint32_t*)malloc(sizeof(uint32_t) * nn);
    float* b = st->buf;
    or_prepared* sp = &st->sp;
    sp->mx = b; sp->my = b + nn; sp->i00 = b + 2 * nn; sp->i01 = b + 3 * nn;
    sp->i11 = b + 4 * nn; sp->alpha = b + 5 * nn; sp->c0 = b + 6 * nn; sp->c1 = b + 7 * nn;
    sp->c2 = b + 8 * nn; sp->rx = b + 9 * nn; sp->ry = b + 10 * nn; sp->orig = st->orig;
    const float* s[11] = {src->mx, src->my, src->i00, src->i01, src->i11, src->alpha,
                          src->c0, src->c1, src->c2, src->rx, src->ry};
    for (int q = 0; q < 11; ++q) memcpy(b + q * nn, s[q], sizeof(float) * (size_t)n);
    memcpy(st->orig, src->orig, sizeof(uint32_t) * (size_t)n);
    st->tiles_x = (W + TILE - 1) / TILE;
    st->tiles_y = (H + TILE - 1) / TILE;
    st->offsets = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(st->tiles_x * st->tiles_y + 1));
    or_tile_grid(sp, n, W, H, st->offsets, NULL, 0, &st->k);
    st->items = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)(st->k ? st->k : 1));
    or_tile_grid(sp, n, W, H, st->offsets, st->items, st->k, &st->k);
}

static void free_stage(stage_t* st) {
    free(st->buf); free(st->orig); free(st->offsets); free(st->items);
}

/* ---------------------------------------------------------------- render */
/* walk_pixel rasterizer.cpp:108-136 + render rasterizer.cpp:144-184. */
static void render_stage(const stage_t* stp, const pattern_t* ptp, const float* bg, float* out_rgb,
                         float* out_T, uint64_t* out_ops, uint64_t* out_evals) {
    const stage_t st = *stp;
    const pattern_t pt = *ptp;
    const int p = pt.p, ox = pt.ox, oy = pt.oy, W = pt.W, H = pt.H;
    const or_prepared* sp = &st.sp;
    const int P = pt.cols * pt.rows;
    for (int i = 0; i < P; ++i) {
        out_rgb[3 * i] = out_rgb[3 * i + 1] = out_rgb[3 * i + 2] = 0.f;
        out_T[i] = 1.f;
    }
    uint64_t ops = 0, evals = 0;
    for (int t = 0; t < st.tiles_x * st.tiles_y; ++t) {
        const uint32_t* items = st.items + st.offsets[t];
        const uint32_t count = st.offsets[t + 1] - st.offsets[t];
        const int tx = t % st.tiles_x, ty = t / st.tiles_x;
        const int px1 = W < (tx + 1) * TILE ? W : (tx + 1) * TILE;
        const int py1 = H < (ty + 1) * TILE ? H : (ty + 1) * TILE;
        const int ax = first_active(&pt, tx * TILE, ox);
        const int ay = first_active(&pt, ty * TILE, oy);
        for (int y = ay; y < py1; y += p) {
            for (int x = ax; x < px1; x += p) {
                const int rank = ((y - oy) / p) * pt.cols + (x - ox) / p;
                const float fx = (float)x + 0.5f, fy = (float)y + 0.5f;
                float T = 1.f, c0 = 0.f, c1 = 0.f, c2 = 0.f;
                uint32_t k = 0;
                for (; k < count; ++k) {
                    const uint32_t j = items[k];
                    const float dx = fx - sp->mx[j];
                    const float dy = fy - sp->my[j];
                    if (!(fabsf(dx) <= sp->rx[j] && fabsf(dy) <= sp->ry[j])) continue;
                    const float q = sp->i00[j] * dx * dx + 2.0f * sp->i01[j] * dx * dy +
                                    sp->i11[j] * dy * dy;
                    const float g = m_expf(-0.5f * q);
                    const float sigma = sp->alpha[j] * g;
                    const float w = sigma * T;
                    c0 += w * sp->c0[j];
                    c1 += w * sp->c1[j];
                    c2 += w * sp->c2[j];
                    T *= (1.0f - sigma);
                    ++ops;
                    if (T < kTermT) { ++k; break; }
                }
                evals += k;
                c0 += T * bg[0];
                c1 += T * bg[1];
                c2 += T * bg[2];
                out_rgb[3 * rank] = c0;
                out_rgb[3 * rank + 1] = c1;
                out_rgb[3 * rank + 2] = c2;
                out_T[rank] = T;
            }
        }
    }
    if (out_ops) *out_ops = ops;
    if (out_evals) *out_evals = evals;
}

int or_render(const or_scene* s, int p, int ox, int oy, int W, int H, const float* bg,
              int lowpass_p, float* out_rgb, float* out_T, uint64_t* out_ops,
              uint64_t* out_evals) {
    pattern_t pt;
    if (make_pattern(p, ox, oy, W, H, &pt)) return 1;
    stage_t st;
    int rc = build_stage(s, lowpass_p > 0 ? lowpass_p : p, W, H, &st);
    if (rc) { free_stage(&st); return rc; }
    render_stage(&st, &pt, bg, out_rgb, out_T, out_ops, out_evals);
    free_stage(&st);
    return 0;
}

int or_render_prepared(const or_prepared* sp, int64_t n, int p, int ox, int oy, int W, int H,
                       const float* bg, float* out_rgb, float* out_T, uint64_t* out_ops,
                       uint64_t* out_evals) {
    pattern_t pt;
    if (make_pattern(p, ox, oy, W, H, &pt)) return 1;
    stage_t st;
    stage_from_prepared(sp, n, W, H, &st);
    render_stage(&st, &pt, bg, out_rgb, out_T, out_ops, out_evals);
    free_stage(&st);
    return 0;
}

/* ---------------------------------------------------------------- backward */
/* backward rasterizer.cpp:218-361: per-tile recompute + exact reverse suffix (:255-287),
 * serial tile-order merge (:301-319), chain rule (:321-346), densify stats (:348-359). */
typedef struct {
    uint32_t k;
    float dx, dy, g, sigma, trans, w;
} contrib_t;

/* Tile phase + tile-order merge over a built stage: acc[10][nn] (gmx gmy s00 s01 s11 alpha c0 c1
 * c2 maxw) and touched[nn], indexed by the splats' orig index, zero-initialised by the caller. */
static void backward_stage(const stage_t* stp, const pattern_t* ptp, const float* bg,
                           const float* dLdC, float* acc, uint8_t* touched, size_t nn) {
    const stage_t st = *stp;
    const pattern_t pt = *ptp;
    const int p = pt.p, ox = pt.ox, oy = pt.oy, W = pt.W, H = pt.H;
    const or_prepared* sp = &st.sp;
    /* tile-local accumulators, sized to the longest list */
    uint32_t maxc = 0;
    for (int t = 0; t < st.tiles_x * st.tiles_y; ++t) {
        const uint32_t c = st.offsets[t + 1] - st.offsets[t];
        if (c > maxc) maxc = c;
    }
    const size_t mc = maxc ? maxc : 1;
    float* loc = (float*)malloc(sizeof(float) * 10 * mc);
    uint8_t* ltouch = (uint8_t*)malloc(mc);
    contrib_t* cb = (contrib_t*)malloc(sizeof(contrib_t) * mc);
    for (int t = 0; t < st.tiles_x * st.tiles_y; ++t) {
        const uint32_t* items = st.items + st.offsets[t];
        const uint32_t count = st.offsets[t + 1] - st.offsets[t];
        if (count == 0) continue;
        memset(loc, 0, sizeof(float) * 10 * count);
        memset(ltouch, 0, count);
        float* L_mx = loc; float* L_my = loc + count; float* L_s00 = loc + 2 * count;
        float* L_s01 = loc + 3 * count; float* L_s11 = loc + 4 * count;
        float* L_a = loc + 5 * count; float* L_c0 = loc + 6 * count; float* L_c1 = loc + 7 * count;
        float* L_c2 = loc + 8 * count; float* L_mw = loc + 9 * count;
        const int tx = t % st.tiles_x, ty = t / st.tiles_x;
        const int px1 = W < (tx + 1) * TILE ? W : (tx + 1) * TILE;
        const int py1 = H < (ty + 1) * TILE ? H : (ty + 1) * TILE;
        const int ax = first_active(&pt, tx * TILE, ox);
        const int ay = first_active(&pt, ty * TILE, oy);
        for (int y = ay; y < py1; y += p) {
            for (int x = ax; x < px1; x += p) {
                const int rank = ((y - oy) / p) * pt.cols + (x - ox) / p;
                const float fx = (float)x + 0.5f, fy = (float)y + 0.5f;
                float T = 1.f;
                uint32_t nc = 0;
                for (uint32_t k = 0; k < count; ++k) {
                    const uint32_t j = items[k];
                    const float dx = fx - sp->mx[j];
                    const float dy = fy - sp->my[j];
                    if (!(fabsf(dx) <= sp->rx[j] && fabsf(dy) <= sp->ry[j])) continue;
                    const float q = sp->i00[j] * dx * dx + 2.0f * sp->i01[j] * dx * dy +
                                    sp->i11[j] * dy * dy;
                    const float g = m_expf(-0.5f * q);
                    const float sigma = sp->alpha[j] * g;
                    const float w = sigma * T;
                    contrib_t c = {k, dx, dy, g, sigma, T, w};
                    cb[nc++] = c;
                    ltouch[k] = 1;
                    if (w > L_mw[k]) L_mw[k] = w;
                    T *= (1.0f - sigma);
                    if (T < kTermT) break;
                }
                const float gx = dLdC[3 * rank], gy = dLdC[3 * rank + 1], gz = dLdC[3 * rank + 2];
                if (gx == 0.f && gy == 0.f && gz == 0.f) continue;
                float S0 = bg[0] * T, S1 = bg[1] * T, S2 = bg[2] * T;
                for (uint32_t ci = nc; ci-- > 0;) {
                    const contrib_t* c = &cb[ci];
                    const uint32_t j = items[c->k];
                    L_c0[c->k] += gx * c->w;
                    L_c1[c->k] += gy * c->w;
                    L_c2[c->k] += gz * c->w;
                    const float inv_rest = 1.0f / (1.0f - c->sigma);
                    const float d0 = sp->c0[j] * c->trans - S0 * inv_rest;
                    const float d1 = sp->c1[j] * c->trans - S1 * inv_rest;
                    const float d2 = sp->c2[j] * c->trans - S2 * inv_rest;
                    const float dsig = gx * d0 + gy * d1 + gz * d2;
                    L_a[c->k] += dsig * c->g;
                    const float dq = dsig * sp->alpha[j] * -0.5f * c->g;
                    const float adx = sp->i00[j] * c->dx + sp->i01[j] * c->dy;
                    const float ady = sp->i01[j] * c->dx + sp->i11[j] * c->dy;
                    L_mx[c->k] += -2.0f * dq * adx;
                    L_my[c->k] += -2.0f * dq * ady;
                    L_s00[c->k] += -dq * adx * adx;
                    L_s01[c->k] += -dq * adx * ady;
                    L_s11[c->k] += -dq * ady * ady;
                    S0 += sp->c0[j] * c->w;
                    S1 += sp->c1[j] * c->w;
                    S2 += sp->c2[j] * c->w;
                }
            }
        }
        /* merge in tile order (rasterizer.cpp:301-319) */
        for (uint32_t k = 0; k < count; ++k) {
            if (!ltouch[k]) continue;
            const uint32_t o = sp->orig[items[k]];
            touched[o] = 1;
            for (int q = 0; q < 9; ++q) acc[q * nn + o] += loc[q * count + k];
            if (L_mw[k] > acc[9 * nn + o]) acc[9 * nn + o] = L_mw[k];
        }
    }
    free(loc); free(ltouch); free(cb);
}

int or_backward_prepared(const or_prepared* sp, int64_t n, int64_t n_orig, int p, int ox, int oy,
                         int W, int H, const float* bg, const float* dLdC, or_screen_grads* screen) {
    pattern_t pt;
    if (make_pattern(p, ox, oy, W, H, &pt)) return 1;
    stage_t st;
    stage_from_prepared(sp, n, W, H, &st);
    const size_t nn = (size_t)(n_orig ? n_orig : 1);
    float* acc = (float*)calloc(10 * nn, sizeof(float));
    uint8_t* touched = (uint8_t*)calloc(nn, 1);
    backward_stage(&st, &pt, bg, dLdC, acc, touched, nn);
    float* dst[10] = {screen->gmx, screen->gmy, screen->gs00, screen->gs01, screen->gs11,
                      screen->galpha, screen->gc0, screen->gc1, screen->gc2, screen->maxw};
    for (int q = 0; q < 10; ++q)
        if (dst[q]) memcpy(dst[q], acc + q * nn, sizeof(float) * (size_t)n_orig);
    if (screen->touched) memcpy(screen->touched, touched, (size_t)n_orig);
    free(acc); free(touched);
    free_stage(&st);
    return 0;
}

int or_backward(or_scene* s, int p, int ox, int oy, int W, int H, const float* bg,
                const float* dLdC, int lowpass_p, float* const* grads, or_screen_grads* screen,
                int update_stats) {
    pattern_t pt;
    if (make_pattern(p, ox, oy, W, H, &pt)) return 1;
    stage_t st;
    int rc = build_stage(s, lowpass_p > 0 ? lowpass_p : p, W, H, &st);
    if (rc) { free_stage(&st); return rc; }
    const int64_t n = s->n;
    const size_t nn = (size_t)(n ? n : 1);
    /* per-Gaussian merged sums: gmx gmy s00 s01 s11 alpha c0 c1 c2 maxw */
    float* acc = (float*)calloc(10 * nn, sizeof(float));
    uint8_t* touched = (uint8_t*)calloc(nn, 1);
    backward_stage(&st, &pt, bg, dLdC, acc, touched, nn);

    for (int q = 0; q < 9; ++q)
        for (int64_t i = 0; i < n; ++i) grads[q][i] = 0.f;
    for (int64_t i = 0; i < n; ++i) {
        if (!touched[i]) continue;
        const float m00 = acc[2 * nn + i], m01 = acc[3 * nn + i], m11 = acc[4 * nn + i];
        grads[0][i] = acc[0 * nn + i];
        grads[1][i] = acc[1 * nn + i];
        const float c = m_cosf(s->rot[i]);
        const float sn = m_sinf(s->rot[i]);
        const float a = m_expf(2.0f * s->lsx[i]);
        const float b = m_expf(2.0f * s->lsy[i]);
        const float cs = c * sn;
        const float amb = a - b;
        grads[2][i] = m00 * (-2.0f * cs * amb) + 2.0f * m01 * ((c * c - sn * sn) * amb) +
                      m11 * (2.0f * cs * amb);
        grads[3][i] = 2.0f * a * (m00 * c * c + 2.0f * m01 * cs + m11 * sn * sn);
        grads[4][i] = 2.0f * b * (m00 * sn * sn - 2.0f * m01 * cs + m11 * c * c);
        const float alpha = activate(s->rop[i]);
        grads[5][i] = acc[5 * nn + i] * (alpha * (1.0f - alpha));
        const float k0 = activate(s->cr[i]), k1 = activate(s->cg[i]), k2 = activate(s->cb[i]);
        grads[6][i] = acc[6 * nn + i] * (k0 * (1.0f - k0));
        grads[7][i] = acc[7 * nn + i] * (k1 * (1.0f - k1));
        grads[8][i] = acc[8 * nn + i] * (k2 * (1.0f - k2));
    }
    if (update_stats && s->pos_acc) {
        for (int64_t i = 0; i < n; ++i) {
            if (acc[9 * nn + i] > kMinVisitW) {
                const float gx = grads[0][i], gy = grads[1][i];
                const float r = grads[6][i], g = grads[7][i], b = grads[8][i];
                s->pos_acc[i] += sqrtf(gx * gx + gy * gy);
                s->col_acc[i] += sqrtf(r * r + g * g + b * b);
                s->accum[i] += 1;
                s->visit[i] += 1;
                s->window[i] += 1;
            }
        }
    }
    if (screen) {
        float* dst[10] = {screen->gmx, screen->gmy, screen->gs00, screen->gs01, screen->gs11,
                          screen->galpha, screen->gc0, screen->gc1, screen->gc2, screen->maxw};
        for (int q = 0; q < 10; ++q)
            if (dst[q]) memcpy(dst[q], acc + q * nn, sizeof(float) * (size_t)n);
        if (screen->touched) memcpy(screen->touched, touched, (size_t)n);
    }
    free(acc); free(touched);
    free_stage(&st);
    return 0;
}

/* ---------------------------------------------------------------- L1 loss */
/* compute_loss, SPEC.md:562-570 (source missing; restated). Dilated/plain L1 over the active
 * pixels: loss = sum |C - target| / (3P) (target read at the pixel's (x, y) in the full-size
 * W x H row-major RGB target); dL/dC = sign(C - target) / (3P), sign(0) = 0. The loss sum is
 * accumulated in double in rank order. */
double or_l1_loss(const float* rgb, int p, int ox, int oy, int W, int H, const float* target,
                  float* dLdC) {
    pattern_t pt;
    if (make_pattern(p, ox, oy, W, H, &pt)) return -1.0;
    const int64_t P = (int64_t)pt.cols * pt.rows;
    if (P == 0) return 0.0;
    const float scale = (float)(1.0 / (3.0 * (double)P));
    double sum = 0.0;
    for (int64_t r = 0; r < P; ++r) {
        const int x = ox + (int)(r % pt.cols) * p;
        const int y = oy + (int)(r / pt.cols) * p;
        for (int c = 0; c < 3; ++c) {
            const float d = rgb[3 * r + c] - target[3 * ((int64_t)y * W + x) + c];
            sum += fabs((double)d);
            if (dLdC) dLdC[3 * r + c] = d > 0.f ? scale : (d < 0.f ? -scale : 0.f);
        }
    }
    return sum / (3.0 * (double)P);
}

/* ---------------------------------------------------------------- L1 + SSIM (dense) */
/* compute_loss (loss.cpp is missing from the reference, restated): dense
 * iterations (p = 1) use L = (1 - lam) L1 + lam (1 - SSIM), dilated ones L1 only. SSIM is the
 * mean over pixels and channels of the 11x11 Gaussian-window (sigma 1.5, normalised) SSIM map
 * with zero padding and C1 = 0.01^2, C2 = 0.03^2 (the 3DGS convention the SPEC names for
 * lam = 0.2, DESIGN DECISIONS). Gradient (analytic, pinned by finite differences in
 * tests/test_spec_kats.py): with the local statistics mu, sigma^2, sigma_xy of the window at
 * pixel p and S = A1 A2 / (B1 B2),
 *   dSSIM/dx_q = (1/3P) [ (G*a)(q) + 2 x_q (G*b)(q) + y_q (G*c)(q) ]
 *   a = dS/dmu_x - 2 mu_x dS/dsxx - mu_y dS/dsxy,  b = dS/dsxx,  c = dS/dsxy.
 * Double precision throughout (this is the checker); float in / out. */
#define SSIM_R 5
static void ssim_window(double g[2 * SSIM_R + 1]) {
    double s = 0.0;
    for (int i = -SSIM_R; i <= SSIM_R; ++i) {
        g[i + SSIM_R] = exp(-(double)(i * i) / (2.0 * 1.5 * 1.5));
        s += g[i + SSIM_R];
    }
    for (int i = 0; i < 2 * SSIM_R + 1; ++i) g[i] /= s;
}

/* separable "same" convolution with zero padding */
static void ssim_conv(const double* in, double* out, double* tmp, int W, int H, const double* g) {
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double acc = 0.0;
            for (int k = -SSIM_R; k <= SSIM_R; ++k) {
                const int xx = x + k;
                if (xx >= 0 && xx < W) acc += g[k + SSIM_R] * in[(int64_t)y * W + xx];
            }
            tmp[(int64_t)y * W + x] = acc;
        }
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            double acc = 0.0;
            for (int k = -SSIM_R; k <= SSIM_R; ++k) {
                const int yy = y + k;
                if (yy >= 0 && yy < H) acc += g[k + SSIM_R] * tmp[(int64_t)yy * W + x];
            }
            out[(int64_t)y * W + x] = acc;
        }
}

double or_loss(const float* rgb, int p, int ox, int oy, int W, int H, const float* target,
               float lam, float* dLdC) {
    if (p != 1 || !(lam > 0.0f)) return or_l1_loss(rgb, p, ox, oy, W, H, target, dLdC);
    if (ox != 0 || oy != 0 || W < 1 || H < 1) return -1.0;
    const int64_t P = (int64_t)W * H;
    const double l1 = or_l1_loss(rgb, 1, 0, 0, W, H, target, dLdC);
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03, inv = 1.0 / (3.0 * (double)P);
    double g[2 * SSIM_R + 1];
    ssim_window(g);
    double* buf = (double*)malloc(sizeof(double) * (size_t)P * 14);
    double *x = buf, *y = x + P, *t = y + P, *mx = t + P, *my = mx + P, *exx = my + P, *eyy = exx + P,
           *exy = eyy + P, *a = exy + P, *b = a + P, *c = b + P, *ga = c + P, *gb = ga + P, *gc = gb + P;
    double ssim_sum = 0.0;
    for (int ch = 0; ch < 3; ++ch) {
        for (int64_t i = 0; i < P; ++i) {
            x[i] = rgb[3 * i + ch];
            y[i] = target[3 * i + ch];
        }
        ssim_conv(x, mx, t, W, H, g);
        ssim_conv(y, my, t, W, H, g);
        for (int64_t i = 0; i < P; ++i) a[i] = x[i] * x[i];
        ssim_conv(a, exx, t, W, H, g);
        for (int64_t i = 0; i < P; ++i) a[i] = y[i] * y[i];
        ssim_conv(a, eyy, t, W, H, g);
        for (int64_t i = 0; i < P; ++i) a[i] = x[i] * y[i];
        ssim_conv(a, exy, t, W, H, g);
        for (int64_t i = 0; i < P; ++i) {
            const double sxx = exx[i] - mx[i] * mx[i], syy = eyy[i] - my[i] * my[i];
            const double sxy = exy[i] - mx[i] * my[i];
            const double A1 = 2.0 * mx[i] * my[i] + C1, A2 = 2.0 * sxy + C2;
            const double B1 = mx[i] * mx[i] + my[i] * my[i] + C1, B2 = sxx + syy + C2;
            const double S = A1 * A2 / (B1 * B2);
            ssim_sum += S;
            const double dmu = 2.0 * my[i] * A2 / (B1 * B2) - 2.0 * mx[i] * S / B1;
            const double dsxx = -S / B2, dsxy = 2.0 * A1 / (B1 * B2);
            a[i] = dmu - 2.0 * mx[i] * dsxx - my[i] * dsxy;
            b[i] = dsxx;
            c[i] = dsxy;
        }
        if (dLdC) {
            ssim_conv(a, ga, t, W, H, g);
            ssim_conv(b, gb, t, W, H, g);
            ssim_conv(c, gc, t, W, H, g);
            for (int64_t i = 0; i < P; ++i) {
                const double dssim = inv * (ga[i] + 2.0 * x[i] * gb[i] + y[i] * gc[i]);
                const double d = (double)rgb[3 * i + ch] - (double)target[3 * i + ch];
                const double sgn = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0);
                dLdC[3 * i + ch] = (float)((1.0 - lam) * sgn * inv - lam * dssim);
            }
        }
    }
    free(buf);
    return (1.0 - lam) * l1 + lam * (1.0 - ssim_sum * inv);
}

/* ---------------------------------------------------------------- Adam */
/* optimizer step, SPEC.md:258-267,283-285 (source missing; restated), clamp_parameters
 * gaussian.hpp:105-116. Float arithmetic in this exact order (the GPU kernel mirrors it):
 *   m = b1*m + (1-b1)*g ; v = b2*v + ((1-b2)*g)*g ; mh = m/bc1 ; vh = v/bc2 ;
 *   theta = theta - (lr*mh) / (sqrtf(vh) + eps)
 * bc1 = 1 - b1^t, bc2 = 1 - b2^t computed in double then rounded (host side in the product).
 * LR groups: pos 1.6e-4*diag*0.01^(t/T) (double, rounded), rot 1e-3, log-scale 5e-3,
 * raw-opacity 5e-2, colour 2.5e-3. */
void or_adam_config(or_adam_cfg* c, int64_t step, int64_t total_steps, double diag) {
    c->beta1 = 0.9f;
    c->beta2 = 0.999f;
    c->eps = 1e-15f;
    const double frac = total_steps > 0 ? (double)step / (double)total_steps : 0.0;
    const float lr_pos = (float)(1.6e-4 * diag * pow(0.01, frac));
    c->lr[0] = c->lr[1] = lr_pos;
    c->lr[2] = 1e-3f;
    c->lr[3] = c->lr[4] = 5e-3f;
    c->lr[5] = 5e-2f;
    c->lr[6] = c->lr[7] = c->lr[8] = 2.5e-3f;
    c->bc1 = (float)(1.0 - pow(0.9, (double)step));
    c->bc2 = (float)(1.0 - pow(0.999, (double)step));
    /* clamp_parameters: lo = log(T(kMinScale)), hi = log(image_diagonal) in T = float */
    c->ls_lo = m_logf((float)kMinScale);
    c->ls_hi = m_logf((float)diag);
    c->raw_cap = (float)kRawCap;
}

static float clampf(float v, float lo, float hi) { return v < lo ? lo : (hi < v ? hi : v); }

void or_adam_step(or_scene* s, float* const* grads, float* const* m, float* const* v,
                  const or_adam_cfg* c) {
    float* th[9] = {s->px, s->py, s->rot, s->lsx, s->lsy, s->rop, s->cr, s->cg, s->cb};
    const float omb1 = 1.0f - c->beta1, omb2 = 1.0f - c->beta2;
    for (int q = 0; q < 9; ++q) {
        for (int64_t i = 0; i < s->n; ++i) {
            const float g = grads[q][i];
            const float mm = c->beta1 * m[q][i] + omb1 * g;
            const float vv = c->beta2 * v[q][i] + omb2 * g * g;
            m[q][i] = mm;
            v[q][i] = vv;
            const float mh = mm / c->bc1;
            const float vh = vv / c->bc2;
            th[q][i] = th[q][i] - (c->lr[q] * mh) / (sqrtf(vh) + c->eps);
        }
    }
    for (int64_t i = 0; i < s->n; ++i) {
        s->lsx[i] = clampf(s->lsx[i], c->ls_lo, c->ls_hi);
        s->lsy[i] = clampf(s->lsy[i], c->ls_lo, c->ls_hi);
        s->rop[i] = clampf(s->rop[i], -c->raw_cap, c->raw_cap);
        s->cr[i] = clampf(s->cr[i], -c->raw_cap, c->raw_cap);
        s->cg[i] = clampf(s->cg[i], -c->raw_cap, c->raw_cap);
        s->cb[i] = clampf(s->cb[i], -c->raw_cap, c->raw_cap);
    }
}

/* ---------------------------------------------------------------- densify */
/* densifier, SPEC.md:300-383 (source missing; restated). Defaults SPEC.md:365-370. */
void or_densify_config(or_densify_cfg* c, float tau_pos) {
    c->tau_pos = tau_pos;
    c->tau_color = 0.01f * tau_pos;
    c->opacity_mask_floor = 0.05f;
    c->opacity_prune_floor = 0.005f;
    c->color_branch_prob = 0.2f;
    c->tau_v_init = 5.0;
    /* inverse_activate<float>(0.1) gaussian.hpp:57-60: log(v / (1 - v)) */
    c->child_raw_opacity = m_logf(0.1f / (1.0f - 0.1f));
}

/* select_candidates SPEC.md:319-327: accum_count > 0 ∧ visit_count > tau_v ∧
 * activate(raw_o) >= floor ∧ (avg_pos > tau_pos ∨ (coin ∧ avg_col > tau_color)). Averages are
 * float divisions by (float)accum_count. */
int64_t or_select_candidates(const or_scene* s, const or_densify_cfg* c, int coin,
                             uint8_t* cand) {
    int64_t cnt = 0;
    for (int64_t i = 0; i < s->n; ++i) {
        uint8_t ok = 0;
        if (s->accum[i] > 0 && (double)s->visit[i] > s->tau_v[i] &&
            activate(s->rop[i]) >= c->opacity_mask_floor) {
            const float cntf = (float)s->accum[i];
            const float ap = s->pos_acc[i] / cntf;
            const float ac = s->col_acc[i] / cntf;
            ok = (ap > c->tau_pos) || (coin && ac > c->tau_color);
        }
        cand[i] = ok;
        cnt += ok;
    }
    return cnt;
}

/* spawn cap SPEC.md:332,336: keep the top budget_remaining candidates by averaged positional
 * norm, ties by lower index. */
static const float* g_key;
static int cmp_desc_key(const void* a, const void* b) {
    const int64_t i = *(const int64_t*)a, j = *(const int64_t*)b;
    if (g_key[i] != g_key[j]) return g_key[i] > g_key[j] ? -1 : 1;
    return i < j ? -1 : (i > j ? 1 : 0);
}

int64_t or_cap_candidates(const or_scene* s, uint8_t* cand, int64_t budget_remaining) {
    int64_t cnt = 0;
    for (int64_t i = 0; i < s->n; ++i) cnt += cand[i];
    if (budget_remaining < 0) budget_remaining = 0;
    if (cnt <= budget_remaining) return cnt;
    int64_t* idx = (int64_t*)malloc(sizeof(int64_t) * (size_t)cnt);
    float* key = (float*)malloc(sizeof(float) * (size_t)(s->n ? s->n : 1));
    int64_t w = 0;
    for (int64_t i = 0; i < s->n; ++i) {
        if (!cand[i]) continue;
        key[i] = s->pos_acc[i] / (float)s->accum[i];
        idx[w++] = i;
    }
    g_key = key;
    qsort(idx, (size_t)cnt, sizeof(int64_t), cmp_desc_key);
    for (int64_t i = budget_remaining; i < cnt; ++i) cand[idx[i]] = 0;
    free(idx);
    free(key);
    return budget_remaining;
}

/* spawn SPEC.md:329-337: one child per selected parent, parents visited in ascending index
 * order, children appended in that order. Per child, 3 draws from the trainer RNG:
 * u1, u2 -> point r=sqrt(u1), th=2*pi*u2 in the unit disk, mapped through R*S (parent 1-sigma
 * ellipse, double arithmetic, rounded to float at the end); then depth_key = (float)uniform.
 * log_scales - ln2 (float), rotation and colour copied, raw_opacity = inverse_activate(0.1),
 * id = next_id++, fresh stats, tau_v = tau_v_init, zero Adam moments.
 * Returns the number of children; they are written at [n, n + children). */
int64_t or_spawn(or_scene* s, int64_t capacity, const uint8_t* sel, or_pcg32* rng,
                 const or_densify_cfg* c, float* const* m, float* const* v) {
    const int64_t n0 = s->n;
    int64_t w = n0;
    const double two_pi = 6.28318530717958647692;
    const float ln2 = 0.693147180559945309f;
    for (int64_t i = 0; i < n0; ++i) {
        if (!sel[i]) continue;
        if (w >= capacity) break;
        const double u1 = or_pcg32_uniform(rng);
        const double u2 = or_pcg32_uniform(rng);
        const double dk = or_pcg32_uniform(rng);
        const double r = sqrt(u1), th = two_pi * u2;
        const double ex = r * cos(th), ey = r * sin(th);
        const double sx = exp((double)s->lsx[i]), sy = exp((double)s->lsy[i]);
        const double cr = cos((double)s->rot[i]), sr = sin((double)s->rot[i]);
        const double ddx = cr * sx * ex - sr * sy * ey;
        const double ddy = sr * sx * ex + cr * sy * ey;
        s->px[w] = (float)((double)s->px[i] + ddx);
        s->py[w] = (float)((double)s->py[i] + ddy);
        s->rot[w] = s->rot[i];
        s->lsx[w] = s->lsx[i] - ln2;
        s->lsy[w] = s->lsy[i] - ln2;
        s->rop[w] = c->child_raw_opacity;
        s->cr[w] = s->cr[i];
        s->cg[w] = s->cg[i];
        s->cb[w] = s->cb[i];
        s->depth[w] = (float)dk;
        s->id[w] = s->next_id++;
        s->pos_acc[w] = 0.f;
        s->col_acc[w] = 0.f;
        s->accum[w] = 0;
        s->visit[w] = 0;
        s->window[w] = 0;
        s->tau_v[w] = c->tau_v_init;
        if (m)
            for (int q = 0; q < 9; ++q) { m[q][w] = 0.f; v[q][w] = 0.f; }
        ++w;
    }
    s->n = w;
    return w - n0;
}

/* prune SPEC.md:339-347 + GaussianModel::compact model.hpp:77-103 (order-preserving, all
 * parallel arrays incl. Adam moments in lockstep). Removes activate(raw_o) <
 * floor. */
int64_t or_prune(or_scene* s, const or_densify_cfg* c, float* const* m, float* const* v) {
    int64_t w = 0;
    for (int64_t r = 0; r < s->n; ++r) {
        if (activate(s->rop[r]) < c->opacity_prune_floor) continue;
        if (w != r) {
            s->px[w] = s->px[r]; s->py[w] = s->py[r]; s->rot[w] = s->rot[r];
            s->lsx[w] = s->lsx[r]; s->lsy[w] = s->lsy[r]; s->rop[w] = s->rop[r];
            s->cr[w] = s->cr[r]; s->cg[w] = s->cg[r]; s->cb[w] = s->cb[r];
            s->depth[w] = s->depth[r]; s->id[w] = s->id[r];
            s->pos_acc[w] = s->pos_acc[r]; s->col_acc[w] = s->col_acc[r];
            s->accum[w] = s->accum[r]; s->visit[w] = s->visit[r]; s->window[w] = s->window[r];
            s->tau_v[w] = s->tau_v[r];
            if (m)
                for (int q = 0; q < 9; ++q) { m[q][w] = m[q][r]; v[q][w] = v[q][r]; }
        }
        ++w;
    }
    const int64_t removed = s->n - w;
    s->n = w;
    return removed;
}

/* DensifyStats::reset_accumulators model.hpp:35-39 */
void or_reset_accumulators(or_scene* s) {
    for (int64_t i = 0; i < s->n; ++i) {
        s->pos_acc[i] = 0.f;
        s->col_acc[i] = 0.f;
        s->accum[i] = 0;
    }
}

/* update_visit_thresholds SPEC.md:349-357: window visits < 5 => tau_v = max(1, tau_v/2);
 * window counters reset. */
void or_visit_audit(or_scene* s) {
    for (int64_t i = 0; i < s->n; ++i) {
        if (s->window[i] < 5) {
            double t = s->tau_v[i] * 0.5;
            s->tau_v[i] = t < 1.0 ? 1.0 : t;
        }
        s->window[i] = 0;
    }
}

/* One densify event (SPEC.md:575(3)): colour coin (one draw) -> select -> cap to
 * budget - count -> spawn -> prune -> reset accumulators. Returns the new count. */
int64_t or_densify_event(or_scene* s, int64_t capacity, const or_densify_cfg* c, int64_t budget,
                         or_pcg32* rng, float* const* m, float* const* v, int64_t* out_spawned,
                         int64_t* out_pruned, int64_t* out_candidates) {
    const int coin = or_pcg32_uniform(rng) < (double)c->color_branch_prob;
    uint8_t* cand = (uint8_t*)malloc((size_t)(s->n ? s->n : 1));
    const int64_t nc = or_select_candidates(s, c, coin, cand);
    int64_t remaining = budget - s->n;
    if (remaining < 0) remaining = 0;
    or_cap_candidates(s, cand, remaining);
    const int64_t sp = or_spawn(s, capacity, cand, rng, c, m, v);
    free(cand);
    const int64_t pr = or_prune(s, c, m, v);
    or_reset_accumulators(s);
    if (out_spawned) *out_spawned = sp;
    if (out_pruned) *out_pruned = pr;
    if (out_candidates) *out_candidates = nc;
    return s->n;
}

/* ---------------------------------------------------------------- budget controller */
/* BudgetController SPEC.md:385-472 (source missing; restated). Design decisions
 * warmup 100, refit every 100, window 200 pairs, alpha_base = mean of the
 * last 5 fitted alpha_history values, alpha = 1 before the first fit. eps = alpha_recent -
 * alpha_history (the [OP] update post-condition). */
void or_budget_init(or_budget* b, double n_init, double m_final) {
    memset(b, 0, sizeof(*b));
    b->n_init = n_init;
    b->m_final = m_final;
    b->m_adaptive = m_final;
    b->alpha = 1.0;
    b->alpha_base = 1.0;
    b->warmup_steps = 100;
    b->window_size = 200;
    b->refit_interval = 100;
    b->ma_depth = 5;
    b->lambda = 0.5;
    b->last_refit = -1;
}

void or_budget_free(or_budget* b) {
    free(b->log_t); free(b->log_ema); free(b->fits);
    b->log_t = b->log_ema = b->fits = NULL;
}

int or_budget_record_loss(or_budget* b, int64_t t, double loss) {
    if (!(loss > 0.0)) return 1;
    b->ema = b->has_ema ? 0.1 * loss + 0.9 * b->ema : loss;
    b->has_ema = 1;
    if (t > b->warmup_steps) {
        if (b->log_len == b->log_cap) {
            b->log_cap = b->log_cap ? 2 * b->log_cap : 256;
            b->log_t = (double*)realloc(b->log_t, sizeof(double) * (size_t)b->log_cap);
            b->log_ema = (double*)realloc(b->log_ema, sizeof(double) * (size_t)b->log_cap);
        }
        b->log_t[b->log_len] = (double)t;
        b->log_ema[b->log_len] = b->ema;
        ++b->log_len;
    }
    return 0;
}

/* fit_power_exponent SPEC.md:419-427: negated least-squares slope of log(y) on log(t). */
int or_fit_power_exponent(const double* t, const double* y, int64_t n, double* out) {
    if (n < 2) return 1;
    double sx = 0, sy = 0;
    for (int64_t i = 0; i < n; ++i) {
        sx += log(t[i]);
        sy += log(y[i]);
    }
    const double mx = sx / (double)n, my = sy / (double)n;
    double sxx = 0, sxy = 0;
    for (int64_t i = 0; i < n; ++i) {
        const double dx = log(t[i]) - mx;
        sxx += dx * dx;
        sxy += dx * (log(y[i]) - my);
    }
    if (!(sxx > 0.0)) return 1;
    *out = -(sxy / sxx);
    return 0;
}

/* update SPEC.md:429-437. */
void or_budget_update(or_budget* b, int64_t t) {
    if (t <= b->warmup_steps) return;
    if (b->last_refit >= 0 && t - b->last_refit < b->refit_interval) return;
    double a_hist, a_recent;
    if (or_fit_power_exponent(b->log_t, b->log_ema, b->log_len, &a_hist)) return;
    const int64_t w = b->log_len < b->window_size ? b->log_len : b->window_size;
    if (or_fit_power_exponent(b->log_t + (b->log_len - w), b->log_ema + (b->log_len - w), w,
                              &a_recent))
        return;
    b->last_refit = t;
    if (b->fit_len == b->fit_cap) {
        b->fit_cap = b->fit_cap ? 2 * b->fit_cap : 64;
        b->fits = (double*)realloc(b->fits, sizeof(double) * (size_t)b->fit_cap);
    }
    b->fits[b->fit_len++] = a_hist;
    const int64_t d = b->fit_len < b->ma_depth ? b->fit_len : b->ma_depth;
    double s = 0;
    for (int64_t i = b->fit_len - d; i < b->fit_len; ++i) s += b->fits[i];
    b->alpha_base = s / (double)d;
    const double rate = a_recent;
    if (rate > 0.05) {
        const double up = b->m_adaptive * 1.1, cap = 1.5 * b->m_final;
        b->m_adaptive = up < cap ? up : cap;
    } else if (rate < -0.05) {
        const double dn = b->m_adaptive * 0.9, flo = 0.5 * b->m_final;
        b->m_adaptive = dn > flo ? dn : flo;
    }
    const double eps = a_recent - a_hist;
    double a = b->alpha_base + b->lambda * tanh(eps);
    b->alpha = a < 0.1 ? 0.1 : (a > 2.0 ? 2.0 : a);
}

/* budget_at SPEC.md:439-447: round(N + (t^a - 1)/(100^a - 1) (M_adaptive - N)), t clamped
 * to [1, 100]. */
int64_t or_budget_at(const or_budget* b, double t) {
    if (t < 1.0) t = 1.0;
    if (t > 100.0) t = 100.0;
    const double frac = (pow(t, b->alpha) - 1.0) / (pow(100.0, b->alpha) - 1.0);
    return (int64_t)llround(b->n_init + frac * (b->m_adaptive - b->n_init));
}

/* t_norm mapping SPEC.md:456. */
double or_budget_t_norm(int64_t step, int64_t warmup, int64_t densify_end) {
    if (densify_end <= warmup) return 100.0;
    double t = 1.0 + 99.0 * (double)(step - warmup) / (double)(densify_end - warmup);
    return t < 1.0 ? 1.0 : (t > 100.0 ? 100.0 : t);
}
