// Densification of the 3-D front end's model (BASELINE north_star item 4 on the 3-D path).
//
// The reference has only the 2-D densifier (densifier.cpp missing; restated in
// densify.cu / oracle/tgs_oracle.c). This is the same event on the 3-D parameters, restated in
// FP64 by oracle/ewa3d.c (or3d_densify_event) — parity is against that restatement, not against
// reference code:
//
//   colour coin (host draw)   -> select3d_kernel: accum = visit - visit_evt > 0, lifetime visits
//                                > tau_v, sigmoid(raw opacity) >= mask floor, averaged screen-space
//                                position norm > tau_pos OR (coin AND averaged SH-DC colour norm
//                                > tau_color)
//   over budget: top-k by averaged position norm, ties by lower index
//   spawn3d_kernel: one child per selected parent, appended in parent order; child j draws 3
//                uniforms from the trainer PCG32 advanced by 3j (the sequential draw order):
//                a point uniform in the parent's 1-sigma ELLIPSOID (radius cbrt(u1), direction
//                z = 1 - 2 u2, phi = 2 pi u3, mapped through R(q) diag(exp(log-scales))), the
//                3-D analogue of SPEC.md:333's 1-sigma ellipse; log-scales - ln 2, quaternion and
//                SH copied, opacity 0.1, fresh id / statistics / tau_v, zero Adam moments
//   prune: sigmoid(raw opacity) < prune floor, order-preserving compaction of every row group
//
//   reset: position / colour sums, visit_evt = visit                       (model.hpp:35-39)
// Rows stay in creation order (the 3-D blend order is per camera), so no reordering is needed.
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>
#include <cmath>
#include <string>

namespace tgsx {

namespace {

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

constexpr int kRowOpacity = 10;  // raw opacity row of the [59][cap] parameters
constexpr double kTauVInitDefault = 5.0;  // SPEC.md:367 (tgsx_densify_config_default)

struct Densify3Dev {
    float tau_pos, tau_color, mask_floor, prune_floor, child_rop;
    double tau_v_init;
};

struct Pcg3 {
    unsigned long long state, inc;
    __device__ void advance(unsigned long long delta) {
        unsigned long long cur_mult = 6364136223846793005ULL, cur_plus = inc;
        unsigned long long acc_mult = 1u, acc_plus = 0u;
        while (delta > 0) {
            if (delta & 1) {
                acc_mult *= cur_mult;
                acc_plus = acc_plus * cur_mult + cur_plus;
            }
            cur_plus = (cur_mult + 1) * cur_plus;
            cur_mult *= cur_mult;
            delta >>= 1;
        }
        state = acc_mult * state + acc_plus;
    }
    __device__ uint32_t next() {
        const unsigned long long old = state;
        state = old * 6364136223846793005ULL + inc;
        const uint32_t xs = (uint32_t)(((old >> 18u) ^ old) >> 27u);
        const uint32_t rot = (uint32_t)(old >> 59u);
        return (xs >> rot) | (xs << ((32u - rot) & 31u));
    }
    __device__ double uniform() { return (double)next() * 0x1p-32; }
};

__global__ void init_rows_kernel(unsigned long long* __restrict__ ids, double* __restrict__ tau_v, int64_t i0,
                                 int64_t i1, double tv) {
    const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= i1) return;
    ids[i] = (unsigned long long)i;
    tau_v[i] = tv;
}

__global__ void select3d_kernel(const float* __restrict__ params, int64_t cap, int64_t n,
                                const float* __restrict__ pos_acc, const float* __restrict__ col_acc,
                                const int32_t* __restrict__ visit, const int32_t* __restrict__ visit_evt,
                                const double* __restrict__ tau_v, Densify3Dev c, int coin,
                                uint32_t* __restrict__ flag, uint32_t* __restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t ok = 0;
    const int32_t cnt = visit[i] - visit_evt[i];
    float ap = 0.f;
    if (cnt > 0 && (double)visit[i] > tau_v[i] && activate_cr(params[kRowOpacity * cap + i]) >= c.mask_floor) {
        const float cf = (float)cnt;
        ap = fdiv_pos(pos_acc[i], cf);
        const float ac = fdiv_pos(col_acc[i], cf);
        ok = (ap > c.tau_pos) || (coin && ac > c.tau_color);
    }
    flag[i] = ok;
    key[i] = ~orderable_key(ap);  // descending average => ascending complement
}

__global__ void compact_candidates3d(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                     const uint32_t* __restrict__ key, int64_t n, uint32_t* __restrict__ ckey,
                                     uint32_t* __restrict__ cidx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    ckey[pos[i]] = key[i];
    cidx[pos[i]] = (uint32_t)i;
}

__global__ void mark_selected3d(const uint32_t* __restrict__ cidx, int64_t k, uint32_t* __restrict__ sel) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) sel[cidx[j]] = 1u;
}

__global__ void spawn3d_kernel(float* __restrict__ params, int64_t cap, int64_t n,
                               unsigned long long* __restrict__ ids, unsigned long long next_id,
                               double* __restrict__ tau_v, const uint32_t* __restrict__ sel,
                               const uint32_t* __restrict__ pos, Pcg3 base, Densify3Dev c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !sel[i]) return;
    const uint32_t j = pos[i];
    Pcg3 r = base;
    r.advance(3ull * j);
    const double u1 = r.uniform(), u2 = r.uniform(), u3 = r.uniform();
    const double two_pi = 6.28318530717958647692;
    // uniform point in the unit ball: radius cbrt(u1), direction uniform on the sphere
    const double rad = cbrt(u1);
    const double z = __dsub_rn(1.0, __dmul_rn(2.0, u2));
    const double rxy = sqrt(fmax(0.0, __dsub_rn(1.0, __dmul_rn(z, z))));
    const double ph = __dmul_rn(two_pi, u3);
    const double e0 = __dmul_rn(__dmul_rn(rad, rxy), cos(ph));
    const double e1 = __dmul_rn(__dmul_rn(rad, rxy), sin(ph));
    const double e2 = __dmul_rn(rad, z);
    // R(q) diag(s) e, q normalised (the forward's Sigma3 = (R S)(R S)^T)
    const double qw = params[3 * cap + i], qx = params[4 * cap + i], qy = params[5 * cap + i],
                 qz = params[6 * cap + i];
    const double qn = sqrt(__dadd_rn(__dadd_rn(__dmul_rn(qw, qw), __dmul_rn(qx, qx)),
                                     __dadd_rn(__dmul_rn(qy, qy), __dmul_rn(qz, qz))));
    const double w = __ddiv_rn(qw, qn), x = __ddiv_rn(qx, qn), y = __ddiv_rn(qy, qn), zq = __ddiv_rn(qz, qn);
    const double d0 = __dmul_rn(exp((double)params[7 * cap + i]), e0);
    const double d1 = __dmul_rn(exp((double)params[8 * cap + i]), e1);
    const double d2 = __dmul_rn(exp((double)params[9 * cap + i]), e2);
    const double R00 = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, y), __dmul_rn(zq, zq))));
    const double R01 = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, y), __dmul_rn(w, zq)));
    const double R02 = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, zq), __dmul_rn(w, y)));
    const double R10 = __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, y), __dmul_rn(w, zq)));
    const double R11 = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(zq, zq))));
    const double R12 = __dmul_rn(2.0, __dsub_rn(__dmul_rn(y, zq), __dmul_rn(w, x)));
    const double R20 = __dmul_rn(2.0, __dsub_rn(__dmul_rn(x, zq), __dmul_rn(w, y)));
    const double R21 = __dmul_rn(2.0, __dadd_rn(__dmul_rn(y, zq), __dmul_rn(w, x)));
    const double R22 = __dsub_rn(1.0, __dmul_rn(2.0, __dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y))));
    const double o0 = __dadd_rn(__dadd_rn(__dmul_rn(R00, d0), __dmul_rn(R01, d1)), __dmul_rn(R02, d2));
    const double o1 = __dadd_rn(__dadd_rn(__dmul_rn(R10, d0), __dmul_rn(R11, d1)), __dmul_rn(R12, d2));
    const double o2 = __dadd_rn(__dadd_rn(__dmul_rn(R20, d0), __dmul_rn(R21, d1)), __dmul_rn(R22, d2));
    const int64_t wr = n + j;
    const float ln2 = 0.693147180559945309f;
    params[wr] = (float)__dadd_rn((double)params[i], o0);
    params[cap + wr] = (float)__dadd_rn((double)params[cap + i], o1);
    params[2 * cap + wr] = (float)__dadd_rn((double)params[2 * cap + i], o2);
#pragma unroll
    for (int k = 3; k < 7; ++k) params[k * cap + wr] = params[k * cap + i];
#pragma unroll
    for (int k = 7; k < 10; ++k) params[k * cap + wr] = fsub(params[k * cap + i], ln2);
    params[kRowOpacity * cap + wr] = c.child_rop;
    for (int k = 11; k < k3dParams; ++k) params[k * cap + wr] = params[k * cap + i];
    ids[wr] = next_id + j;
    tau_v[wr] = c.tau_v_init;
}

__global__ void keep3d_kernel(const float* __restrict__ params, int64_t cap, int64_t n, float floor_,
                              uint32_t* __restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keep[i] = activate_cr(params[kRowOpacity * cap + i]) < floor_ ? 0u : 1u;
}

template <typename T>
__global__ void compact_rows3d(const T* __restrict__ src, T* __restrict__ dst, int64_t cap, int64_t n, int rows,
                               const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !keep[i]) return;
    const uint32_t w = pos[i];
    for (int q = 0; q < rows; ++q) dst[q * cap + w] = src[q * cap + i];
}

__global__ void audit3d_kernel(const int32_t* __restrict__ visit, int32_t* __restrict__ visit_aud,
                               double* __restrict__ tau_v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (visit[i] - visit_aud[i] < 5) {
        const double t = tau_v[i] * 0.5;
        tau_v[i] = t < 1.0 ? 1.0 : t;
    }
    visit_aud[i] = visit[i];
}

cudaError_t scan_count3d(tgsx_ctx* ctx, const uint32_t* flags, uint32_t* pos, int64_t n, uint64_t* total) {
    uint32_t* d_total = reinterpret_cast<uint32_t*>(ctx->ws.counters.as<unsigned long long>() + 6);
    cudaError_t e = launch_exclusive_scan(ctx, flags, pos, n, d_total);
    if (e) return e;
    if ((e = cudaMemcpyAsync(ctx->ws.h_scratch + 32, d_total, 4, cudaMemcpyDeviceToHost, ctx->stream))) return e;
    if ((e = cudaStreamSynchronize(ctx->stream))) return e;
    *total = n ? (uint64_t)(uint32_t)ctx->ws.h_scratch[32] : 0;
    return cudaSuccess;
}

}  // namespace

}  // namespace tgsx

cudaError_t densify3d_init_rows(tgsx_ctx* ctx, tgsx_model3d* m, int64_t i0, int64_t i1) {
    if (i1 <= i0) return cudaSuccess;
    tgsx::init_rows_kernel<<<tgsx::grid_for(i1 - i0, 256), 256, 0, ctx->stream>>>(
        m->ids.as<unsigned long long>(), m->tau_v.as<double>(), i0, i1, tgsx::kTauVInitDefault);
    ctx->launches++;
    return cudaGetLastError();
}

using namespace tgsx;

#define D3CK(expr)                                                          \
    do {                                                                    \
        cudaError_t _e = (expr);                                            \
        if (_e != cudaSuccess) {                                            \
            ctx->err = std::string(#expr) + ": " + cudaGetErrorString(_e);  \
            return TGSX_ECUDA;                                              \
        }                                                                   \
    } while (0)

extern "C" {

int32_t tgsx_densify3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_densify_config* cfg, int64_t budget,
                       uint64_t rng_state[2], tgsx_densify_report* out) {
    if (!ctx || !m || !cfg || !rng_state) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (m->step_views != 0) {
        ctx->err = "tgsx_densify3d: a batched step is in progress (apply it first)";
        return TGSX_ESTATE;
    }
    StageTimer timer(ctx, kStDensify);
    ctx->bin_valid = false;
    const int64_t n0 = m->n;
    tgsx_densify_report rep{};
    const int coin = tgsx_pcg32_uniform(rng_state) < (double)cfg->color_branch_prob ? 1 : 0;
    rep.color_coin = coin;
    Densify3Dev dc;
    dc.tau_pos = cfg->tau_pos;
    dc.tau_color = 0.01f * cfg->tau_pos;
    dc.mask_floor = cfg->opacity_mask_floor;
    dc.prune_floor = cfg->opacity_prune_floor;
    {
        const float v = 0.1f / (1.0f - 0.1f);  // inverse_activate<float>(0.1), gaussian.hpp:57-60
        dc.child_rop = (float)std::log((double)v);
    }
    dc.tau_v_init = cfg->tau_v_init;
    Workspace& ws = ctx->ws;
    const int64_t nn = std::max<int64_t>(n0, 1);
    D3CK(ws.generic.ensure((size_t)nn * 4 * 7));
    uint32_t* flag = ws.generic.as<uint32_t>();
    uint32_t* pos = flag + nn;
    uint32_t* key = pos + nn;
    uint32_t* ck = key + nn;
    uint32_t* ci = ck + nn;
    uint32_t* ck2 = ci + nn;
    uint32_t* ci2 = ck2 + nn;
    uint64_t ncand = 0;
    if (n0) {
        select3d_kernel<<<grid_for(n0, 256), 256, 0, ctx->stream>>>(
            m->params.as<float>(), m->cap, n0, m->pos_acc.as<float>(), m->col_acc.as<float>(), m->visit.as<int32_t>(),
            m->visit_evt.as<int32_t>(), m->tau_v.as<double>(), dc, coin, flag, key);
        ctx->launches++;
        D3CK(cudaGetLastError());
        D3CK(scan_count3d(ctx, flag, pos, n0, &ncand));
    }
    rep.candidates = (int64_t)ncand;
    const int64_t remaining = std::max<int64_t>(0, budget - n0);
    int64_t nsel = (int64_t)ncand;
    if ((int64_t)ncand > remaining) {
        nsel = remaining;
        compact_candidates3d<<<grid_for(n0, 256), 256, 0, ctx->stream>>>(flag, pos, key, n0, ck, ci);
        ctx->launches++;
        uint32_t* kk = ck;
        uint32_t* vv = ci;
        D3CK(sort_pairs(ctx, kk, vv, ck2, ci2, (int64_t)ncand, 32, nullptr));
        D3CK(cudaMemsetAsync(flag, 0, n0 * 4, ctx->stream));
        if (nsel > 0) {
            mark_selected3d<<<grid_for(nsel, 256), 256, 0, ctx->stream>>>(vv, nsel, flag);
            ctx->launches++;
        }
        uint64_t chk = 0;
        D3CK(scan_count3d(ctx, flag, pos, n0, &chk));
    }
    if (nsel > 0) {
        if (n0 + nsel > m->cap) D3CK(model3d_grow(ctx, m, std::max<int64_t>(n0 + nsel, m->cap + m->cap / 2)));
        Pcg3 base{rng_state[0], rng_state[1]};
        spawn3d_kernel<<<grid_for(n0, 256), 256, 0, ctx->stream>>>(m->params.as<float>(), m->cap, n0,
                                                                    m->ids.as<unsigned long long>(), m->next_id,
                                                                    m->tau_v.as<double>(), flag, pos, base, dc);
        ctx->launches++;
        D3CK(cudaGetLastError());
        const int64_t cap = m->cap;
        D3CK(cudaMemsetAsync(m->pos_acc.as<float>() + n0, 0, nsel * 4, ctx->stream));
        D3CK(cudaMemsetAsync(m->col_acc.as<float>() + n0, 0, nsel * 4, ctx->stream));
        D3CK(cudaMemsetAsync(m->visit.as<int32_t>() + n0, 0, nsel * 4, ctx->stream));
        D3CK(cudaMemsetAsync(m->visit_evt.as<int32_t>() + n0, 0, nsel * 4, ctx->stream));
        D3CK(cudaMemsetAsync(m->visit_aud.as<int32_t>() + n0, 0, nsel * 4, ctx->stream));
        D3CK(cudaMemset2DAsync(m->m1.as<float>() + n0, cap * 4, 0, nsel * 4, k3dParams, ctx->stream));
        D3CK(cudaMemset2DAsync(m->m2.as<float>() + n0, cap * 4, 0, nsel * 4, k3dParams, ctx->stream));
        tgsx_pcg32_advance(rng_state, 3ull * (uint64_t)nsel);
        m->next_id += (uint64_t)nsel;
        m->n = n0 + nsel;
    }
    rep.spawned = nsel;
    const int64_t n1 = m->n;
    int64_t kept = n1;
    if (n1) {
        D3CK(ws.generic.ensure((size_t)n1 * 4 * 7));
        uint32_t* keep = ws.generic.as<uint32_t>();
        uint32_t* kpos = keep + n1;
        keep3d_kernel<<<grid_for(n1, 256), 256, 0, ctx->stream>>>(m->params.as<float>(), m->cap, n1, dc.prune_floor,
                                                                   keep);
        ctx->launches++;
        uint64_t k = 0;
        D3CK(scan_count3d(ctx, keep, kpos, n1, &k));
        kept = (int64_t)k;
        if (kept != n1) {
            const int64_t cap = m->cap;
            struct R {
                DevBuf* b;
                int rows;
                int elt;
            } rs[] = {{&m->params, k3dParams, 4}, {&m->m1, k3dParams, 4}, {&m->m2, k3dParams, 4},
                      {&m->pos_acc, 1, 4},        {&m->col_acc, 1, 4},    {&m->visit, 1, 4},
                      {&m->visit_evt, 1, 4},      {&m->visit_aud, 1, 4},  {&m->ids, 1, 8},
                      {&m->tau_v, 1, 8}};
            for (int i = 0; i < (int)(sizeof(rs) / sizeof(rs[0])); ++i) {
                const auto& r = rs[i];
                DevBuf& sp = m->spare[i];
                const size_t bytes = (size_t)r.rows * cap * r.elt;
                if (sp.bytes < bytes) {
                    D3CK(cudaStreamSynchronize(ctx->stream));
                    sp.release();
                    D3CK(cudaMalloc(&sp.p, bytes));
                    sp.bytes = bytes;
                }
                if (r.elt == 4)
                    compact_rows3d<uint32_t><<<grid_for(n1, 256), 256, 0, ctx->stream>>>(
                        r.b->as<uint32_t>(), sp.as<uint32_t>(), cap, n1, r.rows, keep, kpos);
                else
                    compact_rows3d<unsigned long long><<<grid_for(n1, 256), 256, 0, ctx->stream>>>(
                        r.b->as<unsigned long long>(), sp.as<unsigned long long>(), cap, n1, r.rows, keep, kpos);
                ctx->launches++;
                D3CK(cudaGetLastError());
                std::swap(r.b->p, sp.p);
                std::swap(r.b->bytes, sp.bytes);
            }
            m->n = kept;
        }
    }
    rep.pruned = n1 - kept;
    // reset the accumulators (model.hpp:35-39): sums, and the event mark of the visit count
    if (m->n) {
        D3CK(cudaMemsetAsync(m->pos_acc.p, 0, m->n * 4, ctx->stream));
        D3CK(cudaMemsetAsync(m->col_acc.p, 0, m->n * 4, ctx->stream));
        D3CK(cudaMemcpyAsync(m->visit_evt.p, m->visit.p, m->n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    // the packed [62][n] step buffer changes its stride with n: keep it zero
    D3CK(cudaMemsetAsync(m->step.p, 0, m->step.bytes, ctx->stream));
    D3CK(cudaStreamSynchronize(ctx->stream));
    rep.count_after = m->n;
    if (out) *out = rep;
    return TGSX_OK;
}

int32_t tgsx_visit_audit3d(tgsx_ctx* ctx, tgsx_model3d* m) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (m->n) {
        audit3d_kernel<<<grid_for(m->n, 256), 256, 0, ctx->stream>>>(m->visit.as<int32_t>(), m->visit_aud.as<int32_t>(),
                                                                     m->tau_v.as<double>(), m->n);
        ctx->launches++;
        D3CK(cudaGetLastError());
    }
    return TGSX_OK;
}

int32_t tgsx_model3d_download_state(tgsx_ctx* ctx, tgsx_model3d* m, uint64_t* ids, double* tau_v, int32_t* visit_evt,
                                    int32_t* visit_aud, uint64_t* next_id) {
    if (!ctx || !m) return TGSX_EINVAL;
    const int64_t n = m->n;
    cudaStream_t s = ctx->stream;
    if (n) {
        if (ids) D3CK(cudaMemcpyAsync(ids, m->ids.p, n * 8, cudaMemcpyDefault, s));
        if (tau_v) D3CK(cudaMemcpyAsync(tau_v, m->tau_v.p, n * 8, cudaMemcpyDefault, s));
        if (visit_evt) D3CK(cudaMemcpyAsync(visit_evt, m->visit_evt.p, n * 4, cudaMemcpyDefault, s));
        if (visit_aud) D3CK(cudaMemcpyAsync(visit_aud, m->visit_aud.p, n * 4, cudaMemcpyDefault, s));
    }
    if (next_id) *next_id = m->next_id;
    D3CK(cudaStreamSynchronize(s));
    return TGSX_OK;
}

}  // extern "C"
