// Densification on the device (densifier.cpp is missing from the reference,
// so the semantics are the SPEC's, restated identically in oracle/tgs_oracle.c):
//
//   colour coin (host draw)           -> select_kernel    (predicate)
//   exclusive scan of flags           -> count (the one host sync of the event)
//   over budget: stable radix sort of ~orderable(avg pos norm) over candidates in index order
//                = top-k by averaged positional norm, ties by lower index
//   spawn_kernel   one child per selected parent, appended in parent-index order; child j
//                  draws its 3 uniforms from the trainer PCG32 advanced by 3j (LCG jump-ahead),
//                  i.e. exactly the sequential draw order
//   prune          activate(raw_o) < floor -> one order-preserving
//                  stream compaction of every parallel array incl. Adam moments
//                  (GaussianModel::compact, model.hpp:77-103)
//   reset          DensifyStats::reset_accumulators (model.hpp:35-39)
// All predicates compare exactly like the oracle (CR activation, float averages, double tau_v),
// so selections are bit-exact given equal statistics.
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>
#include <cmath>
#include <vector>

namespace tgsx {

namespace {

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

struct DensifyDev {
    float tau_pos, tau_color, mask_floor, prune_floor;
    float child_rop;
    double tau_v_init;
};

__global__ void select_kernel(const float* __restrict__ params, int64_t cap, int64_t n,
                              const float* __restrict__ pos_acc, const float* __restrict__ col_acc,
                              const int32_t* __restrict__ accum, const int64_t* __restrict__ visit,
                              const double* __restrict__ tau_v, DensifyDev c, int coin,
                              uint32_t* __restrict__ flag, uint32_t* __restrict__ key) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t ok = 0;
    const int32_t cnt = accum[i];
    float ap = 0.f;
    if (cnt > 0 && (double)visit[i] > tau_v[i] && activate_cr(params[5 * cap + i]) >= c.mask_floor) {
        const float cf = (float)cnt;
        ap = fdiv_pos(pos_acc[i], cf);
        const float ac = fdiv_pos(col_acc[i], cf);
        ok = (ap > c.tau_pos) || (coin && ac > c.tau_color);
    }
    flag[i] = ok;
    // descending average => ascending complement of the orderable key
    key[i] = ~orderable_key(ap);
}

__global__ void compact_candidates(const uint32_t* __restrict__ flag, const uint32_t* __restrict__ pos,
                                   const uint32_t* __restrict__ key, int64_t n,
                                   uint32_t* __restrict__ ckey, uint32_t* __restrict__ cidx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !flag[i]) return;
    ckey[pos[i]] = key[i];
    cidx[pos[i]] = (uint32_t)i;
}

__global__ void mark_selected(const uint32_t* __restrict__ cidx, int64_t k, uint32_t* __restrict__ sel) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j < k) sel[cidx[j]] = 1u;
}

struct PcgDev {
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

__global__ void spawn_kernel(float* __restrict__ params, int64_t cap, int64_t n,
                             unsigned long long* __restrict__ ids, unsigned long long next_id,
                             double* __restrict__ tau_v, const uint32_t* __restrict__ sel,
                             const uint32_t* __restrict__ pos, PcgDev base, DensifyDev c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !sel[i]) return;
    const uint32_t j = pos[i];
    PcgDev r = base;
    r.advance(3ull * j);
    const double u1 = r.uniform(), u2 = r.uniform(), dk = r.uniform();
    const double two_pi = 6.28318530717958647692;
    const double rr = sqrt(u1), th = __dmul_rn(two_pi, u2);
    const double ex = __dmul_rn(rr, cos(th)), ey = __dmul_rn(rr, sin(th));
    const float px = params[i], py = params[cap + i], rot = params[2 * cap + i];
    const float lx = params[3 * cap + i], ly = params[4 * cap + i];
    const double sx = exp((double)lx), sy = exp((double)ly);
    const double cr = cos((double)rot), sr = sin((double)rot);
    const double ddx = __dsub_rn(__dmul_rn(__dmul_rn(cr, sx), ex), __dmul_rn(__dmul_rn(sr, sy), ey));
    const double ddy = __dadd_rn(__dmul_rn(__dmul_rn(sr, sx), ex), __dmul_rn(__dmul_rn(cr, sy), ey));
    const int64_t w = n + j;
    const float ln2 = 0.693147180559945309f;
    params[w] = (float)__dadd_rn((double)px, ddx);
    params[cap + w] = (float)__dadd_rn((double)py, ddy);
    params[2 * cap + w] = rot;
    params[3 * cap + w] = fsub(lx, ln2);
    params[4 * cap + w] = fsub(ly, ln2);
    params[5 * cap + w] = c.child_rop;
    params[6 * cap + w] = params[6 * cap + i];
    params[7 * cap + w] = params[7 * cap + i];
    params[8 * cap + w] = params[8 * cap + i];
    params[9 * cap + w] = (float)dk;
    ids[w] = next_id + j;
    tau_v[w] = c.tau_v_init;
}

__global__ void keep_kernel(const float* __restrict__ params, int64_t cap, int64_t n, float floor_,
                            uint32_t* __restrict__ keep) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    keep[i] = activate_cr(params[5 * cap + i]) < floor_ ? 0u : 1u;
}

// Order-preserving compaction of `rows` rows of stride cap (element size 4 or 8) into dst.
template <typename T>
__global__ void compact_rows(const T* __restrict__ src, T* __restrict__ dst, int64_t cap, int64_t n,
                             int rows, const uint32_t* __restrict__ keep, const uint32_t* __restrict__ pos) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n || !keep[i]) return;
    const uint32_t w = pos[i];
    for (int q = 0; q < rows; ++q) dst[q * cap + w] = src[q * cap + i];
}

__global__ void visit_audit_kernel(int64_t* __restrict__ window, double* __restrict__ tau_v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    if (window[i] < 5) {
        const double t = tau_v[i] * 0.5;
        tau_v[i] = t < 1.0 ? 1.0 : t;
    }
    window[i] = 0;
}

}  // namespace

}  // namespace tgsx

using namespace tgsx;

namespace {

#define DCK(expr)                                                               \
    do {                                                                        \
        cudaError_t _e = (expr);                                                \
        if (_e != cudaSuccess) {                                                \
            ctx->err = std::string(#expr) + ": " + cudaGetErrorString(_e);      \
            return TGSX_ECUDA;                                                  \
        }                                                                       \
    } while (0)

cudaError_t scan_count(tgsx_ctx* ctx, const uint32_t* flags, uint32_t* pos, int64_t n, uint64_t* total) {
    uint32_t* d_total = reinterpret_cast<uint32_t*>(ctx->ws.counters.as<unsigned long long>() + 6);
    cudaError_t e = launch_exclusive_scan(ctx, flags, pos, n, d_total);
    if (e) return e;
    if ((e = cudaMemcpyAsync(ctx->ws.h_scratch + 32, d_total, 4, cudaMemcpyDeviceToHost, ctx->stream))) return e;
    if ((e = cudaStreamSynchronize(ctx->stream))) return e;
    *total = n ? (uint64_t)(uint32_t)ctx->ws.h_scratch[32] : 0;
    return cudaSuccess;
}

}  // namespace

extern "C" {

void tgsx_densify_config_default(tgsx_densify_config* c) {
    // SPEC.md:365-370
    c->tau_pos = 2e-4f;
    c->opacity_mask_floor = 0.05f;
    c->opacity_prune_floor = 0.005f;
    c->color_branch_prob = 0.2f;
    c->tau_v_init = 5.0;
}

int32_t tgsx_densify(tgsx_ctx* ctx, tgsx_model* m, const tgsx_densify_config* cfg, int64_t budget,
                     uint64_t rng_state[2], tgsx_densify_report* out) {
    if (!ctx || !m || !cfg || !rng_state) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    StageTimer timer(ctx, kStDensify);
    // selection ties, spawn order and compaction follow the logical (creation) order
    DCK(model_to_logical_order(ctx, m));
    ctx->bin_valid = false;  // the model changes (and the scratch below overlaps the binning's)
    const int64_t n0 = m->n;
    tgsx_densify_report rep{};
    // colour coin: one draw per event
    const int coin = tgsx_pcg32_uniform(rng_state) < (double)cfg->color_branch_prob ? 1 : 0;
    rep.color_coin = coin;
    DensifyDev dc;
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
    // scratch: flag, pos, key (n each) + candidate key/idx ping-pong (n each x 4)
    const int64_t nn = std::max<int64_t>(n0, 1);
    DCK(ws.generic.ensure((size_t)nn * 4 * 7));
    uint32_t* flag = ws.generic.as<uint32_t>();
    uint32_t* pos = flag + nn;
    uint32_t* key = pos + nn;
    uint32_t* ck = key + nn;
    uint32_t* ci = ck + nn;
    uint32_t* ck2 = ci + nn;
    uint32_t* ci2 = ck2 + nn;
    uint64_t ncand = 0;
    if (n0) {
        select_kernel<<<grid_for(n0, 256), 256, 0, ctx->stream>>>(
            m->params.as<float>(), m->cap, n0, m->pos_acc.as<float>(), m->col_acc.as<float>(),
            m->accum.as<int32_t>(), m->visit.as<int64_t>(), m->tau_v.as<double>(), dc, coin, flag, key);
        ctx->launches++;
        DCK(cudaGetLastError());
        DCK(scan_count(ctx, flag, pos, n0, &ncand));
    }
    rep.candidates = (int64_t)ncand;
    const int64_t remaining = std::max<int64_t>(0, budget - n0);
    int64_t nsel = (int64_t)ncand;
    if ((int64_t)ncand > remaining) {
        nsel = remaining;
        compact_candidates<<<grid_for(n0, 256), 256, 0, ctx->stream>>>(flag, pos, key, n0, ck, ci);
        ctx->launches++;
        uint32_t* kk = ck;
        uint32_t* vv = ci;
        DCK(sort_pairs(ctx, kk, vv, ck2, ci2, (int64_t)ncand, 32, nullptr));
        DCK(cudaMemsetAsync(flag, 0, n0 * 4, ctx->stream));
        if (nsel > 0) {
            mark_selected<<<grid_for(nsel, 256), 256, 0, ctx->stream>>>(vv, nsel, flag);
            ctx->launches++;
        }
        uint64_t chk = 0;
        DCK(scan_count(ctx, flag, pos, n0, &chk));
    }
    // spawn
    if (nsel > 0) {
        // geometric capacity growth (x1.5) when the children do not fit
        if (n0 + nsel > m->cap) DCK(model_grow(ctx, m, std::max<int64_t>(n0 + nsel, m->cap + m->cap / 2)));
        PcgDev base{rng_state[0], rng_state[1]};
        spawn_kernel<<<grid_for(n0, 256), 256, 0, ctx->stream>>>(
            m->params.as<float>(), m->cap, n0, m->ids.as<unsigned long long>(), m->next_id,
            m->tau_v.as<double>(), flag, pos, base, dc);
        ctx->launches++;
        DCK(cudaGetLastError());
        const int64_t cap = m->cap;
        // fresh stats and zero moments for the children
        DCK(cudaMemsetAsync(m->pos_acc.as<float>() + n0, 0, nsel * 4, ctx->stream));
        DCK(cudaMemsetAsync(m->col_acc.as<float>() + n0, 0, nsel * 4, ctx->stream));
        DCK(cudaMemsetAsync(m->accum.as<int32_t>() + n0, 0, nsel * 4, ctx->stream));
        DCK(cudaMemsetAsync(m->visit.as<int64_t>() + n0, 0, nsel * 8, ctx->stream));
        DCK(cudaMemsetAsync(m->window.as<int64_t>() + n0, 0, nsel * 8, ctx->stream));
        DCK(cudaMemset2DAsync(m->m1.as<float>() + n0, cap * 4, 0, nsel * 4, 9, ctx->stream));
        DCK(cudaMemset2DAsync(m->m2.as<float>() + n0, cap * 4, 0, nsel * 4, 9, ctx->stream));
        DCK(cudaMemsetAsync(m->step.as<StepRec>() + n0, 0, nsel * sizeof(StepRec), ctx->stream));
        tgsx_pcg32_advance(rng_state, 3ull * (uint64_t)nsel);
        m->next_id += (uint64_t)nsel;
        m->n = n0 + nsel;
        m->order_dirty = true;
    }
    rep.spawned = nsel;
    // prune
    const int64_t n1 = m->n;
    int64_t kept = n1;
    if (n1) {
        const int64_t nn1 = n1;
        DCK(ws.generic.ensure((size_t)nn1 * 4 * 7));
        uint32_t* keep = ws.generic.as<uint32_t>();
        uint32_t* kpos = keep + nn1;
        keep_kernel<<<grid_for(n1, 256), 256, 0, ctx->stream>>>(m->params.as<float>(), m->cap, n1,
                                                               dc.prune_floor, keep);
        ctx->launches++;
        uint64_t k = 0;
        DCK(scan_count(ctx, keep, kpos, n1, &k));
        kept = (int64_t)k;
        if (kept != n1) {
            const int64_t cap = m->cap;
            struct R { DevBuf* b; int rows; int elt; } rs[] = {
                {&m->params, 10, 4}, {&m->ids, 1, 8}, {&m->pos_acc, 1, 4}, {&m->col_acc, 1, 4},
                {&m->accum, 1, 4}, {&m->visit, 1, 8}, {&m->window, 1, 8}, {&m->tau_v, 1, 8},
                {&m->m1, 9, 4}, {&m->m2, 9, 4}, {&m->step, 1, (int)sizeof(StepRec)}};
            // compact each row group into its spare (allocated once per capacity) and swap
            for (int i = 0; i < 11; ++i) {
                const auto& r = rs[i];
                DevBuf& sp = m->spare[i];
                const size_t bytes = (size_t)r.rows * cap * r.elt;
                if (sp.bytes < bytes) {
                    DCK(cudaStreamSynchronize(ctx->stream));
                    sp.release();
                    DCK(cudaMalloc(&sp.p, bytes));
                    sp.bytes = bytes;
                }
                if (r.elt == 4)
                    compact_rows<uint32_t><<<grid_for(n1, 256), 256, 0, ctx->stream>>>(
                        r.b->as<uint32_t>(), sp.as<uint32_t>(), cap, n1, r.rows, keep, kpos);
                else if (r.elt == (int)sizeof(StepRec))
                    compact_rows<StepRec><<<grid_for(n1, 256), 256, 0, ctx->stream>>>(
                        r.b->as<StepRec>(), sp.as<StepRec>(), cap, n1, 1, keep, kpos);
                else
                    compact_rows<unsigned long long><<<grid_for(n1, 256), 256, 0, ctx->stream>>>(
                        r.b->as<unsigned long long>(), sp.as<unsigned long long>(), cap, n1, r.rows, keep, kpos);
                ctx->launches++;
                DCK(cudaGetLastError());
                std::swap(r.b->p, sp.p);
                std::swap(r.b->bytes, sp.bytes);
            }
            m->n = kept;
            m->order_dirty = true;
        }
    }
    rep.pruned = n1 - kept;
    // reset accumulators (model.hpp:35-39)
    if (m->n) {
        DCK(cudaMemsetAsync(m->pos_acc.p, 0, m->n * 4, ctx->stream));
        DCK(cudaMemsetAsync(m->col_acc.p, 0, m->n * 4, ctx->stream));
        DCK(cudaMemsetAsync(m->accum.p, 0, m->n * 4, ctx->stream));
    }
    DCK(cudaStreamSynchronize(ctx->stream));
    rep.count_after = m->n;
    if (out) *out = rep;
    return TGSX_OK;
}

int32_t tgsx_visit_audit(tgsx_ctx* ctx, tgsx_model* m) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (m->n) {
        visit_audit_kernel<<<grid_for(m->n, 256), 256, 0, ctx->stream>>>(m->window.as<int64_t>(),
                                                                         m->tau_v.as<double>(), m->n);
        ctx->launches++;
        DCK(cudaGetLastError());
    }
    return TGSX_OK;
}

}  // extern "C"
