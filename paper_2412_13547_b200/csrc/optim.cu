// Per-Gaussian kernels after the blend backward (sm_100a, HBM-bound streaming):
//
//  chain_kernel   merge of the per-(tile, splat) partials in a fixed order (the reference's
//                 tile-order merge, rasterizer.cpp:301-319), chain rule to raw parameters
//                 (rasterizer.cpp:321-346), densify statistics (rasterizer.cpp:348-359) and,
//                 in the fused fit step, the Adam update + clamp_parameters (SPEC.md:258-267,
//                 gaussian.hpp:105-116) — one pass over the Gaussian state instead of four.
//  adam_kernel    Adam with explicit gradients (tgsx_adam_step) or the mean of the batched
//                 step buffer (tgsx_apply_step, SPEC.md:269-277 accumulate).
//
// Bit-exactness: given identical screen-space sums / gradients, the chain rule and Adam round
// exactly like the C oracle (explicit _rn intrinsics, CR transcendentals).
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

namespace tgsx {

namespace {

__device__ __forceinline__ float clampf(float v, float lo, float hi) {
    return v < lo ? lo : (hi < v ? hi : v);
}

// Adam on one Gaussian's 9 components from preloaded state (theta, m, v loaded before the
// partial merge so their latency overlaps it); same rounding as adam_update.
__device__ __forceinline__ void adam_update_pre(float* __restrict__ params, float* __restrict__ m1,
                                                float* __restrict__ m2, int64_t cap, int64_t i,
                                                const float (&g)[9], const float (&th0)[9],
                                                const float (&mm0)[9], const float (&vv0)[9],
                                                const AdamCfg& c) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const int64_t o = (int64_t)q * cap + i;
        const float mm = fadd(fmul(c.b1, mm0[q]), fmul(c.omb1, g[q]));
        const float vv = fadd(fmul(c.b2, vv0[q]), fmul(fmul(c.omb2, g[q]), g[q]));
        m1[o] = mm;
        m2[o] = vv;
        const float mh = fdiv_pos(mm, c.bc1);
        const float vh = fdiv_pos(vv, c.bc2);
        float th = fsub(th0[q], fdiv_pos(fmul(c.lr[q], mh), fadd(fsqrt_nz(vh), c.eps)));
        if (q == 3 || q == 4) th = clampf(th, c.ls_lo, c.ls_hi);
        if (q >= 5) th = clampf(th, -c.raw_cap, c.raw_cap);
        params[o] = th;
    }
}

// Adam on one Gaussian's 9 components + clamp (mirrors oracle or_adam_step exactly).
__device__ __forceinline__ void adam_update(float* __restrict__ params, float* __restrict__ m1,
                                            float* __restrict__ m2, int64_t cap, int64_t i,
                                            const float (&g)[9], const AdamCfg& c) {
#pragma unroll
    for (int q = 0; q < 9; ++q) {
        const int64_t o = (int64_t)q * cap + i;
        const float mm = fadd(fmul(c.b1, m1[o]), fmul(c.omb1, g[q]));
        const float vv = fadd(fmul(c.b2, m2[o]), fmul(fmul(c.omb2, g[q]), g[q]));
        m1[o] = mm;
        m2[o] = vv;
        const float mh = fdiv_pos(mm, c.bc1);
        const float vh = fdiv_pos(vv, c.bc2);
        float th = params[o];
        th = fsub(th, fdiv_pos(fmul(c.lr[q], mh), fadd(fsqrt_nz(vh), c.eps)));
        if (q == 3 || q == 4) th = clampf(th, c.ls_lo, c.ls_hi);
        if (q >= 5) th = clampf(th, -c.raw_cap, c.raw_cap);
        params[o] = th;
    }
}

struct ChainParams {
    const float* params;
    float* params_w;
    int64_t cap, n;
    const uint32_t* rank_of;
    const uint32_t* perm;  // non-null: rows stored in blend order (perm[rank] = logical index)
    const uint32_t* pair_off;  // per rank: first partial slot
    const uint32_t* touched;   // per rank: tiles touched (= partial slots)
    Partials partial;
    float* screen;  // [10][cap] or null
    // stats
    float* pos_acc;
    float* col_acc;
    int32_t* accum;
    int64_t* visit;
    int64_t* window;
    int update_stats;
    // outputs
    int mode;  // 0 grads, 1 adam, 2 accumulate
    float* grads;   // [9][n] (mode 0)
    float* m1;
    float* m2;
    StepRec* step;  // [n] AoS (mode 2)
    int64_t i0, i1; // Gaussian (row) range of this launch (buckets of the pipelined batched step)
    AdamCfg adam;
    const unsigned* fault;  // graph-replayed steps (graph.cpp): non-zero => the step is a no-op
};

// The slot loop and the parameter / moment / statistics streams are latency-bound: every load
// that does not depend on the merge (raw parameters, Adam state, densify statistics) is issued
// before it, which needs ~80 registers — 3 blocks of 256 per SM (4 forces spills; measured C3
// 0.293 -> 0.278 ms with the statistics prefetched at 3 blocks, 6 blocks without prefetch 0.34 ms).
// MODE (= cp.mode) is a template parameter: the gradient-only and accumulate variants carry none
// of the Adam prefetch registers and keep 4 blocks per SM.
template <int MODE>
__global__ void __launch_bounds__(256, MODE == 1 ? 3 : 4) chain_kernel(ChainParams cp) {
    const int64_t i = cp.i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cp.i1) return;
    if (cp.fault && *reinterpret_cast<const volatile unsigned*>(cp.fault)) return;
    const int64_t cap = cp.cap;
    const float* __restrict__ params = cp.params;
    // independent loads first (memory-level parallelism): the raw parameters the chain rule
    // needs, then the dependent gather chain rank -> prepared record -> pair partials
    const float rot = __ldg(params + 2 * cap + i);
    const float lx = __ldg(params + 3 * cap + i), ly = __ldg(params + 4 * cap + i);
    const float rop = __ldg(params + 5 * cap + i);
    float raw_c[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) raw_c[k] = __ldg(params + (6 + k) * cap + i);
    // blend-ordered rows: row i is rank i and its pair slots follow row i-1's (streaming reads);
    // logical rows gather through rank_of. Outputs in logical order go to index `li`.
    const uint32_t r = cp.perm ? (uint32_t)i : __ldg(cp.rank_of + i);
    const int64_t li = cp.perm ? (int64_t)__ldg(cp.perm + i) : i;
    const uint32_t base = __ldg(cp.pair_off + r), cnt = __ldg(cp.touched + r);
    float s[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) s[k] = 0.f;
    // merge in tile order (rasterizer.cpp:301-319): the pair slots of one splat are contiguous
    const float4* __restrict__ pa = cp.partial.a + base;
    const float4* __restrict__ pb = cp.partial.b + base;
    const float2* __restrict__ pc = cp.partial.c + base;
    // fused Adam: its state streams (theta, m, v) do not depend on the merge; issue them first
    float th0[9], mm0[9], vv0[9];
    // densify statistics of a visited Gaussian: loaded up front as well (the increments below
    // would otherwise add a third dependent memory round trip after the merge)
    float pa0 = 0.f, ca0 = 0.f;
    int32_t ac0 = 0;
    int64_t vi0 = 0, wi0 = 0;
    if (cp.update_stats && MODE != 2 && cnt) {
        pa0 = cp.pos_acc[i];
        ca0 = cp.col_acc[i];
        ac0 = cp.accum[i];
        vi0 = cp.visit[i];
        wi0 = cp.window[i];
    }
    if (MODE == 1) {
#pragma unroll
        for (int q = 0; q < 9; ++q) {
            const int64_t o = (int64_t)q * cap + i;
            th0[q] = __ldg(params + o);
            mm0[q] = cp.m1[o];
            vv0[q] = cp.m2[o];
        }
    }
    // four / two slots per step (their loads in flight together); sums in slot order
    uint32_t t = 0;
    for (; t + 3 < cnt; t += 4) {
        float4 a[4], b[4];
        float2 c[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = pa[t + u];
            b[u] = pb[t + u];
            c[u] = pc[t + u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            s[0] += a[u].x; s[1] += a[u].y; s[2] += a[u].z; s[3] += a[u].w;
            s[4] += b[u].x; s[5] += b[u].y; s[6] += b[u].z; s[7] += b[u].w;
            s[8] += c[u].x;
            s[9] = fmaxf(s[9], c[u].y);
        }
    }
    for (; t + 1 < cnt; t += 2) {
        const float4 a0 = pa[t], b0 = pb[t], a1 = pa[t + 1], b1 = pb[t + 1];
        const float2 c0 = pc[t], c1 = pc[t + 1];
        s[0] += a0.x; s[1] += a0.y; s[2] += a0.z; s[3] += a0.w;
        s[4] += b0.x; s[5] += b0.y; s[6] += b0.z; s[7] += b0.w;
        s[8] += c0.x;
        s[9] = fmaxf(s[9], c0.y);
        s[0] += a1.x; s[1] += a1.y; s[2] += a1.z; s[3] += a1.w;
        s[4] += b1.x; s[5] += b1.y; s[6] += b1.z; s[7] += b1.w;
        s[8] += c1.x;
        s[9] = fmaxf(s[9], c1.y);
    }
    if (t < cnt) {
        const float4 a = pa[t], b = pb[t];
        const float2 c = pc[t];
        s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
        s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
        s[8] += c.x;
        s[9] = fmaxf(s[9], c.y);
    }
    if (cp.screen) {
#pragma unroll
        for (int k = 0; k < 10; ++k) cp.screen[k * cap + li] = s[k];
    }
    const bool visited = s[9] > 0.f;
    // chain rule (rasterizer.cpp:324-346)
    float g[9];
    g[0] = s[0];
    g[1] = s[1];
    {
        float sn, c;
        cr_sincosf(rot, &sn, &c);
        const float a = cr_expf(fmul(2.0f, lx));
        const float b = cr_expf(fmul(2.0f, ly));
        const float m00 = s[2], m01 = s[3], m11 = s[4];
        const float cs = fmul(c, sn);
        const float amb = fsub(a, b);
        // m00 * (-2 cs amb) + 2 m01 ((c c - s s) amb) + m11 (2 cs amb)
        g[2] = fadd(fadd(fmul(m00, fmul(fmul(-2.0f, cs), amb)),
                         fmul(fmul(2.0f, m01), fmul(fsub(fmul(c, c), fmul(sn, sn)), amb))),
                    fmul(m11, fmul(fmul(2.0f, cs), amb)));
        // 2 a (m00 c c + 2 m01 cs + m11 s s)
        g[3] = fmul(fmul(2.0f, a), fadd(fadd(fmul(fmul(m00, c), c), fmul(fmul(2.0f, m01), cs)),
                                        fmul(fmul(m11, sn), sn)));
        // 2 b (m00 s s - 2 m01 cs + m11 c c)
        g[4] = fmul(fmul(2.0f, b), fadd(fsub(fmul(fmul(m00, sn), sn), fmul(fmul(2.0f, m01), cs)),
                                        fmul(fmul(m11, c), c)));
        const float al = activate_cr(rop);
        g[5] = fmul(s[5], fmul(al, fsub(1.0f, al)));
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const float ck = activate_cr(raw_c[k]);
            g[6 + k] = fmul(s[6 + k], fmul(ck, fsub(1.0f, ck)));
        }
    }
    // densify statistics (rasterizer.cpp:350-358): norms of the position and raw-colour grads
    float pn = 0.f, cn = 0.f;
    if (visited) {
        pn = __fsqrt_rn(fadd(fmul(g[0], g[0]), fmul(g[1], g[1])));
        cn = __fsqrt_rn(fadd(fadd(fmul(g[6], g[6]), fmul(g[7], g[7])), fmul(g[8], g[8])));
    }
    if (MODE == 2) {
        // batched views: sums in view order; the three counters increment
        // together (rasterizer.cpp:352-357), so one visit count is carried
        StepRec r = cp.step[i];
        r.a.x += g[0]; r.a.y += g[1]; r.a.z += g[2]; r.a.w += g[3];
        r.b.x += g[4]; r.b.y += g[5]; r.b.z += g[6]; r.b.w += g[7];
        r.c.x += g[8];
        if (visited) {
            r.c.y += pn;
            r.c.z += cn;
            r.c.w += 1.0f;
        }
        cp.step[i] = r;
        return;
    }
    if (cp.update_stats && visited) {
        cp.pos_acc[i] = fadd(pa0, pn);
        cp.col_acc[i] = fadd(ca0, cn);
        cp.accum[i] = ac0 + 1;
        cp.visit[i] = vi0 + 1;
        cp.window[i] = wi0 + 1;
    }
    if (MODE == 0) {
#pragma unroll
        for (int q = 0; q < 9; ++q) cp.grads[q * cp.n + li] = g[q];
        return;
    }
    adam_update_pre(cp.params_w, cp.m1, cp.m2, cap, i, g, th0, mm0, vv0, cp.adam);
}

// grads != null: explicit gradients [9][n]; else the batched step buffer (AoS [n], mean over the
// batch, stats applied, record zeroed for the next batch). Rows [i0, i1).
__global__ void __launch_bounds__(256) adam_kernel(float* __restrict__ params, float* __restrict__ m1,
                                                   float* __restrict__ m2, int64_t cap, int64_t n,
                                                   int64_t i0, int64_t i1, const float* __restrict__ grads,
                                                   StepRec* __restrict__ step, float* pos_acc,
                                                   float* col_acc, int32_t* accum, int64_t* visit,
                                                   int64_t* window, AdamCfg c) {
    const int64_t i = i0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= i1) return;
    float g[9];
    if (step) {
        const StepRec r = step[i];
        const float s9[9] = {r.a.x, r.a.y, r.a.z, r.a.w, r.b.x, r.b.y, r.b.z, r.b.w, r.c.x};
#pragma unroll
        for (int q = 0; q < 9; ++q) g[q] = fdiv_pos(s9[q], c.batch);
        if (r.c.w > 0.f) {
            const int32_t cnt = (int32_t)r.c.w;
            pos_acc[i] = fadd(pos_acc[i], r.c.y);
            col_acc[i] = fadd(col_acc[i], r.c.z);
            accum[i] += cnt;
            visit[i] += cnt;
            window[i] += cnt;
        }
        const float4 z = make_float4(0.f, 0.f, 0.f, 0.f);
        step[i] = StepRec{z, z, z};
    } else {
#pragma unroll
        for (int q = 0; q < 9; ++q) g[q] = grads[q * n + i];
    }
    adam_update(params, m1, m2, cap, i, g, c);
}

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

}  // namespace

cudaError_t launch_chain(tgsx_ctx* ctx, tgsx_model* m, ChainMode mode, bool update_stats,
                         float* grads_out, const float* adam_cfg, int64_t i0, int64_t i1) {
    if (i1 < 0) i1 = m->n;
    if (i1 <= i0) return cudaSuccess;
    ChainParams cp{};
    cp.params = m->params.as<float>();
    cp.params_w = m->params.as<float>();
    cp.cap = m->cap;
    cp.n = m->n;
    cp.i0 = i0;
    cp.i1 = i1;
    cp.rank_of = m->rank_of.as<uint32_t>();
    cp.perm = m->blend_phys ? m->perm.as<uint32_t>() : nullptr;
    cp.pair_off = ctx->ws.pair_off.as<uint32_t>();
    cp.touched = ctx->ws.touched.as<uint32_t>();
    cp.partial = Partials::at(ctx->ws.partial.p, ctx->ws.pair_cap);
    // screen-space sums are kept only for the explicit backward (tgsx_stage_screen_grads)
    cp.screen = mode == ChainMode::kGrads ? m->screen.as<float>() : nullptr;
    cp.pos_acc = m->pos_acc.as<float>();
    cp.col_acc = m->col_acc.as<float>();
    cp.accum = m->accum.as<int32_t>();
    cp.visit = m->visit.as<int64_t>();
    cp.window = m->window.as<int64_t>();
    cp.update_stats = update_stats ? 1 : 0;
    cp.mode = mode == ChainMode::kGrads ? 0 : (mode == ChainMode::kAdam ? 1 : 2);
    cp.grads = grads_out;
    cp.m1 = m->m1.as<float>();
    cp.m2 = m->m2.as<float>();
    cp.step = m->step.as<StepRec>();
    if (adam_cfg) cp.adam = *reinterpret_cast<const AdamCfg*>(adam_cfg);
    cp.fault = ctx->graph_capturing ? ctx->graph_fault : nullptr;
    if (cp.mode == 1)
        chain_kernel<1><<<grid_for(i1 - i0, 256), 256, 0, ctx->stream>>>(cp);
    else if (cp.mode == 2)
        chain_kernel<2><<<grid_for(i1 - i0, 256), 256, 0, ctx->stream>>>(cp);
    else
        chain_kernel<0><<<grid_for(i1 - i0, 256), 256, 0, ctx->stream>>>(cp);
    ctx->launches++;
    return cudaGetLastError();
}

// Per-launch Adam hyper-parameters of a captured chain kernel node (graph.cpp): the node's
// ChainParams as captured with only `adam` replaced, for the next launches of `exec`.
cudaError_t chain_node_set_adam(cudaGraphExec_t exec, cudaGraphNode_t node, const AdamCfg& c) {
    cudaKernelNodeParams kp{};
    cudaError_t e = cudaGraphKernelNodeGetParams(node, &kp);
    if (e) return e;
    ChainParams cp = *reinterpret_cast<const ChainParams*>(kp.kernelParams[0]);
    cp.adam = c;
    void* args[1] = {&cp};
    kp.kernelParams = args;
    kp.extra = nullptr;
    return cudaGraphExecKernelNodeSetParams(exec, node, &kp);
}

cudaError_t launch_adam(tgsx_ctx* ctx, tgsx_model* m, const float* grads, const float* adam_cfg,
                        int batch_views, int64_t i0, int64_t i1) {
    if (i1 < 0) i1 = m->n;
    if (i1 <= i0) return cudaSuccess;
    AdamCfg c = *reinterpret_cast<const AdamCfg*>(adam_cfg);
    c.batch = (float)(batch_views > 0 ? batch_views : 1);
    adam_kernel<<<grid_for(i1 - i0, 256), 256, 0, ctx->stream>>>(
        m->params.as<float>(), m->m1.as<float>(), m->m2.as<float>(), m->cap, m->n, i0, i1, grads,
        grads ? nullptr : m->step.as<StepRec>(), m->pos_acc.as<float>(), m->col_acc.as<float>(),
        m->accum.as<int32_t>(), m->visit.as<int64_t>(), m->window.as<int64_t>(), c);
    ctx->launches++;
    return cudaGetLastError();
}

}  // namespace tgsx
