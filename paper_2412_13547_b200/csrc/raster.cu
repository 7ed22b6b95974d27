// Rasterization kernels of the fit hot path (sm_100a, FP32 pipe — no tensor cores: nothing
// here is a dense contraction).
//
//  preprocess_kernel   prepare_splats (rasterizer.cpp:23-46) + tile rectangle / tiles-touched
//                      count (rasterizer.cpp:74-91). One thread per Gaussian in model order
//                      (coalesced SoA reads), scattered 64-B record write to its blend rank.
//                      Bit-exact vs the CR oracle: explicit _rn float ops, FP64 transcendentals.
//  duplicate_kernel    key duplication: (tile, rank) pairs emitted in rank order; fuses the
//                      radix-sort digit histograms (saves one full read of the keys).
//  ranges_kernel       per-tile [start, end) of the sorted keys (== TileGrid::offsets).
//  forward_kernel      walk_pixel + render (rasterizer.cpp:108-136, 144-184): one CTA per
//                      16x16 tile, warps own 8x4 blocks of ACTIVE pixels (dilated variant is
//                      first-class: p selects the warp layout). Splat batches are staged in
//                      shared memory together with exact per-tile column/row box-test masks;
//                      each warp compacts the batch to the splats whose 3-sigma box touches its
//                      pixels, so the per-pixel box test becomes one bit test. Optional fused
//                      L1 loss epilogue.
//  backward_kernel     backward tile phase (rasterizer.cpp:234-292): back-to-front over the
//                      forward's per-pixel last contributor, T recovered as T_{i+1}/(1-sigma_i)
//                      with sigma recomputed bit-identically to the forward; the suffix S is the
//                      reference's exact running sum (rasterizer.cpp:267-287). Per-splat
//                      gradients are reduced across the warp with a transposed butterfly (14
//                      shuffles for 9 values), combined across warps in a fixed order in shared
//                      memory and written once per (tile, splat) to that pair's slot — no global
//                      atomics, deterministic (the reference's tile-order merge contract,
//                      SPEC.md:234).
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>

namespace tgsx {

namespace {

constexpr uint32_t kFull = 0xffffffffu;

// ------------------------------------------------------------------ preprocess
__global__ void __launch_bounds__(256) preprocess_kernel(
    const float* __restrict__ params, int64_t cap, int64_t n,
    const uint32_t* __restrict__ rank_of, int lowpass_p, int W, int H, int tiles_x,
    Prepared* __restrict__ prep, uint32_t* __restrict__ touched, unsigned long long* err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t rank = rank_of[i];
    const float px = params[i], py = params[cap + i], rot = params[2 * cap + i];
    const float lx = params[3 * cap + i], ly = params[4 * cap + i], rop = params[5 * cap + i];
    const float cr = params[6 * cap + i], cg = params[7 * cap + i], cb = params[8 * cap + i];
    // covariance_from_params (gaussian.hpp:63-78)
    if (!isfinite(rot) || !isfinite(lx) || !isfinite(ly)) {
        raise_error(err, rank, 1);
        touched[rank] = 0;
        return;
    }
    float sn, c;
    cr_sincosf(rot, &sn, &c);
    const float a = cr_expf(fmul(2.0f, lx));
    const float b = cr_expf(fmul(2.0f, ly));
    float s00 = fadd(fmul(fmul(c, c), a), fmul(fmul(sn, sn), b));
    const float s01 = fmul(fmul(c, sn), fsub(a, b));
    float s11 = fadd(fmul(fmul(sn, sn), a), fmul(fmul(c, c), b));
    // apply_lowpass (dilation.hpp:73-80), bump 0.3 + 0.5 (p - 1)
    const float bump = fadd(0.3f, fmul(0.5f, (float)(lowpass_p - 1)));
    s00 = fadd(s00, bump);
    s11 = fadd(s11, bump);
    // invert (gaussian.hpp:82-92)
    const float det = fsub(fmul(s00, s11), fmul(s01, s01));
    if (!(det > 0.0f) || !isfinite(det)) {
        raise_error(err, rank, 2);
        touched[rank] = 0;
        return;
    }
    Prepared o;
    o.a = make_float4(px, py, fdiv(s11, det), fdiv(-s01, det));
    const float rx = fmul(kCullSigmas, __fsqrt_rn(s00));
    const float ry = fmul(kCullSigmas, __fsqrt_rn(s11));
    o.b = make_float4(fdiv(s00, det), activate_cr(rop), rx, ry);
    o.c = make_float4(activate_cr(cr), activate_cr(cg), activate_cr(cb), __uint_as_float((uint32_t)i));
    int tx0, tx1, ty0, ty1;
    uint32_t tiles = 0;
    if (tile_rect(px, py, rx, ry, W, H, tx0, tx1, ty0, ty1)) {
        tiles = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
        o.d = make_uint4((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16),
                         0u, tiles);
    } else {
        o.d = make_uint4(0u, 0u, 0u, 0u);
    }
    prep[rank] = o;
    touched[rank] = tiles;
}

// ------------------------------------------------------------------ key duplication
__global__ void __launch_bounds__(256) duplicate_kernel(
    Prepared* __restrict__ prep, const uint32_t* __restrict__ pair_off, int64_t n, int tiles_x,
    int passes, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
    uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_h[3][256];
    for (int t = threadIdx.x; t < 3 * 256; t += blockDim.x) (&s_h[0][0])[t] = 0;
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) {
        const uint4 d = prep[r].d;
        if (d.w) {
            const uint32_t off = pair_off[r];
            prep[r].d.z = off;
            const int tx0 = d.x & 0xffff, tx1 = d.x >> 16, ty0 = d.y & 0xffff, ty1 = d.y >> 16;
            uint32_t o = off;
            for (int ty = ty0; ty <= ty1; ++ty) {
                for (int tx = tx0; tx <= tx1; ++tx) {
                    const uint32_t key = (uint32_t)(ty * tiles_x + tx);
                    keys[o] = key;
                    vals[o] = (uint32_t)r;
                    ++o;
                    for (int p = 0; p < passes; ++p) atomicAdd(&s_h[p][(key >> (8 * p)) & 0xff], 1u);
                }
            }
        }
    }
    __syncthreads();
    for (int t = threadIdx.x; t < passes * 256; t += blockDim.x) {
        const uint32_t c = (&s_h[0][0])[t];
        if (c) atomicAdd(&hist[t], c);
    }
}

__global__ void ranges_kernel(const uint32_t* __restrict__ keys, int64_t K, uint2* __restrict__ ranges) {
    const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= K) return;
    const uint32_t t = keys[s];
    if (s == 0 || keys[s - 1] != t) ranges[t].x = (uint32_t)s;
    if (s == K - 1 || keys[s + 1] != t) ranges[t].y = (uint32_t)(s + 1);
}

// ------------------------------------------------------------------ blend kernels
struct BlendParams {
    const uint2* ranges;
    const uint32_t* items;
    const Prepared* prep;
    int tiles_x, p, ox, oy, W, H, cols;
    float bg0, bg1, bg2;
    float* rgb;
    float* T;
    uint32_t* last;
    unsigned long long* counters;  // [1] blend ops, [2] evaluations
    // fused L1 (forward) / loss gradient input (backward)
    const float* target;
    float* dLdC;
    float* block_loss;
    float loss_scale;
    float4* partial;
};

// Per-lane pixel of the CTA's tile. Warps own 8x4 blocks of active pixels.
template <int NWX>
struct PixelMap {
    int x0, y0, x, y, cbit, rbit, rank;
    bool valid;
    __device__ __forceinline__ void init(const BlendParams& prm, int tile) {
        const int tx = tile % prm.tiles_x, ty = tile / prm.tiles_x;
        x0 = tx * kTile;
        y0 = ty * kTile;
        const int px1 = min(prm.W, x0 + kTile), py1 = min(prm.H, y0 + kTile);
        const int ax = first_active(x0, prm.ox, prm.p), ay = first_active(y0, prm.oy, prm.p);
        const int acols = ax < px1 ? (px1 - ax + prm.p - 1) / prm.p : 0;
        const int arows = ay < py1 ? (py1 - ay + prm.p - 1) / prm.p : 0;
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        const int lx = (warp % NWX) * 8 + (lane & 7);
        const int ly = (warp / NWX) * 4 + (lane >> 3);
        valid = lx < acols && ly < arows;
        x = ax + lx * prm.p;
        y = ay + ly * prm.p;
        cbit = valid ? x - x0 : 0;
        rbit = valid ? y - y0 : 0;
        rank = valid ? ((y - prm.oy) / prm.p) * prm.cols + (x - prm.ox) / prm.p : 0;
    }
};

// Exact per-tile box-test masks (rasterizer.cpp:116-118): bit c set iff
// |float(x0 + c) + 0.5 - mean| <= r, evaluated in float exactly like the reference.
__device__ __forceinline__ uint32_t box_mask(float m, float r, int base) {
    uint32_t mask = 0;
#pragma unroll
    for (int c = 0; c < kTile; ++c) {
        const float d = __fsub_rn(__fadd_rn((float)(base + c), 0.5f), m);
        mask |= (fabsf(d) <= r) ? (1u << c) : 0u;
    }
    return mask;
}

struct SplatSmem {
    float4 a;  // mean x, mean y, inv00, 2*inv01
    float4 b;  // inv11, alpha, r, g
    float2 c;  // b, mask bits (cols | rows << 16)
};

__device__ __forceinline__ void load_splat(const BlendParams& prm, uint32_t rank, int x0, int y0,
                                           float4& sa, float4& sb, float2& sc) {
    const Prepared& P = prm.prep[rank];
    const float4 a = P.a, b = P.b, c = P.c;
    const uint32_t mask = box_mask(a.x, b.z, x0) | (box_mask(a.y, b.w, y0) << 16);
    sa = make_float4(a.x, a.y, a.z, a.w * 2.0f);
    sb = make_float4(b.x, b.y, c.x, c.y);
    sc = make_float2(c.z, __uint_as_float(mask));
}

// Builds the warp's list of batch entries whose box touches the warp's pixels.
template <int BATCH>
__device__ __forceinline__ int build_warp_list(const float2* s_c, int bcount, uint32_t wmask,
                                               uint16_t* wlist, int pos_limit, int bstart) {
    const int lane = threadIdx.x & 31;
    int wcount = 0;
    for (int c0 = 0; c0 < bcount; c0 += 32) {
        const int j = c0 + lane;
        bool rel = false;
        if (j < bcount && bstart + j < pos_limit) {
            const uint32_t m = __float_as_uint(s_c[j].y);
            rel = (m & wmask & 0xffffu) && (m & wmask & 0xffff0000u);
        }
        const uint32_t bal = __ballot_sync(kFull, rel);
        if (rel) wlist[wcount + __popc(bal & lanemask_lt())] = (uint16_t)j;
        wcount += __popc(bal);
    }
    __syncwarp();
    return wcount;
}

template <int NWX, int NWY, int BATCH>
__global__ void __launch_bounds__(NWX * NWY * 32) forward_kernel(BlendParams prm) {
    constexpr int NW = NWX * NWY, NT = NW * 32;
    __shared__ float4 s_a[BATCH];
    __shared__ float4 s_b[BATCH];
    __shared__ float2 s_c[BATCH];
    __shared__ uint16_t s_list[NW][BATCH];
    __shared__ unsigned long long s_red[2][NW];
    __shared__ float s_loss[NW];

    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PixelMap<NWX> pm;
    pm.init(prm, tile);
    const uint32_t wmask = __reduce_or_sync(kFull, pm.valid ? ((1u << pm.cbit) | (1u << (16 + pm.rbit))) : 0u);
    const uint2 range = prm.ranges[tile];
    const int count = (int)(range.y - range.x);
    const float fx = (float)pm.x + 0.5f, fy = (float)pm.y + 0.5f;

    float T = 1.0f, C0 = 0.f, C1 = 0.f, C2 = 0.f;
    uint32_t last = 0, ops = 0;
    bool done = !pm.valid;
    bool warp_done = __all_sync(kFull, done);

    for (int bstart = 0; bstart < count; bstart += BATCH) {
        if (__syncthreads_and(warp_done)) break;
        const int bcount = min(BATCH, count - bstart);
        for (int j = threadIdx.x; j < bcount; j += NT) {
            float4 a, b;
            float2 c;
            load_splat(prm, prm.items[range.x + bstart + j], pm.x0, pm.y0, a, b, c);
            s_a[j] = a;
            s_b[j] = b;
            s_c[j] = c;
        }
        __syncthreads();
        if (warp_done) continue;
        const int wcount = build_warp_list<BATCH>(s_c, bcount, wmask, s_list[warp], 0x7fffffff, 0);
        for (int e = 0; e < wcount; ++e) {
            const int j = s_list[warp][e];
            const float2 c = s_c[j];
            const uint32_t m = __float_as_uint(c.y);
            if (!done && ((m >> pm.cbit) & (m >> (16 + pm.rbit)) & 1u)) {
                const float4 a = s_a[j];
                const float4 b = s_b[j];
                const float dx = __fsub_rn(fx, a.x);
                const float dy = __fsub_rn(fy, a.y);
                const float G = splat_gauss(a.z, a.w, b.x, dx, dy);
                const float sigma = __fmul_rn(b.y, G);
                const float w = __fmul_rn(sigma, T);
                C0 = __fmaf_rn(w, b.z, C0);
                C1 = __fmaf_rn(w, b.w, C1);
                C2 = __fmaf_rn(w, c.x, C2);
                T = __fmul_rn(T, __fsub_rn(1.0f, sigma));
                ++ops;
                last = (uint32_t)(bstart + j + 1);
                if (T < kTermT) done = true;
            }
            if (__all_sync(kFull, done)) {
                warp_done = true;
                break;
            }
        }
    }

    // epilogue: background, outputs, counters, fused L1
    float lsum = 0.f;
    if (pm.valid) {
        C0 = __fmaf_rn(T, prm.bg0, C0);
        C1 = __fmaf_rn(T, prm.bg1, C1);
        C2 = __fmaf_rn(T, prm.bg2, C2);
        const int r = pm.rank;
        if (prm.rgb) {
            prm.rgb[3 * r] = C0;
            prm.rgb[3 * r + 1] = C1;
            prm.rgb[3 * r + 2] = C2;
        }
        prm.T[r] = T;
        prm.last[r] = last;
        if (prm.target) {
            const float* t = prm.target + 3 * ((int64_t)pm.y * prm.W + pm.x);
            const float d0 = C0 - t[0], d1 = C1 - t[1], d2 = C2 - t[2];
            lsum = fabsf(d0) + fabsf(d1) + fabsf(d2);
            const float s = prm.loss_scale;
            prm.dLdC[3 * r] = d0 > 0.f ? s : (d0 < 0.f ? -s : 0.f);
            prm.dLdC[3 * r + 1] = d1 > 0.f ? s : (d1 < 0.f ? -s : 0.f);
            prm.dLdC[3 * r + 2] = d2 > 0.f ? s : (d2 < 0.f ? -s : 0.f);
        }
    }
    unsigned long long o = ops;
    unsigned long long ev = pm.valid ? (done ? last : (uint32_t)count) : 0u;
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        o += __shfl_xor_sync(kFull, o, s);
        ev += __shfl_xor_sync(kFull, ev, s);
        lsum += __shfl_xor_sync(kFull, lsum, s);
    }
    if (lane == 0) {
        s_red[0][warp] = o;
        s_red[1][warp] = ev;
        s_loss[warp] = lsum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long to = 0, te = 0;
        float tl = 0.f;
        for (int w = 0; w < NW; ++w) {
            to += s_red[0][w];
            te += s_red[1][w];
            tl += s_loss[w];
        }
        if (to) atomicAdd(&prm.counters[1], to);
        if (te) atomicAdd(&prm.counters[2], te);
        if (prm.block_loss) prm.block_loss[tile] = tl;
    }
}

// Transposed butterfly: v[0..7] -> lane 4k holds the warp total of v[k]; v8 plain.
__device__ __forceinline__ void warp_reduce9(float (&v)[9]) {
    const int lane = threadIdx.x & 31;
    {
        const bool up = lane & 16;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const float send = up ? v[k] : v[k + 4];
            const float keep = up ? v[k + 4] : v[k];
            v[k] = keep + __shfl_xor_sync(kFull, send, 16);
        }
    }
    {
        const bool up = lane & 8;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const float send = up ? v[k] : v[k + 2];
            const float keep = up ? v[k + 2] : v[k];
            v[k] = keep + __shfl_xor_sync(kFull, send, 8);
        }
    }
    {
        const bool up = lane & 4;
        const float send = up ? v[0] : v[1];
        const float keep = up ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(kFull, send, 4);
    }
    v[0] += __shfl_xor_sync(kFull, v[0], 2);
    v[0] += __shfl_xor_sync(kFull, v[0], 1);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) v[8] += __shfl_xor_sync(kFull, v[8], s);
}

__device__ __forceinline__ uint32_t pair_slot(const Prepared& P, int tx, int ty) {
    const uint4 d = P.d;
    const int tx0 = d.x & 0xffff, tx1 = d.x >> 16, ty0 = d.y & 0xffff;
    return d.z + (uint32_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
}

template <int NWX, int NWY, int BATCH>
__global__ void __launch_bounds__(NWX * NWY * 32) backward_kernel(BlendParams prm) {
    constexpr int NW = NWX * NWY, NT = NW * 32;
    __shared__ float4 s_a[BATCH];
    __shared__ float4 s_b[BATCH];
    __shared__ float2 s_c[BATCH];
    __shared__ uint32_t s_slot[BATCH];
    __shared__ uint32_t s_touch[BATCH];            // bit w: warp w wrote s_w[w][j]
    __shared__ float s_w[NW][BATCH][10];           // per-warp reduced partials (9 + visited)
    __shared__ uint16_t s_list[NW][BATCH];
    __shared__ uint32_t s_maxlast;

    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PixelMap<NWX> pm;
    pm.init(prm, tile);
    const int tx = tile % prm.tiles_x, ty = tile / prm.tiles_x;
    const uint32_t wmask = __reduce_or_sync(kFull, pm.valid ? ((1u << pm.cbit) | (1u << (16 + pm.rbit))) : 0u);
    const uint2 range = prm.ranges[tile];
    const int count = (int)(range.y - range.x);
    const float fx = (float)pm.x + 0.5f, fy = (float)pm.y + 0.5f;

    float T = 1.f, S0 = 0.f, S1 = 0.f, S2 = 0.f, g0 = 0.f, g1 = 0.f, g2 = 0.f;
    uint32_t last = 0;
    if (pm.valid) {
        T = prm.T[pm.rank];
        last = prm.last[pm.rank];
        g0 = prm.dLdC[3 * pm.rank];
        g1 = prm.dLdC[3 * pm.rank + 1];
        g2 = prm.dLdC[3 * pm.rank + 2];
        S0 = __fmul_rn(prm.bg0, T);
        S1 = __fmul_rn(prm.bg1, T);
        S2 = __fmul_rn(prm.bg2, T);
    }
    const uint32_t wlast = __reduce_max_sync(kFull, last);
    if (threadIdx.x == 0) s_maxlast = 0;
    __syncthreads();
    if (lane == 0) atomicMax(&s_maxlast, wlast);
    __syncthreads();
    const int maxlast = (int)s_maxlast;

    // list entries past every pixel's last contributor: zero partials
    for (int j = maxlast + threadIdx.x; j < count; j += NT) {
        const uint32_t slot = pair_slot(prm.prep[prm.items[range.x + j]], tx, ty);
        float4* dst = prm.partial + 3 * (size_t)slot;
        dst[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        dst[1] = make_float4(0.f, 0.f, 0.f, 0.f);
        dst[2] = make_float4(0.f, 0.f, 0.f, 0.f);
    }

    const int nb = (maxlast + BATCH - 1) / BATCH;
    for (int b = nb - 1; b >= 0; --b) {
        const int bstart = b * BATCH;
        const int bcount = min(BATCH, maxlast - bstart);
        __syncthreads();
        for (int j = threadIdx.x; j < bcount; j += NT) {
            const uint32_t rank = prm.items[range.x + bstart + j];
            float4 a, bb;
            float2 c;
            load_splat(prm, rank, pm.x0, pm.y0, a, bb, c);
            s_a[j] = a;
            s_b[j] = bb;
            s_c[j] = c;
            s_slot[j] = pair_slot(prm.prep[rank], tx, ty);
            s_touch[j] = 0u;
        }
        __syncthreads();
        const int wcount = build_warp_list<BATCH>(s_c, bcount, wmask, s_list[warp], (int)wlast, bstart);
        for (int e = wcount - 1; e >= 0; --e) {
            const int j = s_list[warp][e];
            const uint32_t pos = (uint32_t)(bstart + j);
            const float2 c = s_c[j];
            const uint32_t m = __float_as_uint(c.y);
            const bool act = pm.valid && pos < last && ((m >> pm.cbit) & (m >> (16 + pm.rbit)) & 1u);
            const uint32_t actm = __ballot_sync(kFull, act);
            if (!actm) continue;
            float v[9];
#pragma unroll
            for (int k = 0; k < 9; ++k) v[k] = 0.f;
            bool vis = false;
            if (act) {
                const float4 a = s_a[j];
                const float4 bb = s_b[j];
                const float dx = __fsub_rn(fx, a.x);
                const float dy = __fsub_rn(fy, a.y);
                const float G = splat_gauss(a.z, a.w, bb.x, dx, dy);
                const float sigma = __fmul_rn(bb.y, G);
                const float ir = __frcp_rn(__fsub_rn(1.0f, sigma));
                const float Ti = __fmul_rn(T, ir);
                const float w = Ti * sigma;
                const float c0 = bb.z, c1 = bb.w, c2 = c.x;
                v[6] = g0 * w;
                v[7] = g1 * w;
                v[8] = g2 * w;
                const float d0 = c0 * Ti - S0 * ir;
                const float d1 = c1 * Ti - S1 * ir;
                const float d2 = c2 * Ti - S2 * ir;
                const float dsig = g0 * d0 + g1 * d1 + g2 * d2;
                v[5] = dsig * G;
                const float dq = dsig * bb.y * -0.5f * G;
                const float i01 = 0.5f * a.w;
                const float adx = a.z * dx + i01 * dy;
                const float ady = i01 * dx + bb.x * dy;
                v[0] = -2.0f * dq * adx;
                v[1] = -2.0f * dq * ady;
                v[2] = -dq * adx * adx;
                v[3] = -dq * adx * ady;
                v[4] = -dq * ady * ady;
                S0 = __fmaf_rn(c0, w, S0);
                S1 = __fmaf_rn(c1, w, S1);
                S2 = __fmaf_rn(c2, w, S2);
                T = Ti;
                vis = w > kMinVisitW;
            }
            const bool anyvis = __any_sync(kFull, vis);
            warp_reduce9(v);
            float* dst = s_w[warp][j];
            if ((lane & 3) == 0) dst[lane >> 2] = v[0];
            if (lane == 1) {
                dst[8] = v[8];
                dst[9] = anyvis ? 1.0f : 0.0f;
                atomicOr(&s_touch[j], 1u << warp);
            }
        }
        __syncthreads();
        // fixed-order cross-warp combine, one write per (tile, splat) pair slot
        for (int j = threadIdx.x; j < bcount; j += NT) {
            float acc[10];
#pragma unroll
            for (int k = 0; k < 10; ++k) acc[k] = 0.f;
            const uint32_t touch = s_touch[j];
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                if (touch & (1u << w)) {
#pragma unroll
                    for (int k = 0; k < 9; ++k) acc[k] += s_w[w][j][k];
                    acc[9] = fmaxf(acc[9], s_w[w][j][9]);
                }
            }
            float4* dst = prm.partial + 3 * (size_t)s_slot[j];
            dst[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
            dst[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
            dst[2] = make_float4(acc[8], acc[9], 0.f, 0.f);
        }
    }
}

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

BlendParams make_params(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items) {
    Workspace& ws = ctx->ws;
    BlendParams prm{};
    prm.ranges = ws.ranges.as<uint2>();
    prm.items = items;
    prm.prep = ws.prep.as<Prepared>();
    prm.tiles_x = ws.tiles_x;
    prm.p = ra.p;
    prm.ox = ra.ox;
    prm.oy = ra.oy;
    prm.W = ra.W;
    prm.H = ra.H;
    prm.cols = ra.cols;
    prm.bg0 = ra.bg[0];
    prm.bg1 = ra.bg[1];
    prm.bg2 = ra.bg[2];
    prm.rgb = ws.rgb.as<float>();
    prm.T = ws.T.as<float>();
    prm.last = ws.last.as<uint32_t>();
    prm.counters = ws.counters.as<unsigned long long>();
    prm.dLdC = ws.dLdC.as<float>();
    prm.block_loss = ws.block_loss.as<float>();
    prm.partial = ws.partial.as<float4>();
    return prm;
}

}  // namespace

int key_bits_for(int tiles) {
    int b = 0;
    while ((1ll << b) < (long long)tiles) ++b;
    return b;
}

cudaError_t launch_preprocess(tgsx_ctx* ctx, tgsx_model* m, int lowpass_p, int W, int H) {
    Workspace& ws = ctx->ws;
    const int64_t n = m->n;
    cudaError_t e;
    if ((e = ws.prep.ensure(std::max<int64_t>(n, 1) * sizeof(Prepared)))) return e;
    if ((e = ws.touched.ensure((n + 1) * 4))) return e;
    if ((e = ws.pair_off.ensure((n + 1) * 4))) return e;
    ws.tiles_x = (W + kTile - 1) / kTile;
    ws.tiles_y = (H + kTile - 1) / kTile;
    if (n == 0) return cudaSuccess;
    preprocess_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        m->params.as<float>(), m->cap, n, m->rank_of.as<uint32_t>(), lowpass_p, W, H, ws.tiles_x,
        ws.prep.as<Prepared>(), ws.touched.as<uint32_t>(), ws.counters.as<unsigned long long>());
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_duplicate(tgsx_ctx* ctx, tgsx_model* m, int W, int H, int key_bits) {
    Workspace& ws = ctx->ws;
    const int64_t n = m->n;
    (void)W;
    (void)H;
    const int passes = (key_bits + 7) / 8;
    cudaError_t e;
    // histogram lives at the head of sort_tmp (sort_pairs reads it from there)
    if ((e = ws.sort_tmp.ensure(4 * 256 * 4))) return e;
    if ((e = cudaMemsetAsync(ws.sort_tmp.p, 0, 4 * 256 * 4, ctx->stream))) return e;
    if (n == 0 || ws.K == 0) return cudaSuccess;
    duplicate_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        ws.prep.as<Prepared>(), ws.pair_off.as<uint32_t>(), n, ws.tiles_x, passes,
        ws.keys[0].as<uint32_t>(), ws.vals[0].as<uint32_t>(), ws.sort_tmp.as<uint32_t>());
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_ranges(tgsx_ctx* ctx, const uint32_t* keys, int64_t K, int tiles) {
    Workspace& ws = ctx->ws;
    cudaError_t e;
    if ((e = ws.ranges.ensure((size_t)std::max(tiles, 1) * sizeof(uint2)))) return e;
    if ((e = cudaMemsetAsync(ws.ranges.p, 0, (size_t)tiles * sizeof(uint2), ctx->stream))) return e;
    if (K == 0) return cudaSuccess;
    ranges_kernel<<<grid_for(K, 256), 256, 0, ctx->stream>>>(keys, K, ws.ranges.as<uint2>());
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_forward(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items,
                           bool fused_loss) {
    Workspace& ws = ctx->ws;
    BlendParams prm = make_params(ctx, ra, items);
    if (fused_loss) {
        prm.target = ra.target;
        prm.loss_scale = ra.P > 0 ? (float)(1.0 / (3.0 * (double)ra.P)) : 0.f;
    } else {
        prm.target = nullptr;
        prm.block_loss = nullptr;
    }
    const unsigned tiles = (unsigned)(ws.tiles_x * ws.tiles_y);
    if (ra.p == 1) {
        forward_kernel<2, 4, 256><<<tiles, 256, 0, ctx->stream>>>(prm);
    } else if (ra.p <= 3) {
        forward_kernel<1, 2, 128><<<tiles, 64, 0, ctx->stream>>>(prm);
    } else {
        forward_kernel<1, 1, 128><<<tiles, 32, 0, ctx->stream>>>(prm);
    }
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_backward(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items) {
    Workspace& ws = ctx->ws;
    BlendParams prm = make_params(ctx, ra, items);
    const unsigned tiles = (unsigned)(ws.tiles_x * ws.tiles_y);
    if (ra.p == 1) {
        backward_kernel<2, 4, 64><<<tiles, 256, 0, ctx->stream>>>(prm);
    } else if (ra.p <= 3) {
        backward_kernel<1, 2, 128><<<tiles, 64, 0, ctx->stream>>>(prm);
    } else {
        backward_kernel<1, 1, 128><<<tiles, 32, 0, ctx->stream>>>(prm);
    }
    ctx->launches++;
    return cudaGetLastError();
}

}  // namespace tgsx
