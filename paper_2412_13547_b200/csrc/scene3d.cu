// 3-D front end of the fit hot path (BASELINE.json north_star item 1):
// per-Gaussian EWA projection to a 2-D covariance, SH-degree-3 colour, near-plane / tile-rect
// culling, and the chain rule from the blend's screen-space sums back to the 3-D parameters,
// fused with Adam. Everything between the 2-D record and the screen-space sums — tile binning,
// blend forward / backward, L1 — is the 2-D path's own kernels unchanged (raster.cu, sort.cu,
// blend.cu): the 3-D front end produces the same 64-B Prepared records in blend order.
//
// The reference is 2-D only: this row follows the published 3DGS algorithm,
// restated in FP64 by oracle/ewa3d.c (parity unpinned at the reference; the oracle is pinned
// by formula known-answers and finite differences, tests/test_oracle3d.py).
//
//  preprocess3d_kernel  one thread per Gaussian, SoA [59][cap] reads (coalesced), writes the
//                       record in row order + the (depth key, row) pair for the blend sort
//  bin3d_kernel         one thread per blend rank after the depth sort: gathers the row's
//                       record into rank order, tile rectangle + slab slot claims (as the 2-D
//                       preprocess does), perm / rank_of
//  chain3d_kernel       one thread per Gaussian (row order): tile-order merge of the pair
//                       partials, chain rule to mean / quaternion / log-scales / opacity / 48 SH
//                       coefficients, densify statistics, fused Adam (or gradients out)
//
// FP32 throughout (contraction allowed): no bit-exactness claim except Adam given equal
// gradients (explicit _rn ops, the oracle's order).
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>

namespace tgsx {

namespace {

constexpr int kFillStride = 32;  // as raster.cu: one slot cursor per 128-B line
constexpr uint32_t kCulledKey = 0xffffffffu;

constexpr float SH_C0 = 0.28209479177387814f;
constexpr float SH_C1 = 0.4886025119029199f;
constexpr float SH_C2_0 = 1.0925484305920792f, SH_C2_1 = -1.0925484305920792f,
                SH_C2_2 = 0.31539156525252005f, SH_C2_3 = -1.0925484305920792f,
                SH_C2_4 = 0.5462742152960396f;
constexpr float SH_C3_0 = -0.5900435899266435f, SH_C3_1 = 2.890611442640554f,
                SH_C3_2 = -0.4570457994644658f, SH_C3_3 = 0.3731763325901154f,
                SH_C3_4 = -0.4570457994644658f, SH_C3_5 = 1.445305721320277f,
                SH_C3_6 = -0.5900435899266435f;

// Explicit _rn products / sums: the basis is evaluated by two kernels of the fused step
// (chain rule and Adam) and by the explicit-gradient path; no FMA contraction keeps them bitwise equal.
__device__ __forceinline__ void sh_basis(float x, float y, float z, float (&b)[16]) {
    const float xx = fmul(x, x), yy = fmul(y, y), zz = fmul(z, z);
    const float xy = fmul(x, y), yz = fmul(y, z), xz = fmul(x, z);
    b[0] = SH_C0;
    b[1] = fmul(-SH_C1, y);
    b[2] = fmul(SH_C1, z);
    b[3] = fmul(-SH_C1, x);
    b[4] = fmul(SH_C2_0, xy);
    b[5] = fmul(SH_C2_1, yz);
    b[6] = fmul(SH_C2_2, fsub(fsub(fmul(2.f, zz), xx), yy));
    b[7] = fmul(SH_C2_3, xz);
    b[8] = fmul(SH_C2_4, fsub(xx, yy));
    b[9] = fmul(fmul(SH_C3_0, y), fsub(fmul(3.f, xx), yy));
    b[10] = fmul(fmul(SH_C3_1, xy), z);
    b[11] = fmul(fmul(SH_C3_2, y), fsub(fsub(fmul(4.f, zz), xx), yy));
    b[12] = fmul(fmul(SH_C3_3, z), fsub(fsub(fmul(2.f, zz), fmul(3.f, xx)), fmul(3.f, yy)));
    b[13] = fmul(fmul(SH_C3_4, x), fsub(fsub(fmul(4.f, zz), xx), yy));
    b[14] = fmul(fmul(SH_C3_5, z), fsub(xx, yy));
    b[15] = fmul(fmul(SH_C3_6, x), fsub(xx, fmul(3.f, yy)));
}

// d/d(dir) of sum_k w_k b_k(dir) (dir components treated as independent)
__device__ __forceinline__ void sh_basis_grad(float x, float y, float z, const float (&w)[16],
                                              float& gx, float& gy, float& gz) {
    const float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    gx = -SH_C1 * w[3] + SH_C2_0 * y * w[4] - 2.f * SH_C2_2 * x * w[6] + SH_C2_3 * z * w[7] +
         2.f * SH_C2_4 * x * w[8] + 6.f * SH_C3_0 * xy * w[9] + SH_C3_1 * yz * w[10] -
         2.f * SH_C3_2 * xy * w[11] - 6.f * SH_C3_3 * xz * w[12] +
         SH_C3_4 * (4.f * zz - 3.f * xx - yy) * w[13] + 2.f * SH_C3_5 * xz * w[14] +
         SH_C3_6 * (3.f * xx - 3.f * yy) * w[15];
    gy = -SH_C1 * w[1] + SH_C2_0 * x * w[4] + SH_C2_1 * z * w[5] - 2.f * SH_C2_2 * y * w[6] -
         2.f * SH_C2_4 * y * w[8] + SH_C3_0 * (3.f * xx - 3.f * yy) * w[9] + SH_C3_1 * xz * w[10] +
         SH_C3_2 * (4.f * zz - xx - 3.f * yy) * w[11] - 6.f * SH_C3_3 * yz * w[12] -
         2.f * SH_C3_4 * xy * w[13] - 2.f * SH_C3_5 * yz * w[14] - 6.f * SH_C3_6 * xy * w[15];
    gz = SH_C1 * w[2] + SH_C2_1 * y * w[5] + 4.f * SH_C2_2 * z * w[6] + SH_C2_3 * x * w[7] +
         SH_C3_1 * xy * w[10] + 8.f * SH_C3_2 * yz * w[11] +
         SH_C3_3 * (6.f * zz - 3.f * xx - 3.f * yy) * w[12] + 8.f * SH_C3_4 * xz * w[13] +
         SH_C3_5 * (xx - yy) * w[14];
}

// Geometry of one Gaussian (everything the chain rule needs again).
struct Geo3 {
    float tc[3], iz, cxz, cyz;
    bool clx, cly;
    float T[2][3];
    float qn[4], qinv;
    float Rq[3][3], s[3], M[3][3];
    float S3[3][3];
    float s00, s01, s11;
};

// Returns false when culled by the near plane. Requires finite inputs.
__device__ __forceinline__ bool geometry(const Cam3& cam, float bump, const float (&mu)[3],
                                         const float (&q)[4], const float (&ls)[3], Geo3& g) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        g.tc[i] = cam.R[3 * i] * mu[0] + cam.R[3 * i + 1] * mu[1] + cam.R[3 * i + 2] * mu[2] + cam.t[i];
    if (!(g.tc[2] > cam.znear)) return false;
    g.iz = 1.0f / g.tc[2];
    const float rx = g.tc[0] * g.iz, ry = g.tc[1] * g.iz;
    g.clx = rx < -cam.limx || rx > cam.limx;
    g.cly = ry < -cam.limy || ry > cam.limy;
    g.cxz = fminf(fmaxf(rx, -cam.limx), cam.limx);
    g.cyz = fminf(fmaxf(ry, -cam.limy), cam.limy);
    const float J00 = cam.fx * g.iz, J02 = -cam.fx * g.cxz * g.iz;
    const float J11 = cam.fy * g.iz, J12 = -cam.fy * g.cyz * g.iz;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        g.T[0][j] = J00 * cam.R[j] + J02 * cam.R[6 + j];
        g.T[1][j] = J11 * cam.R[3 + j] + J12 * cam.R[6 + j];
    }
    const float qq = q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3];
    g.qinv = rsqrtf(qq);
    const float r = q[0] * g.qinv, x = q[1] * g.qinv, y = q[2] * g.qinv, z = q[3] * g.qinv;
    g.qn[0] = r; g.qn[1] = x; g.qn[2] = y; g.qn[3] = z;
    g.Rq[0][0] = 1.f - 2.f * (y * y + z * z); g.Rq[0][1] = 2.f * (x * y - r * z); g.Rq[0][2] = 2.f * (x * z + r * y);
    g.Rq[1][0] = 2.f * (x * y + r * z); g.Rq[1][1] = 1.f - 2.f * (x * x + z * z); g.Rq[1][2] = 2.f * (y * z - r * x);
    g.Rq[2][0] = 2.f * (x * z - r * y); g.Rq[2][1] = 2.f * (y * z + r * x); g.Rq[2][2] = 1.f - 2.f * (x * x + y * y);
#pragma unroll
    for (int j = 0; j < 3; ++j) g.s[j] = expf(ls[j]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j) g.M[i][j] = g.Rq[i][j] * g.s[j];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            g.S3[i][j] = g.M[i][0] * g.M[j][0] + g.M[i][1] * g.M[j][1] + g.M[i][2] * g.M[j][2];
    float U[2][3];
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            U[i][j] = g.T[i][0] * g.S3[0][j] + g.T[i][1] * g.S3[1][j] + g.T[i][2] * g.S3[2][j];
    g.s00 = U[0][0] * g.T[0][0] + U[0][1] * g.T[0][1] + U[0][2] * g.T[0][2] + bump;
    g.s01 = U[0][0] * g.T[1][0] + U[0][1] * g.T[1][1] + U[0][2] * g.T[1][2];
    g.s11 = U[1][0] * g.T[1][0] + U[1][1] * g.T[1][1] + U[1][2] * g.T[1][2] + bump;
    return true;
}

__device__ __forceinline__ void view_dir(const Cam3& cam, const float (&mu)[3], float (&d)[3],
                                         float& ilen) {
    const float dx = mu[0] - cam.C[0], dy = mu[1] - cam.C[1], dz = mu[2] - cam.C[2];
    ilen = rsqrtf(dx * dx + dy * dy + dz * dz);
    d[0] = dx * ilen;
    d[1] = dy * ilen;
    d[2] = dz * ilen;
}

__device__ __forceinline__ float sigmoidf(float x) { return 1.0f / (1.0f + expf(-x)); }

// ------------------------------------------------------------------ preprocess
// One Gaussian (row i): the 2-D record (d left zero) and its orderable depth key. Returns false
// when culled (near plane) or invalid (error raised).
__device__ __forceinline__ bool prepare3d_one(const float* __restrict__ params, int64_t cap, int64_t i,
                                              const Cam3& cam, float bump, Prepared& o, uint32_t& key,
                                              unsigned long long* err) {
    key = kCulledKey;
    o.d = make_uint4(0u, 0u, 0u, 0u);
    float mu[3], q[4], ls[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) mu[k] = __ldg(params + k * cap + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = __ldg(params + (3 + k) * cap + i);
#pragma unroll
    for (int k = 0; k < 3; ++k) ls[k] = __ldg(params + (7 + k) * cap + i);
    const float rop = __ldg(params + 10 * cap + i);
    float sh[48];
    bool finite = isfinite(rop);
#pragma unroll
    for (int k = 0; k < 48; ++k) {
        sh[k] = __ldg(params + (11 + k) * cap + i);
        finite &= isfinite(sh[k]);
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) finite &= isfinite(mu[k]) && isfinite(ls[k]);
#pragma unroll
    for (int k = 0; k < 4; ++k) finite &= isfinite(q[k]);
    finite &= (q[0] != 0.f || q[1] != 0.f || q[2] != 0.f || q[3] != 0.f);
    if (!finite) {
        raise_error(err, (uint32_t)i, 1);
        return false;
    }
    Geo3 g;
    if (!geometry(cam, bump, mu, q, ls, g)) return false;
    const float det = g.s00 * g.s11 - g.s01 * g.s01;
    if (!(det > 0.0f) || !isfinite(det)) {
        raise_error(err, (uint32_t)i, 2);
        return false;
    }
    float d[3], ilen;
    view_dir(cam, mu, d, ilen);
    float b[16];
    sh_basis(d[0], d[1], d[2], b);
    float rgb[3];
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float acc = 0.5f;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += b[k] * sh[3 * k + c];
        rgb[c] = fmaxf(acc, 0.0f);
    }
    const float idet = 1.0f / det;
    o.a = make_float4(cam.fx * g.tc[0] * g.iz + cam.cx, cam.fy * g.tc[1] * g.iz + cam.cy,
                      g.s11 * idet, -g.s01 * idet);
    o.b = make_float4(g.s00 * idet, sigmoidf(rop), kCullSigmas * sqrtf(g.s00),
                      kCullSigmas * sqrtf(g.s11));
    o.c = make_float4(rgb[0], rgb[1], rgb[2], __uint_as_float((uint32_t)i));
    key = __float_as_uint(g.tc[2]) | 0x80000000u;  // positive depth: orderable key
    return true;
}

// Tile rectangle of a visible record into o.d (rect packed, tiles); returns the tile count.
__device__ __forceinline__ uint32_t rect3d(Prepared& o, int W, int H) {
    int tx0, tx1, ty0, ty1;
    if (!tile_rect(o.a.x, o.a.y, o.b.z, o.b.w, W, H, tx0, tx1, ty0, ty1)) {
        o.d = make_uint4(0u, 0u, 0u, 0u);
        return 0;
    }
    const uint32_t tiles = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
    o.d = make_uint4((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16), 0u, tiles);
    return tiles;
}

// Slab claims of one record (the 2-D preprocess's claim loop), slot value `v`.
__device__ __forceinline__ void claim3d(const uint4& d, int tiles_x, uint32_t v, uint32_t* __restrict__ fill,
                                        uint32_t* __restrict__ slab) {
    const int tx0 = d.x & 0xffff, tx1 = d.x >> 16, ty0 = d.y & 0xffff;
    const int w = tx1 - tx0 + 1, cnt = (int)d.w;
    for (int q0 = 0; q0 < cnt; q0 += 4) {
        uint32_t pos[4], tt[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (q0 + u < cnt) {
                const int q = q0 + u;
                tt[u] = (uint32_t)((ty0 + q / w) * tiles_x + tx0 + q % w);
                pos[u] = atomicAdd(&fill[(size_t)tt[u] * kFillStride], 1u);
            }
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (q0 + u < cnt && pos[u] < (uint32_t)kSegCap) slab[(size_t)tt[u] * kSegCap + pos[u]] = v;
    }
}

// Global-sort path: records in row order + (depth key, row) pairs for the blend sort.
__global__ void __launch_bounds__(256) preprocess3d_kernel(
    const float* __restrict__ params, int64_t cap, int64_t n, Cam3 cam, float bump,
    Prepared* __restrict__ prep_row, uint32_t* __restrict__ keys, uint32_t* __restrict__ vals,
    unsigned long long* err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    vals[i] = (uint32_t)i;
    Prepared o;
    uint32_t key;
    if (prepare3d_one(params, cap, i, cam, bump, o, key, err)) prep_row[i] = o;
    keys[i] = key;
}

// Per-tile path (no global sort): records stay in ROW order; every visible row claims its slab
// slots with its row index, the pair-offset scan runs fused (blocks in dispatch order), and the
// per-tile warp sort (seg_sort3d_kernel) orders each list by (depth key, row) — the blend order
// restricted to the tile, which is all the blend kernels read.
__global__ void __launch_bounds__(256, 3) preprocess3d_bin_kernel(
    const float* __restrict__ params, int64_t cap, int64_t n, Cam3 cam, float bump, int W, int H,
    int tiles_x, Prepared* __restrict__ prep, uint32_t* __restrict__ keys, uint32_t* __restrict__ touched,
    uint32_t* __restrict__ pair_off, uint32_t* __restrict__ fill, uint32_t* __restrict__ slab,
    unsigned long long* err, unsigned long long* status, uint32_t* ticket, uint32_t* d_total) {
    const uint32_t bid = lookback_block(ticket);
    const int64_t i = (int64_t)bid * 256 + threadIdx.x;
    Prepared o;
    uint32_t key = kCulledKey, tiles = 0;
    bool live = false;
    if (i < n) {
        live = prepare3d_one(params, cap, i, cam, bump, o, key, err);
        if (live) tiles = rect3d(o, W, H);
    }
    const uint32_t excl = block_scan_lookback(tiles, bid, n, status, d_total);
    if (i < n) {
        o.d.z = excl;
        if (live) prep[i] = o;
        else prep[i].d = make_uint4(0u, 0u, excl, 0u);
        keys[i] = key;
        touched[i] = tiles;
        pair_off[i] = excl;
        // claims after the scan: the block barrier never waits on their atomics
        if (tiles) claim3d(o.d, tiles_x, (uint32_t)i, fill, slab);
    }
}

// Bitonic sort of 32*E 64-bit keys held by one warp (lane L owns positions L*E .. L*E+E-1).
template <int E>
__device__ __forceinline__ void warp_bitonic64(unsigned long long (&x)[E], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {
                const int lm = j / E;
                const bool lower = (lane & lm) == 0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const unsigned long long y = __shfl_xor_sync(0xffffffffu, x[e], lm);
                    const bool asc = ((lane * E + e) & k) == 0;
                    x[e] = (asc == lower) ? min(x[e], y) : max(x[e], y);
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if ((e & j) == 0) {
                        const bool asc = ((lane * E + e) & k) == 0;
                        const unsigned long long a = x[e], b = x[e | j];
                        x[e] = asc ? min(a, b) : max(a, b);
                        x[e | j] = asc ? max(a, b) : min(a, b);
                    }
                }
            }
        }
    }
}

template <int E>
__device__ __forceinline__ void warp_sort_rows(uint32_t* __restrict__ list, int n, const uint32_t* __restrict__ keys,
                                               int lane) {
    unsigned long long x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int t = lane * E + e;
        if (t < n) {
            const uint32_t row = list[t];
            x[e] = ((unsigned long long)__ldg(keys + row) << 32) | row;
        } else {
            x[e] = ~0ull;
        }
    }
    warp_bitonic64<E>(x, lane);
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (lane * E + e < n) list[lane * E + e] = (uint32_t)x[e];
}

// One warp per tile: the tile's rows (claimed in arbitrary order) sorted by (depth key, row).
template <int MAXE>
__global__ void __launch_bounds__(256) seg_sort3d_kernel(const uint2* __restrict__ ranges, int tiles,
                                                         uint32_t* __restrict__ items,
                                                         const uint32_t* __restrict__ keys) {
    const int lane = threadIdx.x & 31;
    const int tile = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (tile >= tiles) return;
    const uint2 rg = ranges[tile];
    const int n = (int)(rg.y - rg.x);
    uint32_t* list = items + rg.x;
    if (n <= 1) return;
    // three network sizes only: the fully unrolled 64-bit networks are large, and warps of one SM
    // running many different sizes thrash the instruction cache (ncu: no_instruction stalls)
    if (n <= 64) warp_sort_rows<2>(list, n, keys, lane);
    else if (MAXE <= 16 || n <= 512) warp_sort_rows<MAXE < 16 ? MAXE : 16>(list, n, keys, lane);
    else warp_sort_rows<MAXE>(list, n, keys, lane);
}

// ------------------------------------------------------------------ rank-order gather + binning
// One thread per blend rank (blocks in dispatch order): gathers the row's record, claims its slab
// slots like the 2-D preprocess, and runs the pair-offset scan fused in (block_scan_lookback):
// pair_off / touched / the record's first pair slot / the total K leave this kernel.
__global__ void __launch_bounds__(256) bin3d_kernel(
    const uint32_t* __restrict__ skeys, const uint32_t* __restrict__ svals, int64_t n,
    const Prepared* __restrict__ prep_row, int W, int H, int tiles_x, Prepared* __restrict__ prep,
    uint32_t* __restrict__ touched, uint32_t* __restrict__ pair_off, uint32_t* __restrict__ fill,
    uint32_t* __restrict__ slab, uint32_t* __restrict__ perm, uint32_t* __restrict__ rank_of,
    unsigned long long* status, uint32_t* ticket, uint32_t* d_total) {
    const uint32_t bid = lookback_block(ticket);
    const int64_t r = (int64_t)bid * 256 + threadIdx.x;
    Prepared o;
    o.d = make_uint4(0u, 0u, 0u, 0u);
    uint32_t tiles = 0;
    const bool live = r < n && skeys[r] != kCulledKey;
    if (r < n) {
        const uint32_t row = svals[r];
        perm[r] = row;
        rank_of[row] = (uint32_t)r;
        if (live) o = prep_row[row];
    }
    if (live) tiles = rect3d(o, W, H);
    const uint32_t excl = block_scan_lookback(tiles, bid, n, status, d_total);
    if (r < n) {
        o.d.z = excl;
        if (live) prep[r] = o;
        else prep[r].d = o.d;
        touched[r] = tiles;
        pair_off[r] = excl;
        if (tiles) claim3d(o.d, tiles_x, (uint32_t)r, fill, slab);
    }
}

// ------------------------------------------------------------------ chain rule (+ Adam)
__device__ __forceinline__ int adam3d_group(int k) {
    return k < 3 ? 0 : (k < 7 ? 1 : (k < 10 ? 2 : (k == 10 ? 3 : (k < 14 ? 4 : 5))));
}

// Adam on one component from loaded state (the oracle's or3d_adam_step order, explicit _rn ops).
__device__ __forceinline__ void adam3d_math(float& th, float& m, float& v, float g, float lr, bool clamp,
                                            const Adam3dCfg& c) {
    m = fadd(fmul(c.b1, m), fmul(c.omb1, g));
    v = fadd(fmul(c.b2, v), fmul(fmul(c.omb2, g), g));
    const float mh = fdiv_pos(m, c.bc1);
    const float vh = fdiv_pos(v, c.bc2);
    th = fsub(th, fdiv_pos(fmul(lr, mh), fadd(fsqrt_nz(vh), c.eps)));
    if (clamp) th = th < -c.raw_cap ? -c.raw_cap : (c.raw_cap < th ? c.raw_cap : th);
}

// Adam over components K0 .. K0+NK-1 of row i: all 3*NK loads issued before any store (the
// streams are independent; the restrict pointers let the loads run ahead).
template <int K0, int NK, typename GradFn>
__device__ __forceinline__ void adam3d_chunk(float* __restrict__ P, float* __restrict__ M1,
                                             float* __restrict__ M2, int64_t cap, int64_t i,
                                             GradFn grad, const Adam3dCfg& c) {
    float th[NK], m[NK], v[NK];
#pragma unroll
    for (int j = 0; j < NK; ++j) {
        const int64_t o = (int64_t)(K0 + j) * cap + i;
        th[j] = P[o];
        m[j] = M1[o];
        v[j] = M2[o];
    }
#pragma unroll
    for (int j = 0; j < NK; ++j) {
        adam3d_math(th[j], m[j], v[j], grad(K0 + j), c.lr[adam3d_group(K0 + j)], K0 + j == 10, c);
        const int64_t o = (int64_t)(K0 + j) * cap + i;
        P[o] = th[j];
        M1[o] = m[j];
        M2[o] = v[j];
    }
}

struct Chain3Params {
    float* params;
    int64_t cap, n;
    Cam3 cam;
    float bump;
    const uint32_t* rank_of;
    const uint32_t* pair_off;
    const uint32_t* touched;
    Partials partial;
    int mode;       // 0 gradients out, 1 fused Adam, 2 accumulate into the batched step buffer
    float* grads;   // [59][n] (mode 0)
    float* screen;  // [10][n] or null
    float* pos_acc;
    float* col_acc;
    int32_t* visit;
    int update_stats;
    float* gbuf;    // [17][n] (mode 1): gradients 0..10, masked colour gradient, view direction
    float* step;    // [62][n] packed (mode 2): 59 gradient sums, position-norm sum, colour-norm sum, visits
};

// Gradients of one Gaussian from its merged screen-space sums s[0..8]: the 11 geometric /
// opacity components into gg (rows 0..10), the SH gradients as b[k] * dcol[c] (rows 11+3k+c).
// Mirrors or3d_chain (oracle/ewa3d.c).
__device__ __forceinline__ void chain3d_grads(const Cam3& cam, const Geo3& g, const float (&mu)[3],
                                              float rop, const float* __restrict__ P, int64_t cap, int64_t i,
                                              const float (&s)[10], float (&gg)[11], float (&b)[16],
                                              float (&dcol)[3], float (&d)[3]) {
    // ---- colour: SH basis, raw colour, clamp mask, direction gradient
    float ilen;
    view_dir(cam, mu, d, ilen);
    sh_basis(d[0], d[1], d[2], b);
    float sh[48];
#pragma unroll
    for (int k = 0; k < 48; ++k) sh[k] = __ldg(P + (11 + k) * cap + i);
#pragma unroll
    for (int c = 0; c < 3; ++c) {
        float acc = 0.5f;
#pragma unroll
        for (int k = 0; k < 16; ++k) acc += b[k] * sh[3 * k + c];
        dcol[c] = acc < 0.f ? 0.f : s[6 + c];
    }
    float w[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) w[k] = dcol[0] * sh[3 * k] + dcol[1] * sh[3 * k + 1] + dcol[2] * sh[3 * k + 2];
    float gdx, gdy, gdz;
    sh_basis_grad(d[0], d[1], d[2], w, gdx, gdy, gdz);
    const float dd = gdx * d[0] + gdy * d[1] + gdz * d[2];
    const float dmu[3] = {(gdx - d[0] * dd) * ilen, (gdy - d[1] * dd) * ilen, (gdz - d[2] * dd) * ilen};
    // ---- opacity
    const float al = sigmoidf(rop);
    gg[10] = s[5] * al * (1.f - al);
    // ---- mean projection + EWA covariance
    const float fx = cam.fx, fy = cam.fy, iz = g.iz, iz2 = iz * iz;
    float dt[3];
    dt[0] = s[0] * fx * iz;
    dt[1] = s[1] * fy * iz;
    dt[2] = -(s[0] * fx * g.tc[0] + s[1] * fy * g.tc[1]) * iz2;
    const float G00 = s[2], G01 = s[3], G11 = s[4];
    float GT[2][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        GT[0][j] = G00 * g.T[0][j] + G01 * g.T[1][j];
        GT[1][j] = G01 * g.T[0][j] + G11 * g.T[1][j];
    }
    float dS3[3][3];
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) dS3[a][c] = g.T[0][a] * GT[0][c] + g.T[1][a] * GT[1][c];
    float dT[2][3];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            dT[a][j] = 2.f * (GT[a][0] * g.S3[0][j] + GT[a][1] * g.S3[1][j] + GT[a][2] * g.S3[2][j]);
    const float* R = cam.R;
    const float dJ00 = dT[0][0] * R[0] + dT[0][1] * R[1] + dT[0][2] * R[2];
    const float dJ02 = dT[0][0] * R[6] + dT[0][1] * R[7] + dT[0][2] * R[8];
    const float dJ11 = dT[1][0] * R[3] + dT[1][1] * R[4] + dT[1][2] * R[5];
    const float dJ12 = dT[1][0] * R[6] + dT[1][1] * R[7] + dT[1][2] * R[8];
    dt[2] += -fx * iz2 * dJ00 - fy * iz2 * dJ11;
    if (g.clx) {
        dt[2] += dJ02 * fx * g.cxz * iz2;
    } else {
        dt[0] -= dJ02 * fx * iz2;
        dt[2] += dJ02 * 2.f * fx * g.cxz * iz2;
    }
    if (g.cly) {
        dt[2] += dJ12 * fy * g.cyz * iz2;
    } else {
        dt[1] -= dJ12 * fy * iz2;
        dt[2] += dJ12 * 2.f * fy * g.cyz * iz2;
    }
#pragma unroll
    for (int j = 0; j < 3; ++j) gg[j] = R[j] * dt[0] + R[3 + j] * dt[1] + R[6 + j] * dt[2] + dmu[j];
    // ---- Σ3 = M Mᵀ, M = Rq diag(s)
    float dR[3][3];
#pragma unroll
    for (int j = 0; j < 3; ++j) {
        float ds = 0.f;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float dM = 2.f * (dS3[a][0] * g.M[0][j] + dS3[a][1] * g.M[1][j] + dS3[a][2] * g.M[2][j]);
            dR[a][j] = dM * g.s[j];
            ds += dM * g.Rq[a][j];
        }
        gg[7 + j] = ds * g.s[j];
    }
    const float qr = g.qn[0], qx = g.qn[1], qy = g.qn[2], qz = g.qn[3];
    float dq[4];
    dq[0] = 2.f * (-qz * dR[0][1] + qy * dR[0][2] + qz * dR[1][0] - qx * dR[1][2] - qy * dR[2][0] + qx * dR[2][1]);
    dq[1] = 2.f * (qy * dR[0][1] + qz * dR[0][2] + qy * dR[1][0] - 2.f * qx * dR[1][1] - qr * dR[1][2] +
                   qz * dR[2][0] + qr * dR[2][1] - 2.f * qx * dR[2][2]);
    dq[2] = 2.f * (-2.f * qy * dR[0][0] + qx * dR[0][1] + qr * dR[0][2] + qx * dR[1][0] + qz * dR[1][2] -
                   qr * dR[2][0] + qz * dR[2][1] - 2.f * qy * dR[2][2]);
    dq[3] = 2.f * (-2.f * qz * dR[0][0] - qr * dR[0][1] + qx * dR[0][2] + qr * dR[1][0] - 2.f * qz * dR[1][1] +
                   qy * dR[1][2] + qx * dR[2][0] + qy * dR[2][1]);
    const float qd = qr * dq[0] + qx * dq[1] + qy * dq[2] + qz * dq[3];
#pragma unroll
    for (int k = 0; k < 4; ++k) gg[3 + k] = (dq[k] - g.qn[k] * qd) * g.qinv;
}

// MODE (= cp.mode) as a template parameter: each variant keeps only its own output path live.
// The accumulate variant (batched multi-camera steps) runs at 3 blocks per SM (C7 chain 1.72 ->
// 1.57 ms per step); the fused variant keeps 2 (3 forces spills: C6 0.389 -> 0.41 ms).
template <int MODE>
__global__ void __launch_bounds__(256, MODE == 2 ? 3 : 2) chain3d_kernel(Chain3Params cp) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= cp.n) return;
    const int64_t cap = cp.cap;
    const float* __restrict__ P = cp.params;
    // per-tile path: pair slots by row; global-sort path: by blend rank
    const uint32_t r = cp.rank_of ? __ldg(cp.rank_of + i) : (uint32_t)i;
    const uint32_t cnt = __ldg(cp.touched + r);
    // the geometric parameters and the statistics do not depend on the merge: issued first
    float mu[3], q[4], ls[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) mu[k] = __ldg(P + k * cap + i);
#pragma unroll
    for (int k = 0; k < 4; ++k) q[k] = __ldg(P + (3 + k) * cap + i);
#pragma unroll
    for (int k = 0; k < 3; ++k) ls[k] = __ldg(P + (7 + k) * cap + i);
    const float rop = __ldg(P + 10 * cap + i);
    float pa0 = 0.f, ca0 = 0.f;
    int32_t vi0 = 0;
    if (cp.update_stats && MODE != 2) {
        pa0 = cp.pos_acc[i];
        ca0 = cp.col_acc[i];
        vi0 = cp.visit[i];
    }
    float s[10];
#pragma unroll
    for (int k = 0; k < 10; ++k) s[k] = 0.f;
    if (cnt) {
        // tile-order merge (rasterizer.cpp:301-319): the splat's pair slots are contiguous
        const uint32_t base = __ldg(cp.pair_off + r);
        const float4* __restrict__ pa = cp.partial.a + base;
        const float4* __restrict__ pb = cp.partial.b + base;
        const float2* __restrict__ pc = cp.partial.c + base;
        for (uint32_t t = 0; t < cnt; ++t) {
            const float4 a = pa[t], b = pb[t];
            const float2 c = pc[t];
            s[0] += a.x; s[1] += a.y; s[2] += a.z; s[3] += a.w;
            s[4] += b.x; s[5] += b.y; s[6] += b.z; s[7] += b.w;
            s[8] += c.x;
            s[9] = fmaxf(s[9], c.y);
        }
    }
    if (cp.screen) {
#pragma unroll
        for (int k = 0; k < 10; ++k) cp.screen[(int64_t)k * cp.n + i] = s[k];
    }
    Geo3 g;
    float gg[11], b[16], dcol[3], dir[3] = {0.f, 0.f, 1.f};
    bool visited = false;
    float pn = 0.f, cn = 0.f;
    // untouched by this view: zero gradient (Adam still advances its moments)
    if (cnt != 0 && geometry(cp.cam, cp.bump, mu, q, ls, g)) {
        chain3d_grads(cp.cam, g, mu, rop, P, cap, i, s, gg, b, dcol, dir);
        // densify statistics: screen-space position norm, DC colour-gradient norm
        visited = s[9] > 0.f;
        if (visited) {
            pn = sqrtf(s[0] * s[0] + s[1] * s[1]);
            cn = SH_C0 * sqrtf(dcol[0] * dcol[0] + dcol[1] * dcol[1] + dcol[2] * dcol[2]);
        }
        if (cp.update_stats && visited && MODE != 2) {
            cp.pos_acc[i] = pa0 + pn;
            cp.col_acc[i] = ca0 + cn;
            cp.visit[i] = vi0 + 1;
        }
    } else {
#pragma unroll
        for (int k = 0; k < 11; ++k) gg[k] = 0.f;
#pragma unroll
        for (int k = 0; k < 16; ++k) b[k] = 0.f;
        dcol[0] = dcol[1] = dcol[2] = 0.f;
    }
    if (MODE != 1) {
        auto grad = [&](int k) -> float { return k < 11 ? gg[k] : fmul(b[(k - 11) / 3], dcol[(k - 11) % 3]); };
        if (MODE == 0) {
            float* __restrict__ G = cp.grads;
#pragma unroll
            for (int k = 0; k < 59; ++k) G[(int64_t)k * cp.n + i] = grad(k);
            return;
        }
        // batched views: sums in view order (tgsx_view_accumulate3d)
        float* __restrict__ ST = cp.step;
#pragma unroll
        for (int k0 = 0; k0 < 59; k0 += 8) {  // 8 loads in flight, then 8 stores
            float old[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < 59) old[k] = ST[(int64_t)(k0 + k) * cp.n + i];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k0 + k < 59) ST[(int64_t)(k0 + k) * cp.n + i] = old[k] + grad(k0 + k);
        }
        if (cp.update_stats && visited) {
            ST[59 * cp.n + i] += pn;
            ST[60 * cp.n + i] += cn;
            ST[61 * cp.n + i] += 1.0f;
        }
        return;
    }
    // fused step: 17 floats per Gaussian (11 gradients, the clamp-masked colour gradient, the
    // view direction) for the elementwise Adam kernel, which recomputes the SH basis
    float* __restrict__ GB = cp.gbuf;
#pragma unroll
    for (int k = 0; k < 11; ++k) GB[(int64_t)k * cp.n + i] = gg[k];
#pragma unroll
    for (int c = 0; c < 3; ++c) GB[(int64_t)(11 + c) * cp.n + i] = dcol[c];
#pragma unroll
    for (int c = 0; c < 3; ++c) GB[(int64_t)(14 + c) * cp.n + i] = dir[c];
}

// Adam over one group of components of every Gaussian (grid.y = group, kAdamGroups groups):
// groups 0..3 = rows 0-2, 3-5, 6-8, 9-10 (mean, quaternion, log-scales, opacity); group 4 + k = SH
// function k, all three channels (rows 11 + 3k ..). <= 3 components per thread: small register
// footprint, full occupancy for the streams.
constexpr int kAdamGroups = 20;

template <int G>
__device__ __forceinline__ void adam3d_group_apply(float* __restrict__ P, float* __restrict__ M1,
                                                   float* __restrict__ M2, int64_t cap, int64_t n,
                                                   int64_t i, const float* __restrict__ GB,
                                                   const Adam3dCfg& c) {
    if (G < 4) {
        constexpr int K0 = 3 * G, NK = G == 3 ? 2 : 3;
        float gg[NK];
#pragma unroll
        for (int k = 0; k < NK; ++k) gg[k] = GB[(int64_t)(K0 + k) * n + i];
        adam3d_chunk<K0, NK>(P, M1, M2, cap, i, [&](int k) { return gg[k - K0]; }, c);
    } else {
        float dcol[3], d[3], b[16];
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            dcol[k] = GB[(int64_t)(11 + k) * n + i];
            d[k] = GB[(int64_t)(14 + k) * n + i];
        }
        sh_basis(d[0], d[1], d[2], b);
        constexpr int K0 = 11 + 3 * (G - 4);
        adam3d_chunk<K0, 3>(P, M1, M2, cap, i,
                            [&](int k) { return fmul(b[(k - 11) / 3], dcol[(k - 11) % 3]); }, c);
    }
}

__global__ void __launch_bounds__(256) adam3d_apply_kernel(float* __restrict__ P, float* __restrict__ M1,
                                                           float* __restrict__ M2, int64_t cap, int64_t n,
                                                           const float* __restrict__ GB, Adam3dCfg c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    switch (blockIdx.y) {
        case 0: adam3d_group_apply<0>(P, M1, M2, cap, n, i, GB, c); break;
        case 1: adam3d_group_apply<1>(P, M1, M2, cap, n, i, GB, c); break;
        case 2: adam3d_group_apply<2>(P, M1, M2, cap, n, i, GB, c); break;
        case 3: adam3d_group_apply<3>(P, M1, M2, cap, n, i, GB, c); break;
        case 4: adam3d_group_apply<4>(P, M1, M2, cap, n, i, GB, c); break;
        case 5: adam3d_group_apply<5>(P, M1, M2, cap, n, i, GB, c); break;
        case 6: adam3d_group_apply<6>(P, M1, M2, cap, n, i, GB, c); break;
        case 7: adam3d_group_apply<7>(P, M1, M2, cap, n, i, GB, c); break;
        case 8: adam3d_group_apply<8>(P, M1, M2, cap, n, i, GB, c); break;
        case 9: adam3d_group_apply<9>(P, M1, M2, cap, n, i, GB, c); break;
        case 10: adam3d_group_apply<10>(P, M1, M2, cap, n, i, GB, c); break;
        case 11: adam3d_group_apply<11>(P, M1, M2, cap, n, i, GB, c); break;
        case 12: adam3d_group_apply<12>(P, M1, M2, cap, n, i, GB, c); break;
        case 13: adam3d_group_apply<13>(P, M1, M2, cap, n, i, GB, c); break;
        case 14: adam3d_group_apply<14>(P, M1, M2, cap, n, i, GB, c); break;
        case 15: adam3d_group_apply<15>(P, M1, M2, cap, n, i, GB, c); break;
        case 16: adam3d_group_apply<16>(P, M1, M2, cap, n, i, GB, c); break;
        case 17: adam3d_group_apply<17>(P, M1, M2, cap, n, i, GB, c); break;
        case 18: adam3d_group_apply<18>(P, M1, M2, cap, n, i, GB, c); break;
        default: adam3d_group_apply<19>(P, M1, M2, cap, n, i, GB, c); break;
    }
}

// Adam with explicit gradients [59][n] (tgsx_adam3d_step): grid.y = group of components as above
__global__ void __launch_bounds__(256) adam3d_kernel(float* __restrict__ params, float* __restrict__ m1,
                                                     float* __restrict__ m2, int64_t cap, int64_t n,
                                                     const float* __restrict__ grads, Adam3dCfg c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto grad = [&](int k) -> float { return grads[(int64_t)k * n + i]; };
    switch (blockIdx.y) {
        case 0: adam3d_chunk<0, 6>(params, m1, m2, cap, i, grad, c); break;
        case 1: adam3d_chunk<6, 5>(params, m1, m2, cap, i, grad, c); break;
        case 2: adam3d_chunk<11, 6>(params, m1, m2, cap, i, grad, c); break;
        case 3: adam3d_chunk<17, 6>(params, m1, m2, cap, i, grad, c); break;
        case 4: adam3d_chunk<23, 6>(params, m1, m2, cap, i, grad, c); break;
        case 5: adam3d_chunk<29, 6>(params, m1, m2, cap, i, grad, c); break;
        case 6: adam3d_chunk<35, 6>(params, m1, m2, cap, i, grad, c); break;
        case 7: adam3d_chunk<41, 6>(params, m1, m2, cap, i, grad, c); break;
        case 8: adam3d_chunk<47, 6>(params, m1, m2, cap, i, grad, c); break;
        default: adam3d_chunk<53, 6>(params, m1, m2, cap, i, grad, c); break;
    }
}

// Batched step (tgsx_apply_step3d): gradient = step sum / views (SPEC.md:269-277 accumulate),
// statistics from the summed increments, Adam; the step buffer is zeroed for the next batch.
__global__ void __launch_bounds__(256) adam3d_step_kernel(float* __restrict__ params, float* __restrict__ m1,
                                                          float* __restrict__ m2, int64_t cap, int64_t n,
                                                          float* __restrict__ step, float batch,
                                                          float* __restrict__ pos_acc, float* __restrict__ col_acc,
                                                          int32_t* __restrict__ visit, Adam3dCfg c) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    auto grad = [&](int k) -> float {
        float* p = step + (int64_t)k * n + i;  // packed [62][n]
        const float v = *p;
        *p = 0.f;
        return fdiv_pos(v, batch);
    };
    switch (blockIdx.y) {
        case 0: {
            adam3d_chunk<0, 6>(params, m1, m2, cap, i, grad, c);
            const float v = step[61 * n + i];
            if (v > 0.f) {
                pos_acc[i] += step[59 * n + i];
                col_acc[i] += step[60 * n + i];
                visit[i] += (int32_t)v;
            }
            step[59 * n + i] = 0.f;
            step[60 * n + i] = 0.f;
            step[61 * n + i] = 0.f;
            break;
        }
        case 1: adam3d_chunk<6, 5>(params, m1, m2, cap, i, grad, c); break;
        case 2: adam3d_chunk<11, 6>(params, m1, m2, cap, i, grad, c); break;
        case 3: adam3d_chunk<17, 6>(params, m1, m2, cap, i, grad, c); break;
        case 4: adam3d_chunk<23, 6>(params, m1, m2, cap, i, grad, c); break;
        case 5: adam3d_chunk<29, 6>(params, m1, m2, cap, i, grad, c); break;
        case 6: adam3d_chunk<35, 6>(params, m1, m2, cap, i, grad, c); break;
        case 7: adam3d_chunk<41, 6>(params, m1, m2, cap, i, grad, c); break;
        case 8: adam3d_chunk<47, 6>(params, m1, m2, cap, i, grad, c); break;
        default: adam3d_chunk<53, 6>(params, m1, m2, cap, i, grad, c); break;
    }
}

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

}  // namespace

cudaError_t launch_adam3d_step(tgsx_ctx* ctx, tgsx_model3d* m, int batch_views, const Adam3dCfg& cfg) {
    if (m->n == 0) return cudaSuccess;
    adam3d_step_kernel<<<dim3(grid_for(m->n, 256), 10), 256, 0, ctx->stream>>>(
        m->params.as<float>(), m->m1.as<float>(), m->m2.as<float>(), m->cap, m->n, m->step.as<float>(),
        (float)(batch_views > 0 ? batch_views : 1), m->pos_acc.as<float>(), m->col_acc.as<float>(),
        m->visit.as<int32_t>(), cfg);
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_adam3d(tgsx_ctx* ctx, tgsx_model3d* m, const float* grads, const Adam3dCfg& cfg) {
    if (m->n == 0) return cudaSuccess;
    adam3d_kernel<<<dim3(grid_for(m->n, 256), 10), 256, 0, ctx->stream>>>(m->params.as<float>(), m->m1.as<float>(),
                                                                m->m2.as<float>(), m->cap, m->n, grads, cfg);
    ctx->launches++;
    return cudaGetLastError();
}

static cudaError_t prepare3d_buffers(tgsx_ctx* ctx, tgsx_model3d* m, int W, int H) {
    Workspace& ws = ctx->ws;
    const int64_t c = std::max<int64_t>(m->n, 1);
    cudaError_t e;
    if ((e = ws.prep.ensure(c * sizeof(Prepared)))) return e;
    if ((e = m->prep_row.ensure(c * sizeof(Prepared)))) return e;
    if ((e = ws.touched.ensure((c + 1) * 4))) return e;
    if ((e = ws.pair_off.ensure((c + 1) * 4))) return e;
    for (int k = 0; k < 2; ++k) {
        if ((e = ws.keys[k].ensure(c * 4))) return e;
        if ((e = ws.vals[k].ensure(c * 4))) return e;
    }
    ws.tiles_x = (W + kTile - 1) / kTile;
    ws.tiles_y = (H + kTile - 1) / kTile;
    const size_t tiles = (size_t)std::max(ws.tiles_x * ws.tiles_y, 1);
    if ((e = ws.tile_fill.ensure(tiles * 4 * kFillStride))) return e;
    if ((e = ws.tile_slab.ensure(tiles * 4 * kSegCap))) return e;
    return cudaMemsetAsync(ws.tile_fill.p, 0, tiles * 4 * kFillStride, ctx->stream);
}

cudaError_t launch_preprocess3d(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p,
                                int W, int H) {
    Workspace& ws = ctx->ws;
    const int64_t n = m->n;
    cudaError_t e;
    if ((e = prepare3d_buffers(ctx, m, W, H))) return e;
    if (n == 0) return cudaSuccess;
    const float bump = 0.3f + 0.5f * (float)(lowpass_p - 1);
    preprocess3d_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        m->params.as<float>(), m->cap, n, cam, bump, m->prep_row.as<Prepared>(),
        ws.keys[0].as<uint32_t>(), ws.vals[0].as<uint32_t>(), ws.counters.as<unsigned long long>());
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_preprocess3d_bin(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int W, int H,
                                    uint32_t* d_total) {
    Workspace& ws = ctx->ws;
    cudaError_t e;
    if ((e = prepare3d_buffers(ctx, m, W, H))) return e;
    const int64_t n = m->n;
    if (n == 0) return cudaMemsetAsync(d_total, 0, sizeof(uint32_t), ctx->stream);
    const int64_t blocks = grid_for(n, 256);
    const size_t need = 64 + (size_t)blocks * sizeof(unsigned long long);
    if ((e = ws.scan_tmp.ensure(need))) return e;
    if ((e = cudaMemsetAsync(ws.scan_tmp.p, 0, need, ctx->stream))) return e;
    const float bump = 0.3f + 0.5f * (float)(lowpass_p - 1);
    preprocess3d_bin_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(
        m->params.as<float>(), m->cap, n, cam, bump, W, H, ws.tiles_x, ws.prep.as<Prepared>(),
        ws.keys[0].as<uint32_t>(), ws.touched.as<uint32_t>(), ws.pair_off.as<uint32_t>(),
        ws.tile_fill.as<uint32_t>(), ws.tile_slab.as<uint32_t>(), ws.counters.as<unsigned long long>(),
        reinterpret_cast<unsigned long long*>(ws.scan_tmp.as<char>() + 64), ws.scan_tmp.as<uint32_t>(), d_total);
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_seg_sort3d(tgsx_ctx* ctx, int tiles, int64_t max_list) {
    if (tiles == 0) return cudaSuccess;
    const uint2* rg = ctx->ws.ranges.as<uint2>();
    uint32_t* items = ctx->ws.tile_slab.as<uint32_t>();
    const uint32_t* keys = ctx->ws.keys[0].as<uint32_t>();
    const unsigned grid = grid_for(tiles, 8);
    if (max_list <= 256)
        seg_sort3d_kernel<8><<<grid, 256, 0, ctx->stream>>>(rg, tiles, items, keys);
    else if (max_list <= 512)
        seg_sort3d_kernel<16><<<grid, 256, 0, ctx->stream>>>(rg, tiles, items, keys);
    else
        seg_sort3d_kernel<32><<<grid, 256, 0, ctx->stream>>>(rg, tiles, items, keys);
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_bin3d(tgsx_ctx* ctx, tgsx_model3d* m, const uint32_t* skeys, const uint32_t* svals,
                         int W, int H, uint32_t* d_total) {
    Workspace& ws = ctx->ws;
    const int64_t n = m->n;
    if (n == 0) return cudaMemsetAsync(d_total, 0, sizeof(uint32_t), ctx->stream);
    const int64_t blocks = grid_for(n, 256);
    const size_t need = 64 + (size_t)blocks * sizeof(unsigned long long);
    cudaError_t e;
    if ((e = ws.scan_tmp.ensure(need))) return e;
    if ((e = cudaMemsetAsync(ws.scan_tmp.p, 0, need, ctx->stream))) return e;
    bin3d_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(
        skeys, svals, n, m->prep_row.as<Prepared>(), W, H, ws.tiles_x, ws.prep.as<Prepared>(),
        ws.touched.as<uint32_t>(), ws.pair_off.as<uint32_t>(), ws.tile_fill.as<uint32_t>(),
        ws.tile_slab.as<uint32_t>(), m->perm.as<uint32_t>(), m->rank_of.as<uint32_t>(),
        reinterpret_cast<unsigned long long*>(ws.scan_tmp.as<char>() + 64), ws.scan_tmp.as<uint32_t>(), d_total);
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_chain3d(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int mode,
                           bool update_stats, float* grads, float* screen, const Adam3dCfg* cfg) {
    const bool adam = mode == 1;
    if (m->n == 0) return cudaSuccess;
    Chain3Params cp{};
    cp.params = m->params.as<float>();
    cp.cap = m->cap;
    cp.n = m->n;
    cp.cam = cam;
    cp.bump = 0.3f + 0.5f * (float)(lowpass_p - 1);
    cp.rank_of = m->rank_ordered ? m->rank_of.as<uint32_t>() : nullptr;
    cp.pair_off = ctx->ws.pair_off.as<uint32_t>();
    cp.touched = ctx->ws.touched.as<uint32_t>();
    cp.partial = Partials::at(ctx->ws.partial.p, ctx->ws.pair_cap);
    cp.mode = mode;
    cp.step = m->step.as<float>();
    cp.grads = grads;
    cp.screen = screen;
    cp.pos_acc = m->pos_acc.as<float>();
    cp.col_acc = m->col_acc.as<float>();
    cp.visit = m->visit.as<int32_t>();
    cp.update_stats = update_stats ? 1 : 0;
    cudaError_t e;
    if (adam) {
        if ((e = m->gbuf.ensure((size_t)std::max<int64_t>(m->n, 1) * 17 * 4))) return e;
        cp.gbuf = m->gbuf.as<float>();
    }
    if (mode == 1)
        chain3d_kernel<1><<<grid_for(m->n, 256), 256, 0, ctx->stream>>>(cp);
    else if (mode == 2)
        chain3d_kernel<2><<<grid_for(m->n, 256), 256, 0, ctx->stream>>>(cp);
    else
        chain3d_kernel<0><<<grid_for(m->n, 256), 256, 0, ctx->stream>>>(cp);
    ctx->launches++;
    if (adam) {
        adam3d_apply_kernel<<<dim3(grid_for(m->n, 256), kAdamGroups), 256, 0, ctx->stream>>>(
            m->params.as<float>(), m->m1.as<float>(), m->m2.as<float>(), m->cap, m->n, cp.gbuf, *cfg);
        ctx->launches++;
    }
    return cudaGetLastError();
}

}  // namespace tgsx
