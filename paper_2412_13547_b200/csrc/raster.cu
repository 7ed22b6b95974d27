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
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>

namespace tgsx {

namespace {

// per-tile counters one per 128-B line: neighbouring tiles' atomics do not serialise on one L2 line
constexpr int kFillStride = 32;

// ------------------------------------------------------------------ preprocess
// Slab binning: claim a slot in every tile of the record's rectangle (d = packed rect, tiles):
// kSegCap entries per tile, arbitrary order inside a tile (the per-tile sort restores blend
// order). Four claims in flight per step: the returning atomics' latency dominates.
__device__ __forceinline__ void claim_slots(const uint4& d, int tiles_x, uint32_t v, uint32_t* __restrict__ fill,
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

// One Gaussian (row i, blend rank `rank`): the prepared record, the number of tiles it touches
// and (slab binning) its slot claims. Returns the tile count; 0 on an error (raised in err).
__device__ __forceinline__ uint32_t prepare_one(const float* __restrict__ params, int64_t cap, int64_t i,
                                                uint32_t rank, uint32_t orig, int lowpass_p, int W, int H,
                                                int tiles_x, Prepared& o, uint32_t* __restrict__ fill,
                                                uint32_t* __restrict__ slab, unsigned long long* err) {
    const float px = params[i], py = params[cap + i], rot = params[2 * cap + i];
    const float lx = params[3 * cap + i], ly = params[4 * cap + i], rop = params[5 * cap + i];
    const float cr = params[6 * cap + i], cg = params[7 * cap + i], cb = params[8 * cap + i];
    o.d = make_uint4(0u, 0u, 0u, 0u);
    // covariance_from_params (gaussian.hpp:63-78)
    if (!isfinite(rot) || !isfinite(lx) || !isfinite(ly)) {
        raise_error(err, rank, 1);
        return 0;
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
        return 0;
    }
    o.a = make_float4(px, py, fdiv_pos(s11, det), fdiv_pos(-s01, det));
    const float rx = fmul(kCullSigmas, __fsqrt_rn(s00));
    const float ry = fmul(kCullSigmas, __fsqrt_rn(s11));
    o.b = make_float4(fdiv_pos(s00, det), activate_cr(rop), rx, ry);
    o.c = make_float4(activate_cr(cr), activate_cr(cg), activate_cr(cb), __uint_as_float(orig));
    int tx0, tx1, ty0, ty1;
    uint32_t tiles = 0;
    if (tile_rect(px, py, rx, ry, W, H, tx0, tx1, ty0, ty1)) {
        tiles = (uint32_t)((tx1 - tx0 + 1) * (ty1 - ty0 + 1));
        o.d = make_uint4((uint32_t)tx0 | ((uint32_t)tx1 << 16), (uint32_t)ty0 | ((uint32_t)ty1 << 16),
                         0u, tiles);
        if (fill) claim_slots(o.d, tiles_x, rank, fill, slab);
    }
    return tiles;
}

__global__ void __launch_bounds__(256) preprocess_kernel(
    const float* __restrict__ params, int64_t cap, int64_t n,
    const uint32_t* __restrict__ rank_of, const uint32_t* __restrict__ perm, int blend_phys,
    int lowpass_p, int W, int H, int tiles_x,
    Prepared* __restrict__ prep, uint32_t* __restrict__ touched, uint32_t* __restrict__ fill,
    uint32_t* __restrict__ slab, unsigned long long* err) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    // row i is rank i when the model is stored in blend order (logical index perm[i])
    const uint32_t rank = blend_phys ? (uint32_t)i : rank_of[i];
    const uint32_t orig = blend_phys ? perm[i] : (uint32_t)i;
    Prepared o;
    const uint32_t tiles = prepare_one(params, cap, i, rank, orig, lowpass_p, W, H, tiles_x, o, fill, slab, err);
    prep[rank] = o;
    touched[rank] = tiles;
}

// Rows in blend order (rank == row), with the pair-offset scan fused in: blocks (in dispatch
// order, lookback_block) reduce their tile counts and find their prefix by decoupled look-back
// (block_scan_lookback), so each record leaves with its first pair slot (d.z) and pair_off /
// touched / the total K are written here: the separate scan and pair-base passes over the
// Gaussians disappear from the step.
__global__ void __launch_bounds__(256) preprocess_scan_kernel(
    const float* __restrict__ params, int64_t cap, int64_t n, const uint32_t* __restrict__ perm,
    int lowpass_p, int W, int H, int tiles_x, Prepared* __restrict__ prep, uint32_t* __restrict__ touched,
    uint32_t* __restrict__ pair_off, uint32_t* __restrict__ fill, uint32_t* __restrict__ slab,
    unsigned long long* err, unsigned long long* status, uint32_t* ticket, uint32_t* d_total,
    uint2* __restrict__ rect) {
    const uint32_t bid = lookback_block(ticket);
    const int64_t i = (int64_t)bid * 256 + threadIdx.x;
    Prepared o;
    uint32_t tiles = 0;
    // the slot claims come after the scan: the block barrier never waits on their atomics
    if (i < n) tiles = prepare_one(params, cap, i, (uint32_t)i, perm[i], lowpass_p, W, H, tiles_x, o, nullptr, slab, err);
    const uint32_t excl = block_scan_lookback(tiles, bid, n, status, d_total);
    if (i < n) {
        o.d.z = excl;
        prep[i] = o;
        touched[i] = tiles;
        pair_off[i] = excl;
        // compact rectangle for the claim kernel (an empty rectangle has tiles == 0: tx1 < tx0)
        if (rect) rect[i] = tiles ? make_uint2(o.d.x, o.d.y) : make_uint2(1u, 1u);
        if (tiles && fill) claim_slots(o.d, tiles_x, (uint32_t)i, fill, slab);
    }
}

// ------------------------------------------------------------------ slot claims
// Slab slot claims of every (tile, splat) pair, taken in SPATIAL order: thread i handles blend
// rank spatial[i] (ranks ordered by the top-left tile of their rectangle), so a warp's pairs fall
// on a handful of tiles. The warp flattens its 32 splats' pairs (exclusive scan of the tile
// counts), takes them 32 at a time (lane j: pair base + j, its owner found by a 5-step binary
// search over the scan), groups equal tiles with match.any and claims one run of slots per
// distinct tile with a single atomic. A slot's position inside its tile is arbitrary (the
// per-tile sort restores blend order), so the claim order changes nothing but the atomic count:
// in blend (depth) order neighbouring threads hit unrelated tiles and every pair was one
// contended L2 atomic.
__global__ void __launch_bounds__(256) claim_kernel(const uint32_t* __restrict__ spatial,
                                                    const uint2* __restrict__ rect, int64_t n, int tiles_x,
                                                    uint32_t* __restrict__ fill, uint32_t* __restrict__ slab) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int lane = threadIdx.x & 31;
    uint32_t rank = 0;
    uint2 d = make_uint2(1u, 1u);  // empty
    if (i < n) {
        rank = __ldcs(spatial + i);
        d = __ldg(&rect[rank]);
    }
    const int rw = (int)(d.x >> 16) - (int)(d.x & 0xffffu) + 1, rh = (int)(d.y >> 16) - (int)(d.y & 0xffffu) + 1;
    const uint32_t cnt = rw > 0 && rh > 0 ? (uint32_t)(rw * rh) : 0u;
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    const uint32_t excl = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t tx0 = d.x & 0xffffu, ty0 = d.y & 0xffffu, w = (d.x >> 16) - tx0 + 1u;
    const uint32_t lt = lanemask_lt();
    for (uint32_t base = 0; base < total; base += 32) {
        const uint32_t j = base + (uint32_t)lane;
        int o = 0;  // owner: the last lane whose exclusive offset is <= j (it has j inside its run)
#pragma unroll
        for (int s = 16; s > 0; s >>= 1) {
            const uint32_t e = __shfl_sync(0xffffffffu, excl, o + s);
            if (e <= j) o += s;
        }
        const uint32_t q = j - __shfl_sync(0xffffffffu, excl, o);
        const uint32_t orank = __shfl_sync(0xffffffffu, rank, o);
        const uint32_t otx0 = __shfl_sync(0xffffffffu, tx0, o), oty0 = __shfl_sync(0xffffffffu, ty0, o);
        const uint32_t ow = __shfl_sync(0xffffffffu, w, o);
        const bool valid = j < total;
        const uint32_t qy = valid ? q / ow : 0u;
        const uint32_t tile = valid ? (oty0 + qy) * (uint32_t)tiles_x + otx0 + (q - qy * ow) : 0xffffffffu;
        const uint32_t peers = __match_any_sync(0xffffffffu, tile);
        const int leader = __ffs(peers) - 1;
        uint32_t pos = 0;
        if (valid && lane == leader) pos = atomicAdd(&fill[(size_t)tile * kFillStride], (uint32_t)__popc(peers));
        pos = __shfl_sync(0xffffffffu, pos, leader) + (uint32_t)__popc(peers & lt);
        if (valid && pos < (uint32_t)kSegCap) slab[(size_t)tile * kSegCap + pos] = orank;
    }
}

// spatial order key of blend rank r: the top-left tile of its rectangle (unbinned: last)
__global__ void spatial_keys_kernel(const uint2* __restrict__ rect, int64_t n, int tiles_x, uint32_t* __restrict__ keys,
                                    uint32_t* __restrict__ vals) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const uint2 d = __ldg(&rect[r]);
    const bool empty = (d.x >> 16) < (d.x & 0xffffu);
    keys[r] = empty ? 0x7fffffffu : (d.y & 0xffffu) * (uint32_t)tiles_x + (d.x & 0xffffu);
    vals[r] = (uint32_t)r;
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

// ------------------------------------------------------------------ slab binning
// Preprocess claims every (tile, splat) slot in the tile's fixed-size slab (kSegCap entries,
// claim order arbitrary); the per-tile sort restores blend (rank) order, so the lists are
// deterministic and equal TileGrid's (rasterizer.cpp:92-100). A tile whose list exceeds the
// slab makes the view take the onesweep path.
__global__ void slab_finalize_kernel(const uint32_t* __restrict__ fill, int tiles,
                                     uint2* __restrict__ ranges, unsigned long long* __restrict__ max_cnt) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t c = 0;
    if (t < tiles) {
        c = fill[(size_t)t * kFillStride];
        const uint32_t o = (uint32_t)t * (uint32_t)kSegCap;
        ranges[t] = make_uint2(o, o + min(c, (uint32_t)kSegCap));
    }
    c = __reduce_max_sync(0xffffffffu, c);
    if ((threadIdx.x & 31) == 0 && c) atomicMax(max_cnt, (unsigned long long)c);
}

// Bitonic sort of 32*E keys held by one warp, lane L owning positions L*E .. L*E+E-1:
// partners closer than E are in-register compare-exchanges, farther ones one shuffle.
template <int E>
__device__ __forceinline__ void warp_bitonic(uint32_t (&x)[E], int lane) {
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {
                const int lm = j / E;
                const bool lower = (lane & lm) == 0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const uint32_t y = __shfl_xor_sync(0xffffffffu, x[e], lm);
                    const bool asc = ((lane * E + e) & k) == 0;
                    x[e] = (asc == lower) ? min(x[e], y) : max(x[e], y);
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if ((e & j) == 0) {
                        const bool asc = ((lane * E + e) & k) == 0;
                        const uint32_t a = x[e], b = x[e | j];
                        x[e] = asc ? min(a, b) : max(a, b);
                        x[e | j] = asc ? max(a, b) : min(a, b);
                    }
                }
            }
        }
    }
}

template <int E>
__device__ __forceinline__ void warp_sort_list(uint32_t* __restrict__ list, int n, int lane) {
    uint32_t x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = lane * E + e < n ? list[lane * E + e] : 0xffffffffu;
    warp_bitonic<E>(x, lane);
#pragma unroll
    for (int e = 0; e < E; ++e)
        if (lane * E + e < n) list[lane * E + e] = x[e];
}

// One warp per tile: the tile's ranks (claimed in arbitrary order by the scatter) sorted back
// into blend order in registers (lists <= kSegCap = 1024).
// MAXE: largest per-lane width instantiated (lists <= 32 * MAXE); chosen on the host from the
// longest list, so the common case does not pay the registers of the 1024-entry network
template <int MAXE>
__global__ void __launch_bounds__(256) seg_sort_kernel(const uint2* __restrict__ ranges, int tiles,
                                                       uint32_t* __restrict__ items) {
    const int lane = threadIdx.x & 31;
    const int tile = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (tile >= tiles) return;
    const uint2 rg = ranges[tile];
    const int n = (int)(rg.y - rg.x);
    uint32_t* list = items + rg.x;
    if (n <= 1) return;
    // three network sizes: warps of one SM running many different fully unrolled networks
    // thrash the instruction cache
    if (n <= 64) warp_sort_list<2>(list, n, lane);
    else if (MAXE <= 16 || n <= 512) warp_sort_list<MAXE < 16 ? MAXE : 16>(list, n, lane);
    else warp_sort_list<MAXE>(list, n, lane);
}

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

}  // namespace

cudaError_t launch_slab_finalize(tgsx_ctx* ctx, int tiles) {
    Workspace& ws = ctx->ws;
    cudaError_t e;
    if ((e = ws.ranges.ensure((size_t)std::max(tiles, 1) * sizeof(uint2)))) return e;
    if (tiles == 0) return cudaSuccess;
    slab_finalize_kernel<<<grid_for(tiles, 256), 256, 0, ctx->stream>>>(
        ws.tile_fill.as<uint32_t>(), tiles, ws.ranges.as<uint2>(), ws.counters.as<unsigned long long>() + 5);
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_seg_sort(tgsx_ctx* ctx, uint32_t* items, int tiles, int64_t max_list) {
    if (tiles == 0) return cudaSuccess;
    const uint2* rg = ctx->ws.ranges.as<uint2>();
    const unsigned grid = grid_for(tiles, 8);
    if (max_list <= 256)
        seg_sort_kernel<8><<<grid, 256, 0, ctx->stream>>>(rg, tiles, items);
    else if (max_list <= 512)
        seg_sort_kernel<16><<<grid, 256, 0, ctx->stream>>>(rg, tiles, items);
    else
        seg_sort_kernel<32><<<grid, 256, 0, ctx->stream>>>(rg, tiles, items);
    ctx->launches++;
    return cudaGetLastError();
}


int key_bits_for(int tiles) {
    int b = 0;
    while ((1ll << b) < (long long)tiles) ++b;
    return b;
}

// Spatial claim order of the model's blend ranks (claim_kernel): ranks sorted by the top-left
// tile of their rectangles in the records of the current preprocess. Rebuilt when the blend
// ranks change (depth sort) and every kSpatialRefresh binnings (splats move while fitting; any
// permutation is correct, the order only sets how many atomics the claims need).
constexpr int kSpatialRefresh = 64;

cudaError_t launch_claims(tgsx_ctx* ctx, tgsx_model* m) {
    Workspace& ws = ctx->ws;
    const int64_t n = m->n;
    cudaError_t e;
    if (n == 0) return cudaSuccess;
    const int tiles = ws.tiles_x * ws.tiles_y;
    if (!m->spatial_valid || (m->spatial_age >= kSpatialRefresh && !ctx->graph_capturing)) {
        if ((e = m->spatial.ensure((size_t)m->cap * 4))) return e;
        for (int b = 0; b < 2; ++b) {
            if ((e = ws.keys[b].ensure(std::max<int64_t>(m->cap, n) * 4))) return e;
            if ((e = ws.vals[b].ensure(std::max<int64_t>(m->cap, n) * 4))) return e;
        }
        ctx->bin_valid = false;  // the sort reuses the binning buffers
        uint32_t *k = ws.keys[0].as<uint32_t>(), *v = ws.vals[0].as<uint32_t>();
        spatial_keys_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(ws.rect.as<uint2>(), n, ws.tiles_x, k, v);
        ctx->launches++;
        if ((e = sort_pairs(ctx, k, v, ws.keys[1].as<uint32_t>(), ws.vals[1].as<uint32_t>(), n,
                            key_bits_for(tiles + 1), nullptr)))
            return e;
        if ((e = cudaMemcpyAsync(m->spatial.p, v, n * 4, cudaMemcpyDeviceToDevice, ctx->stream))) return e;
        m->spatial_valid = true;
        m->spatial_age = 0;
    }
    ++m->spatial_age;
    claim_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(m->spatial.as<uint32_t>(), ws.rect.as<uint2>(), n,
                                                            ws.tiles_x, ws.tile_fill.as<uint32_t>(),
                                                            ws.tile_slab.as<uint32_t>());
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_preprocess(tgsx_ctx* ctx, tgsx_model* m, int lowpass_p, int W, int H, uint32_t* d_total) {
    Workspace& ws = ctx->ws;
    const int64_t n = m->n;
    // per-splat buffers sized by the model's capacity: a fit that grows its model (densify up to
    // a reserved budget) never reallocates them mid-run
    const int64_t nc = std::max<int64_t>(m->cap, n);
    cudaError_t e;
    if ((e = ws.prep.ensure(std::max<int64_t>(nc, 1) * sizeof(Prepared)))) return e;
    if ((e = ws.touched.ensure((nc + 1) * 4))) return e;
    if ((e = ws.pair_off.ensure((nc + 1) * 4))) return e;
    if ((e = ws.rect.ensure((nc + 1) * 8))) return e;
    ws.tiles_x = (W + kTile - 1) / kTile;
    ws.tiles_y = (H + kTile - 1) / kTile;
    const size_t tiles = (size_t)std::max(ws.tiles_x * ws.tiles_y, 1);
    if ((e = ws.tile_fill.ensure(tiles * 4 * kFillStride))) return e;
    if ((e = ws.tile_slab.ensure(tiles * 4 * kSegCap))) return e;
    if ((e = cudaMemsetAsync(ws.tile_fill.p, 0, tiles * 4 * kFillStride, ctx->stream))) return e;
    if (n == 0) {
        if (d_total) return cudaMemsetAsync(d_total, 0, sizeof(uint32_t), ctx->stream);
        return cudaSuccess;
    }
    if (d_total) {
        // fused pair-offset scan: rows must be in blend order
        if (!m->blend_phys) return cudaErrorInvalidValue;
        const int64_t blocks = grid_for(n, 256);
        const size_t need = 64 + (size_t)blocks * sizeof(unsigned long long);
        if ((e = ws.scan_tmp.ensure(need))) return e;
        if ((e = cudaMemsetAsync(ws.scan_tmp.p, 0, need, ctx->stream))) return e;
        preprocess_scan_kernel<<<(unsigned)blocks, 256, 0, ctx->stream>>>(
            m->params.as<float>(), m->cap, n, m->perm.as<uint32_t>(), lowpass_p, W, H, ws.tiles_x,
            ws.prep.as<Prepared>(), ws.touched.as<uint32_t>(), ws.pair_off.as<uint32_t>(), nullptr,
            ws.tile_slab.as<uint32_t>(), ws.counters.as<unsigned long long>(),
            reinterpret_cast<unsigned long long*>(ws.scan_tmp.as<char>() + 64), ws.scan_tmp.as<uint32_t>(),
            d_total, ws.rect.as<uint2>());
        ctx->launches++;
        if ((e = cudaGetLastError())) return e;
        return launch_claims(ctx, m);
    }
    preprocess_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        m->params.as<float>(), m->cap, n, m->rank_of.as<uint32_t>(), m->perm.as<uint32_t>(),
        m->blend_phys ? 1 : 0, lowpass_p, W, H, ws.tiles_x,
        ws.prep.as<Prepared>(), ws.touched.as<uint32_t>(), ws.tile_fill.as<uint32_t>(),
        ws.tile_slab.as<uint32_t>(), ws.counters.as<unsigned long long>());
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_duplicate(tgsx_ctx* ctx, int64_t n, int key_bits) {
    Workspace& ws = ctx->ws;
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

}  // namespace tgsx
