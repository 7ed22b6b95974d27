// Device-wide primitives for the binning stage, hand-written for sm_100a:
//  * exclusive_scan_kernel — single-pass u32 exclusive scan with decoupled look-back
//    (replaces the serial prefix sum of build_tile_grid, rasterizer.cpp:92).
//  * onesweep_pass — one 8-bit digit pass of a stable LSD radix sort of (u32 key, u32 value)
//    pairs (Adinets & Merrill "Onesweep"): warp-private digit ranking with match_any,
//    per-digit decoupled look-back across blocks, direct scatter. Stability + keys emitted in
//    blend order reproduce the reference's per-tile lists exactly (rasterizer.cpp:93-100).
//  * histogram_kernel — all digit histograms of a key array in one read.
//  * depth ordering — GaussianModel::sorted_order (model.hpp:106-119): stable sort by
//    orderable(depth_key) over index order (index order == id order when ids are monotone;
//    otherwise an id pre-sort establishes the tie order).
//
// All three are HBM/L2-bound integer kernels: coalesced 128-bit loads where layout allows,
// grids sized to the data (thousands of blocks), no tensor-core reshaping.
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>
#include <utility>

namespace tgsx {

namespace {

constexpr int kScanBT = 256;
constexpr int kScanIT = 8;
constexpr int kScanTile = kScanBT * kScanIT;

constexpr int kSortBT = 256;
constexpr int kSortIT = 8;  // 2048 keys per block: ~60 registers, 4 blocks per SM
constexpr int kSortTile = kSortBT * kSortIT;
constexpr int kRadix = 256;

constexpr unsigned long long kScanAgg = 1ull << 62;
constexpr unsigned long long kScanIncl = 2ull << 62;
constexpr unsigned long long kScanValMask = (1ull << 62) - 1;

constexpr uint32_t kSortAgg = 1u << 30;
constexpr uint32_t kSortIncl = 2u << 30;
constexpr uint32_t kSortValMask = (1u << 30) - 1;

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *reinterpret_cast<const volatile unsigned long long*>(p);
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
    *reinterpret_cast<volatile unsigned long long*>(p) = v;
}
__device__ __forceinline__ uint32_t ld_volatile_u32(const uint32_t* p) {
    return *reinterpret_cast<const volatile uint32_t*>(p);
}
__device__ __forceinline__ void st_volatile_u32(uint32_t* p, uint32_t v) {
    *reinterpret_cast<volatile uint32_t*>(p) = v;
}

// ------------------------------------------------------------------ exclusive scan
// status[b]: flag (2 bits) | value (62 bits); blocks look back in dispatch order (lookback_block) so a
// block only ever waits on blocks that are already resident.
__global__ void __launch_bounds__(kScanBT) exclusive_scan_kernel(
    const uint32_t* __restrict__ in, uint32_t* __restrict__ out, int64_t n,
    unsigned long long* status, uint32_t* ticket, uint32_t* d_total) {
    __shared__ unsigned long long s_warp[kScanBT / 32];
    __shared__ unsigned long long s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t bid = lookback_block(ticket);
    const int64_t base = (int64_t)bid * kScanTile + (int64_t)tid * kScanIT;

    uint32_t v[kScanIT];
    if (base + kScanIT <= n && ((reinterpret_cast<uintptr_t>(in + base) & 15) == 0)) {
        const uint4 a = *reinterpret_cast<const uint4*>(in + base);
        const uint4 b = *reinterpret_cast<const uint4*>(in + base + 4);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
        v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else {
#pragma unroll
        for (int i = 0; i < kScanIT; ++i) v[i] = (base + i < n) ? in[base + i] : 0u;
    }
    unsigned long long tsum = 0;
#pragma unroll
    for (int i = 0; i < kScanIT; ++i) tsum += v[i];
    // warp inclusive scan of thread sums
    unsigned long long incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        unsigned long long w = lane < kScanBT / 32 ? s_warp[lane] : 0ull;
        unsigned long long wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned long long t = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += t;
        }
        if (lane < kScanBT / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
        const unsigned long long block_total = __shfl_sync(0xffffffffu, wi, 31);
        // decoupled look-back, one warp, 32 predecessors per window
        unsigned long long prefix = 0;
        if (bid == 0) {
            if (lane == 0) st_volatile_u64(&status[0], kScanIncl | block_total);
        } else {
            if (lane == 0) st_volatile_u64(&status[bid], kScanAgg | block_total);
            int64_t j = (int64_t)bid - 1 - lane;
            while (true) {
                unsigned long long s = 0;
                if (j >= 0) {
                    do {
                        s = ld_volatile_u64(&status[j]);
                    } while ((s >> 62) == 0);
                } else {
                    s = kScanIncl;  // virtual inclusive zero before block 0
                }
                const uint32_t incl_mask = __ballot_sync(0xffffffffu, (s >> 62) == 2);
                if (incl_mask) {
                    const int first = __ffs(incl_mask) - 1;  // nearest inclusive predecessor
                    unsigned long long val = lane <= first ? (s & kScanValMask) : 0ull;
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                    prefix += val;
                    break;
                }
                unsigned long long val = s & kScanValMask;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(0xffffffffu, val, o);
                prefix += val;
                j -= 32;
            }
            if (lane == 0) st_volatile_u64(&status[bid], kScanIncl | (prefix + block_total));
        }
        if (lane == 0) {
            s_prefix = prefix;
            if ((int64_t)(bid + 1) * kScanTile >= n && d_total) *d_total = (uint32_t)(prefix + block_total);
        }
    }
    __syncthreads();
    unsigned long long run = s_prefix + s_warp[warp] + (incl - tsum);
    uint32_t o[kScanIT];
#pragma unroll
    for (int i = 0; i < kScanIT; ++i) {
        o[i] = (uint32_t)run;
        run += v[i];
    }
    if (base + kScanIT <= n && ((reinterpret_cast<uintptr_t>(out + base) & 15) == 0)) {
        *reinterpret_cast<uint4*>(out + base) = make_uint4(o[0], o[1], o[2], o[3]);
        *reinterpret_cast<uint4*>(out + base + 4) = make_uint4(o[4], o[5], o[6], o[7]);
    } else {
#pragma unroll
        for (int i = 0; i < kScanIT; ++i)
            if (base + i < n) out[base + i] = o[i];
    }
}

// ------------------------------------------------------------------ radix sort
__global__ void __launch_bounds__(256) histogram_kernel(const uint32_t* __restrict__ keys,
                                                        int64_t n, int passes,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t s_h[4][kRadix];
    for (int i = threadIdx.x; i < 4 * kRadix; i += blockDim.x) (&s_h[0][0])[i] = 0;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t k = keys[i];
        for (int p = 0; p < passes; ++p) atomicAdd(&s_h[p][(k >> (8 * p)) & 0xff], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += blockDim.x) {
        const uint32_t c = (&s_h[0][0])[i];
        if (c) atomicAdd(&hist[i], c);
    }
}

__global__ void __launch_bounds__(kSortBT) onesweep_pass(
    const uint32_t* __restrict__ keys_in, const uint32_t* __restrict__ vals_in,
    uint32_t* __restrict__ keys_out, uint32_t* __restrict__ vals_out, int64_t n, int shift,
    const uint32_t* __restrict__ hist, uint32_t* status, uint32_t* ticket) {
    __shared__ uint32_t s_warp[kSortBT / 32][kRadix];
    __shared__ uint32_t s_base[kRadix];
    __shared__ uint32_t s_wsum[kSortBT / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < (kSortBT / 32) * kRadix; i += kSortBT) (&s_warp[0][0])[i] = 0;
    // global digit offsets: exclusive scan of this pass's histogram (thread tid = digit)
    const uint32_t hcount = hist[tid];
    uint32_t hincl = hcount;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, hincl, o);
        if (lane >= o) hincl += t;
    }
    if (lane == 31) s_wsum[warp] = hincl;
    __syncthreads();
    uint32_t wpre = 0;
    for (int w = 0; w < warp; ++w) wpre += s_wsum[w];
    const uint32_t g_off = wpre + hincl - hcount;
    const uint32_t bid = lookback_block(ticket);

    const int64_t base = (int64_t)bid * kSortTile + (int64_t)warp * (32 * kSortIT) + lane;
    uint32_t k[kSortIT], v[kSortIT];
    uint16_t r[kSortIT];
#pragma unroll
    for (int i = 0; i < kSortIT; ++i) {
        const int64_t idx = base + (int64_t)i * 32;
        if (idx < n) {
            k[i] = keys_in[idx];
            v[i] = vals_in[idx];
        }
    }
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int i = 0; i < kSortIT; ++i) {
        const int64_t idx = base + (int64_t)i * 32;
        const bool valid = idx < n;
        const uint32_t vm = __ballot_sync(0xffffffffu, valid);
        uint32_t before = 0, peers = 0, d = 0;
        if (valid) {
            d = (k[i] >> shift) & 0xffu;
            peers = __match_any_sync(vm, d);
            before = s_warp[warp][d];
            r[i] = (uint16_t)(before + __popc(peers & lt));
        }
        __syncwarp();
        if (valid && (lane == __ffs(peers) - 1)) s_warp[warp][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // thread tid = digit: cross-warp exclusive prefix, block count, look-back
    {
        uint32_t run = 0;
#pragma unroll
        for (int w = 0; w < kSortBT / 32; ++w) {
            const uint32_t t = s_warp[w][tid];
            s_warp[w][tid] = run;
            run += t;
        }
        const uint32_t cnt = run;
        uint32_t excl = 0;
        if (bid == 0) {
            st_volatile_u32(&status[tid], kSortIncl | cnt);
        } else {
            st_volatile_u32(&status[(size_t)bid * kRadix + tid], kSortAgg | cnt);
            int64_t j = (int64_t)bid - 1;
            while (true) {
                uint32_t s;
                do {
                    s = ld_volatile_u32(&status[(size_t)j * kRadix + tid]);
                } while ((s >> 30) == 0);
                excl += s & kSortValMask;
                if ((s >> 30) == 2) break;
                --j;
            }
            st_volatile_u32(&status[(size_t)bid * kRadix + tid], kSortIncl | (excl + cnt));
        }
        s_base[tid] = g_off + excl;
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < kSortIT; ++i) {
        const int64_t idx = base + (int64_t)i * 32;
        if (idx < n) {
            const uint32_t d = (k[i] >> shift) & 0xffu;
            const uint32_t pos = s_base[d] + s_warp[warp][d] + r[i];
            keys_out[pos] = k[i];
            vals_out[pos] = v[i];
        }
    }
}

__global__ void iota_kernel(uint32_t* v, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) v[i] = (uint32_t)i;
}

// keys[j] = orderable(depth[vals[j]]) / id words of vals[j]
__global__ void gather_sort_keys(const uint32_t* __restrict__ vals, const float* __restrict__ depth,
                                 const uint64_t* __restrict__ ids, int which, uint32_t* keys,
                                 int64_t n) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const uint32_t i = vals[j];
    uint32_t k;
    if (which == 0) k = orderable_key(depth[i]);
    else if (which == 1) k = (uint32_t)(ids[i] & 0xffffffffu);
    else k = (uint32_t)(ids[i] >> 32);
    keys[j] = k;
}

__global__ void invert_perm_kernel(const uint32_t* __restrict__ perm, uint32_t* __restrict__ rank_of,
                                   int64_t n) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r < n) rank_of[perm[r]] = (uint32_t)r;
}

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

}  // namespace

// ------------------------------------------------------------------ launchers
cudaError_t launch_exclusive_scan(tgsx_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                                  uint32_t* d_total) {
    if (n <= 0) {
        if (d_total) return cudaMemsetAsync(d_total, 0, sizeof(uint32_t), ctx->stream);
        return cudaSuccess;
    }
    const int64_t blocks = (n + kScanTile - 1) / kScanTile;
    const size_t need = 64 + (size_t)blocks * sizeof(unsigned long long);
    cudaError_t e = ctx->ws.scan_tmp.ensure(need);
    if (e) return e;
    uint32_t* ticket = ctx->ws.scan_tmp.as<uint32_t>();
    unsigned long long* status =
        reinterpret_cast<unsigned long long*>(ctx->ws.scan_tmp.as<char>() + 64);
    if ((e = cudaMemsetAsync(ctx->ws.scan_tmp.p, 0, need, ctx->stream))) return e;
    exclusive_scan_kernel<<<(unsigned)blocks, kScanBT, 0, ctx->stream>>>(in, out, n, status,
                                                                         ticket, d_total);
    ctx->launches++;
    return cudaGetLastError();
}

// Scratch (histograms + tickets + look-back status) sort_pairs needs for n keys.
size_t sort_scratch_bytes(int64_t n, int key_bits) {
    const int passes = std::max((key_bits + 7) / 8, 1);
    const int64_t blocks = (n + kSortTile - 1) / kSortTile;
    return 4 * kRadix * sizeof(uint32_t) + 64 + (size_t)passes * blocks * kRadix * sizeof(uint32_t);
}

// Sorts (keys, vals) on the low key_bits bits. keys/vals are updated to point at whichever
// buffer holds the result. d_hist (optional): precomputed [passes][256] histograms.
cudaError_t sort_pairs(tgsx_ctx* ctx, uint32_t*& keys, uint32_t*& vals, uint32_t* keys_alt,
                       uint32_t* vals_alt, int64_t n, int key_bits, const uint32_t* d_hist) {
    if (n <= 1 || key_bits <= 0) return cudaSuccess;
    const int passes = (key_bits + 7) / 8;
    const int64_t blocks = (n + kSortTile - 1) / kSortTile;
    const size_t hist_bytes = 4 * kRadix * sizeof(uint32_t);
    const size_t ticket_bytes = 64;
    const size_t status_bytes = (size_t)passes * blocks * kRadix * sizeof(uint32_t);
    cudaError_t e = ctx->ws.sort_tmp.ensure(hist_bytes + ticket_bytes + status_bytes);
    if (e) return e;
    char* base = ctx->ws.sort_tmp.as<char>();
    uint32_t* hist = reinterpret_cast<uint32_t*>(base);
    uint32_t* tickets = reinterpret_cast<uint32_t*>(base + hist_bytes);
    uint32_t* status = reinterpret_cast<uint32_t*>(base + hist_bytes + ticket_bytes);
    if (d_hist) {
        if ((e = cudaMemsetAsync(tickets, 0, ticket_bytes + status_bytes, ctx->stream))) return e;
        hist = const_cast<uint32_t*>(d_hist);
    } else {
        if ((e = cudaMemsetAsync(base, 0, hist_bytes + ticket_bytes + status_bytes, ctx->stream)))
            return e;
        const unsigned g = (unsigned)std::min<int64_t>(blocks * 4, 148 * 8);
        histogram_kernel<<<g, 256, 0, ctx->stream>>>(keys, n, passes, hist);
        ctx->launches++;
    }
    for (int p = 0; p < passes; ++p) {
        onesweep_pass<<<(unsigned)blocks, kSortBT, 0, ctx->stream>>>(
            keys, vals, keys_alt, vals_alt, n, 8 * p, hist + p * kRadix,
            status + (size_t)p * blocks * kRadix, tickets + p);
        ctx->launches++;
        std::swap(keys, keys_alt);
        std::swap(vals, vals_alt);
    }
    return cudaGetLastError();
}

// Blend order: perm[rank] = model index, rank_of[index] = rank.
cudaError_t launch_sort_depth(tgsx_ctx* ctx, tgsx_model* m) {
    const int64_t n = m->n;
    if (n == 0) {
        m->order_dirty = false;
        return cudaSuccess;
    }
    Workspace& ws = ctx->ws;
    cudaError_t e;
    // ties are broken by id in logical order: sort the logical layout
    if ((e = model_to_logical_order(ctx, m))) return e;
    ctx->bin_valid = false;  // the sort reuses the binning buffers
    for (int i = 0; i < 2; ++i) {
        if ((e = ws.keys[i].ensure(std::max<int64_t>(m->cap, n) * 4))) return e;  // by capacity (growing fits)
        if ((e = ws.vals[i].ensure(std::max<int64_t>(m->cap, n) * 4))) return e;
    }
    uint32_t* k = ws.keys[0].as<uint32_t>();
    uint32_t* v = ws.vals[0].as<uint32_t>();
    uint32_t* k2 = ws.keys[1].as<uint32_t>();
    uint32_t* v2 = ws.vals[1].as<uint32_t>();
    const float* depth = m->params.as<float>() + 9 * m->cap;
    const uint64_t* ids = m->ids.as<uint64_t>();
    iota_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(v, n);
    ctx->launches++;
    if (!m->ids_monotone) {
        // LSD: id low word, id high word, then depth (stable at every stage)
        const bool hi = m->next_id > 0xffffffffull;
        for (int which = 1; which <= (hi ? 2 : 1); ++which) {
            gather_sort_keys<<<grid_for(n, 256), 256, 0, ctx->stream>>>(v, depth, ids, which, k, n);
            ctx->launches++;
            // 4 passes: the result lands back in (k, v)
            if ((e = sort_pairs(ctx, k, v, k2, v2, n, 32, nullptr))) return e;
        }
    }
    gather_sort_keys<<<grid_for(n, 256), 256, 0, ctx->stream>>>(v, depth, ids, 0, k, n);
    ctx->launches++;
    if ((e = sort_pairs(ctx, k, v, k2, v2, n, 32, nullptr))) return e;
    if ((e = cudaMemcpyAsync(m->perm.p, v, n * 4, cudaMemcpyDeviceToDevice, ctx->stream))) return e;
    invert_perm_kernel<<<grid_for(n, 256), 256, 0, ctx->stream>>>(
        m->perm.as<uint32_t>(), m->rank_of.as<uint32_t>(), n);
    ctx->launches++;
    m->order_dirty = false;
    m->spatial_valid = false;  // the ranks changed: the claim order is rebuilt at the next binning
    return cudaGetLastError();
}

}  // namespace tgsx
