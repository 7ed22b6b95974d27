// Device-side helpers shared by the tgsx kernels (sm_100a).
//
// Bit-exact stages (preprocess, binning, Adam, densify predicates) must round exactly like
// the reference built with -ffp-contract=off (proj/CMakeLists.txt:12): every float op there
// is written with an explicit round-to-nearest intrinsic so nvcc can never contract it into
// an FMA. Transcendentals follow the correctly-rounded contract (oracle/cr_libm.c):
// f(float x) := round_to_float(f_double((double)x)).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tgsx {

constexpr int kTile = 16;                 // rasterizer.hpp:12
constexpr float kTermT = 1e-4f;           // rasterizer.hpp:14 (float(1e-4))
constexpr float kMinVisitW = 1e-4f;       // rasterizer.hpp:17
constexpr float kCullSigmas = 3.0f;       // rasterizer.hpp:19
constexpr double kMinScale = 1e-4;        // gaussian.hpp:14
constexpr double kRawCap = 12.0;          // gaussian.hpp:18
constexpr int kParams = 9;                // optimised components per Gaussian
constexpr int kStepFloats = 12;           // step buffer: 9 grads + pos norm + col norm + visits
// One Gaussian's step-buffer record. The batched-view step buffer is AoS [n][12] floats (48 B per
// Gaussian, rows in the model's physical order): any Gaussian range is one contiguous slice, so the
// all-reduce moves exactly 48 n bytes and a bucket [i0, i1) of the chain -> all-reduce -> Adam
// pipeline is one contiguous NCCL buffer.
struct alignas(16) StepRec {
    float4 a, b, c;  // (g0..g3), (g4..g7), (g8, pos norm, colour norm, visits)
};

// Kernel error word: (rank << 2) | code, lowest wins; all-ones = no error.
constexpr unsigned long long kErrNone = ~0ull;

// ------------------------------------------------------------------ CR transcendentals
__device__ __forceinline__ float cr_expf(float x) { return __double2float_rn(exp((double)x)); }
__device__ __forceinline__ float cr_logf(float x) { return __double2float_rn(log((double)x)); }
__device__ __forceinline__ void cr_sincosf(float x, float* s, float* c) {
    double sd, cd;
    sincos((double)x, &sd, &cd);
    *s = __double2float_rn(sd);
    *c = __double2float_rn(cd);
}

// ------------------------------------------------------------------ exact float ops
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float fdiv(float a, float b) { return __fdiv_rn(a, b); }

// a / b correctly rounded (== __fdiv_rn) for b > 0, without the division's slow-path subroutine
// for a zero dividend: FCHK sends any lane with a zero / denormal operand there, and one such lane
// makes the whole warp pay (Adam moments of components that never saw a gradient are exactly 0).
// +-0 / b = +-0 for b > 0, so the substitution is exact.
__device__ __forceinline__ float fdiv_pos(float a, float b) {
    const float q = __fdiv_rn(a == 0.0f ? 1.0f : a, b);
    return a == 0.0f ? a : q;
}
// sqrt correctly rounded (== __fsqrt_rn) without the slow path for a zero argument.
__device__ __forceinline__ float fsqrt_nz(float a) {
    const float r = __fsqrt_rn(a == 0.0f ? 1.0f : a);
    return a == 0.0f ? a : r;
}

// activate (gaussian.hpp:47-49): 1 / (1 + exp(-raw))
__device__ __forceinline__ float activate_cr(float raw) {
    return fdiv(1.0f, fadd(1.0f, cr_expf(-raw)));
}

// static_cast<int>(double) as the reference's x86-64 build executes it (cvttsd2si): values
// outside int range and NaN become INT_MIN ("integer indefinite"), where the GPU's native
// conversion would saturate. Keeps off-image / non-finite splats unbinned exactly like the
// reference.
__device__ __forceinline__ int x86_double_to_int(double v) {
    return (v >= -2147483648.0 && v < 2147483648.0) ? (int)v : (int)0x80000000;
}

// pixel_span (rasterizer.cpp:50-56): float m±r, then double ceil/floor of (value - 0.5).
__device__ __forceinline__ void pixel_span(float m, float r, int limit, int& lo, int& hi) {
    lo = x86_double_to_int(ceil(__dsub_rn((double)fsub(m, r), 0.5)));
    hi = x86_double_to_int(floor(__dsub_rn((double)fadd(m, r), 0.5)));
    if (lo < 0) lo = 0;
    if (hi > limit - 1) hi = limit - 1;
}

// Tile rectangle of a prepared splat (rasterizer.cpp:74-84); false when off-image.
__device__ __forceinline__ bool tile_rect(float mx, float my, float rx, float ry, int W, int H,
                                          int& tx0, int& tx1, int& ty0, int& ty1) {
    int px0, px1, py0, py1;
    pixel_span(mx, rx, W, px0, px1);
    pixel_span(my, ry, H, py0, py1);
    if (px0 > px1 || py0 > py1) return false;
    tx0 = px0 / kTile;
    tx1 = px1 / kTile;
    ty0 = py0 / kTile;
    ty1 = py1 / kTile;
    return true;
}

// DilationPattern::first_active_at_or_after (dilation.hpp:49-53)
__device__ __forceinline__ int first_active(int v, int offset, int p) {
    if (v <= offset) return offset;
    const int k = (v - offset + p - 1) / p;
    return offset + k * p;
}

// Orderable u32 of a float depth key (ascending float order; -0 canonicalised to +0 so that
// -0 == +0 ties fall through to the id order like the reference comparator, model.hpp:111).
__device__ __forceinline__ uint32_t orderable_key(float f) {
    uint32_t u = __float_as_uint(f);
    if (u == 0x80000000u) u = 0u;
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}

// ------------------------------------------------------------------ fused block scan
// Block index of a fused decoupled look-back: 1-D grids are dispatched in blockIdx order, so every
// predecessor a block waits on is resident or finished (the CUB DeviceScan convention). A
// launch-order ticket — one global atomic on a single counter per block, with the whole block
// waiting for it at a barrier — measured 9 us (C2) / 16 us (C3) slower per 2-D preprocess; the
// ticket word stays in the signature (zeroed by the launcher) but is not used.
__device__ __forceinline__ uint32_t lookback_block(const uint32_t* /*ticket*/) { return blockIdx.x; }

// Exclusive prefix of `v` over a launch-ordered sequence of 256-thread blocks (block `bid`, all
// threads call it): block scan + decoupled look-back over status[] (flag 2 bits | value 62 bits,
// zeroed before the launch; bid = lookback_block(): a block only waits on dispatched blocks).
// The block holding element n-1 writes the grand total to *d_total.
constexpr unsigned long long kLbAgg = 1ull << 62, kLbIncl = 2ull << 62, kLbMask = (1ull << 62) - 1;

__device__ __forceinline__ uint32_t block_scan_lookback(uint32_t v, uint32_t bid, int64_t n,
                                                        unsigned long long* status, uint32_t* d_total) {
    __shared__ uint32_t s_warp[8];
    __shared__ unsigned long long s_prefix;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t incl = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, incl, d);
        if (lane >= d) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const uint32_t w = lane < 8 ? s_warp[lane] : 0u;
        uint32_t wi = w;
#pragma unroll
        for (int d = 1; d < 8; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, wi, d);
            if (lane >= d) wi += t;
        }
        if (lane < 8) s_warp[lane] = wi - w;
        const unsigned long long block_total = __shfl_sync(0xffffffffu, wi, 7);
        unsigned long long prefix = 0;
        if (bid == 0) {
            if (lane == 0) atomicExch(&status[0], kLbIncl | block_total);
        } else {
            if (lane == 0) atomicExch(&status[bid], kLbAgg | block_total);
            int64_t j = (int64_t)bid - 1 - lane;
            while (true) {
                unsigned long long s = kLbIncl;  // virtual inclusive zero before block 0
                if (j >= 0) {
                    do {
                        s = *reinterpret_cast<volatile unsigned long long*>(&status[j]);
                    } while ((s >> 62) == 0);
                }
                const uint32_t im = __ballot_sync(0xffffffffu, (s >> 62) == 2);
                unsigned long long val = (!im || lane <= __ffs(im) - 1) ? (s & kLbMask) : 0ull;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) val += __shfl_xor_sync(0xffffffffu, val, d);
                prefix += val;
                if (im) break;
                j -= 32;
            }
            if (lane == 0) atomicExch(&status[bid], kLbIncl | (prefix + block_total));
        }
        if (lane == 0) {
            s_prefix = prefix;
            if ((int64_t)(bid + 1) * 256 >= n) *d_total = (uint32_t)(prefix + block_total);
        }
    }
    __syncthreads();
    return (uint32_t)s_prefix + s_warp[warp] + (incl - v);
}

// ------------------------------------------------------------------ prepared splat record
// 64 B per splat, blend (rank) order:
//   a = (mean x, mean y, inv00, inv01)   b = (inv11, alpha, rx, ry)
//   c = (r, g, b, orig as bits)          d = (rect x packed, rect y packed, pair offset, tiles)
// (pair offset = the splat's first partial slot = pair_off[rank], written by the binning)
// rect packed = lo | hi << 16 (tile units); tiles == 0 => not binned.
struct __align__(16) Prepared {
    float4 a, b, c;
    uint4 d;
};

// ------------------------------------------------------------------ backward partials
// One entry per (tile, splat) pair slot, SoA (40 B/pair):
//   a[s] = (d mean x, d mean y, d Sigma'00, d Sigma'01)
//   b[s] = (d Sigma'11, d alpha, d r, d g)
//   c[s] = (d b, visited 0/1)
struct Partials {
    float4* a;
    float4* b;
    float2* c;
    __host__ __device__ static Partials at(void* base, int64_t cap) {
        Partials p;
        p.a = reinterpret_cast<float4*>(base);
        p.b = p.a + cap;
        p.c = reinterpret_cast<float2*>(p.b + cap);
        return p;
    }
};

// ------------------------------------------------------------------ blend math
// log2(e) * -0.5: G = exp(-q/2) = exp2(q * kNegHalfLog2e). Shared by forward and backward so
// the recomputed sigma is bit-identical (the backward's T recovery relies on it).
constexpr float kNegHalfLog2e = -0.72134752044448170368f;

__device__ __forceinline__ float fast_exp2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// q = inv00 dx^2 + 2 inv01 dx dy + inv11 dy^2 with a fixed FMA schedule; returns G.
__device__ __forceinline__ float splat_gauss(float i00, float i01x2, float i11, float dx,
                                             float dy) {
    const float t = __fmul_rn(i11, dy);
    const float u = __fmaf_rn(i01x2, dx, t);          // 2 i01 dx + i11 dy
    const float v = __fmul_rn(u, dy);                 // (2 i01 dx + i11 dy) dy
    const float q = __fmaf_rn(__fmul_rn(i00, dx), dx, v);
    return fast_exp2(__fmul_rn(q, kNegHalfLog2e));
}

// Same quadratic form with the conic pre-scaled by kNegHalfLog2e (ka = inv00 K, kb = 2 inv01 K,
// kc = inv11 K): G = exp2(ka dx^2 + kb dx dy + kc dy^2). The blend kernels use this form in
// both passes (identical instruction sequence => bit-identical sigma for the T recovery).
__device__ __forceinline__ float conic_gauss(float ka, float kb, float kc, float dx, float dy) {
    const float v = __fmul_rn(__fmaf_rn(kb, dx, __fmul_rn(kc, dy)), dy);
    return fast_exp2(__fmaf_rn(__fmul_rn(ka, dx), dx, v));
}

// Exact box-test mask over the tile's active columns (or rows): bit c set iff
// |float(a0 + c p) + 0.5 - m| <= r (rasterizer.cpp:116-118, same float rounding). The centres
// increase with c and the rounded difference is monotonic in the centre, so the passing
// columns form one interval: its ends are estimated in real arithmetic (off by at most one
// column) and then settled with the exact test itself.
__device__ __forceinline__ bool box_pass(float m, float r, int a0, int p, int c) {
    const float d = __fsub_rn(__fadd_rn((float)(a0 + c * p), 0.5f), m);
    return fabsf(d) <= r;
}
__device__ __forceinline__ uint32_t box_mask(float m, float r, int a0, int p, int count) {
    if (count <= 0) return 0u;
    const float base = (float)a0 + 0.5f, inv_p = 1.0f / (float)p;
    float lo = ceilf(((m - r) - base) * inv_p), hi = floorf(((m + r) - base) * inv_p);
    lo = fminf(fmaxf(lo, 0.f), (float)count);
    hi = fminf(fmaxf(hi, -1.f), (float)(count - 1));
    int cl = (int)lo, ch = (int)hi;
    if (cl > 0 && box_pass(m, r, a0, p, cl - 1)) --cl;
    else if (cl < count && !box_pass(m, r, a0, p, cl)) ++cl;
    if (ch < count - 1 && box_pass(m, r, a0, p, ch + 1)) ++ch;
    else if (ch >= 0 && !box_pass(m, r, a0, p, ch)) --ch;
    if (cl > ch) return 0u;
    return (uint32_t)((2ull << ch) - (1ull << cl));
}

__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// 32-bit shared-window loads/stores (keeps address arithmetic out of the hot loops)
__device__ __forceinline__ float4 lds_f4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float2 lds_f2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds_f1(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f1(uint32_t a, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v));
}
__device__ __forceinline__ void sts_f2(uint32_t a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1,%2};" ::"r"(a), "f"(v.x), "f"(v.y));
}
__device__ __forceinline__ void sts_f4(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w));
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

// ------------------------------------------------------------------ TMA bulk copies
// 1-D bulk copies global -> shared on the TMA engine (cp.async.bulk), completion counted in
// bytes on a shared-memory mbarrier (arrive.expect_tx by one lane, complete_tx by the copies).
// The blend kernels gather their prepared records one 64-B bulk copy per list entry, a chunk
// ahead of the walk, so the record gathers' DRAM latency overlaps the previous chunk's blending.
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
// makes mbarrier initialisation visible to the async (TMA) proxy
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// orders this thread's earlier generic-proxy shared accesses before later async-proxy writes
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// ------------------------------------------------------------------ misc
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

__device__ __forceinline__ void raise_error(unsigned long long* err, uint32_t rank,
                                            uint32_t code) {
    // lowest (rank, code) wins, i.e. the first failing splat in blend order (the reference
    // throws at the first failure while walking sorted order, rasterizer.cpp:28-32)
    atomicMin(err, ((unsigned long long)rank << 2) | code);
}

}  // namespace tgsx
