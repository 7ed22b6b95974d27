// Alpha-blend forward and backward over the per-tile splat lists (sm_100a, FP32 pipe).
//
// The tile's active pixels (the dilated variant keeps only x%p==ox, y%p==oy, so p selects the
// geometry and the same kernels serve p = 1 and the paper's 4K dilated rendering) are covered
// by warps. The tile's splat list is consumed in chunks of 32 staged as 48-byte shared-memory
// records together with exact per-tile box-test masks (rasterizer.cpp:116-118, evaluated once
// per (tile, splat) in float: the passing active columns / rows form one interval, settled by
// the exact test at its two ends). Per chunk one 5-stage shuffle bit-transpose of the 32 masks
// hands lane c the set of splats passing active column c and lane 16 + r those passing row r;
// a pixel's pass set is one AND of a column and a row set (two shuffles). Per pixel the order is
// the list order and box-failing splats contribute nothing, exactly as in walk_pixel
// (rasterizer.cpp:108-136).
//
// forward_pairs_kernel (p = 1: one CTA per tile, one warp per 8x8 block, two pixels per lane as
//   packed FP32x2, 256-record staging batches): walk_pixel + render (rasterizer.cpp:144-184),
//   optional fused L1 epilogue. Records per pixel the final T and the last
//   blended list position.
// forward_dilated_kernel (p >= 2: one warp per tile, the next chunk's records gathered by
//   cp.async while the current chunk is walked): the same walk for the tile's <= 8x8 active pixels.
// backward_kernel (ONE WARP PER TILE from a tile queue, independent warps, no block barriers;
//   backward_cta_kernel for views with few tiles: one CTA per tile, a warp per 8x8 group, the
//   group sums added through shared memory): backward tile phase (rasterizer.cpp:234-292), per
//   chunk and 8x4 pixel group:
//   1. per pixel, back to front over the union of the group's walked splats (all lanes on the
//      same splat): T_i = T_{i+1} / (1 - sigma_i) with sigma recomputed bit-identically to the
//      forward; g.dC/dsigma_i = T_i (g.c_i) - (g.S_i)/(1 - sigma_i) with the reference's exact
//      suffix S_i (rasterizer.cpp:266-287) carried as the scalar g.S; records u = dL/dsigma * G
//      and the blend weight w per (splat, pixel) in a dense shared-memory row per splat;
//   2. per record row and half (lane 2i + h), dense over the half's 32 pixels: every position /
//      covariance gradient of rasterizer.cpp:276-285 is linear in the moments sum(u), sum(u dx),
//      sum(u dy), sum(u dx^2), sum(u dx dy), sum(u dy^2) and the colour gradient is sum(g w);
//      with fixed pixel offsets these are packed FADD2 / FFMA2 sums, handed (through the just
//      read rows) to lane j = the row's splat and accumulated across the tile's groups in its
//      registers. After the chunk lane j converts them to the 9 screen-space gradients
//      and writes its (tile, splat) pair slot once — no reductions, no atomics, deterministic;
//      the per-Gaussian merge in optim.cu walks the slots in tile order like
//      rasterizer.cpp:301-319.
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>

namespace tgsx {

namespace {

constexpr uint32_t kFull = 0xffffffffu;
constexpr int kRec = 48;        // bytes per staged splat record
constexpr int kWPB = 4;         // warps (tiles) per CTA
#ifndef TGSX_BWD_MINB
#define TGSX_BWD_MINB 4
#endif

struct BlendParams {
    const uint2* ranges;
    const uint32_t* items;
    const Prepared* prep;
    int tiles, tiles_x, p, ox, oy, W, H, cols;
    float bg0, bg1, bg2;
    float* rgb;
    float* T;
    uint32_t* last;
    unsigned long long* counters;  // [1] blend ops, [2] evaluations
    const float* target;           // fused L1 (forward)
    int target_rows;               // > 1: target holds only the active rows (dilated host targets)
    float* dLdC;
    float* block_loss;
    float loss_scale;
    Partials partial;              // backward output, one entry per pair slot
    unsigned int* tile_queue;      // backward: next tile to take (zeroed before the launch)
    // graph-replayed steps (graph.cpp): the backward checks the binning counters against the
    // capacities the graph was captured with; a violation (or a kernel error) sets *fault, which
    // turns this and every later replayed step into a no-op until the host re-runs them eagerly
    unsigned* fault;
    uint32_t guard_pairs, guard_list;
};

struct TileGeo {
    int tx, ty, ax, ay, acols, arows;
    __device__ __forceinline__ void init(const BlendParams& prm, int tile) {
        tx = tile % prm.tiles_x;
        ty = tile / prm.tiles_x;
        const int x0 = tx * kTile, y0 = ty * kTile;
        const int px1 = min(prm.W, x0 + kTile), py1 = min(prm.H, y0 + kTile);
        ax = first_active(x0, prm.ox, prm.p);
        ay = first_active(y0, prm.oy, prm.p);
        acols = ax < px1 ? (px1 - ax + prm.p - 1) / prm.p : 0;
        arows = ay < py1 ? (py1 - ay + prm.p - 1) / prm.p : 0;
    }
};

// 32x32 bit-matrix transpose across the warp: in lane j bit l = M[j][l]; out lane l bit j.
__device__ __forceinline__ uint32_t transpose32(uint32_t v) {
    const int lane = threadIdx.x & 31;
    const uint32_t ms[5] = {0x0000ffffu, 0x00ff00ffu, 0x0f0f0f0fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int s = 0; s < 5; ++s) {
        const int k = 16 >> s;
        const uint32_t m = ms[s];
        const uint32_t x = __shfl_xor_sync(kFull, v, k);
        v = (lane & k) ? ((v & ~m) | ((x & ~m) >> k)) : ((v & m) | ((x & m) << k));
    }
    return v;
}

// Stages one prepared splat (and its pair slot) as a 48-byte record:
//   +0 (mean x, mean y, ka, kb)  +16 (kc, alpha, r, g)  +32 (b, tile mask, pair slot, -)
// (ka, kb, kc) = (inv00, 2 inv01, inv11) * kNegHalfLog2e; mask = active cols | rows << 16.
__device__ __forceinline__ void stage_splat(const Prepared& P, const TileGeo& g, int p, uint32_t slot,
                                            uint32_t dst) {
    const float4 a = P.a, b = P.b, c = P.c;
    const uint32_t mask =
        box_mask(a.x, b.z, g.ax, p, g.acols) | (box_mask(a.y, b.w, g.ay, p, g.arows) << 16);
    sts_f4(dst, make_float4(a.x, a.y, __fmul_rn(a.z, kNegHalfLog2e), __fmul_rn(a.w * 2.0f, kNegHalfLog2e)));
    sts_f4(dst + 16, make_float4(__fmul_rn(b.x, kNegHalfLog2e), b.y, c.x, c.y));
    sts_f4(dst + 32, make_float4(c.z, __uint_as_float(mask), __uint_as_float(slot), 0.f));
}

// ------------------------------------------------------------------------ forward (pairs)
// Exponent of conic_gauss for two pixels in the same column (rows fyA, fyB) as packed FP32x2,
// the same op sequence (and rounding) per pixel as conic_gauss: a = (mx, my, ka, kb), kc.
__device__ __forceinline__ float2 pair_quad(const float4& a, float kc, float fx, float fyA, float fyB) {
    const float dx = __fsub_rn(fx, a.x);
    const float2 dy = __fadd2_rn(make_float2(fyA, fyB), make_float2(-a.y, -a.y));  // exact negation
    const float2 t = __fmul2_rn(make_float2(kc, kc), dy);
    const float2 u = __ffma2_rn(make_float2(a.w, a.w), make_float2(dx, dx), t);
    const float2 v = __fmul2_rn(u, dy);
    const float kadx = __fmul_rn(a.z, dx);
    return __ffma2_rn(make_float2(kadx, kadx), make_float2(dx, dx), v);
}


// One chunk (<= 32 staged records at cbase, list positions lbase-1 ...) of walk_pixel
// (rasterizer.cpp:108-136) for the lane's two pixels of the 8x8 block (bx, by) of active pixels:
// masks transposed (lane c < 16 holds the chunk's splats passing active column c, lane 16 + r
// those passing row r; a pixel's pass set is column & row), then the union of the lane's two
// pass sets front to back, two splats per iteration, packed FP32x2. Returns true when every
// pixel of the warp has terminated.
__device__ __forceinline__ bool walk_chunk(uint32_t cbase, int ccount, uint32_t lbase, int bx, int by, float fx,
                                           float fyA, float fyB, float2& T, float2& C0, float2& C1, float2& C2,
                                           uint32_t& lastA, uint32_t& lastB, uint32_t& ops, bool& doneA,
                                           bool& doneB) {
    const int lane = threadIdx.x & 31;
    // pass sets: bit k = splat k of the chunk
    const uint32_t bits = transpose32(lane < ccount ? __float_as_uint(lds_f1(cbase + lane * kRec + 36)) : 0u);
    const uint32_t X = __shfl_sync(kFull, bits, bx * 8 + (lane & 7));
    uint32_t colA = X & __shfl_sync(kFull, bits, 16 + by * 8 + 2 * (lane >> 3));
    uint32_t colB = X & __shfl_sync(kFull, bits, 17 + by * 8 + 2 * (lane >> 3));
    if (doneA) colA = 0;
    if (doneB) colB = 0;
    const uint32_t colA0 = colA, colB0 = colB;
    int termA = 32, termB = 32;  // splat of each pixel's terminating blend, 32 = none
    uint32_t colU = colA | colB;
    // Two splats (k1 < k2) per iteration, lowest first (x & -x, its index one FLO): their
    // Gaussians are independent (ILP), the blends are applied in order and a ray that terminates
    // at k1 does not blend k2. Branch-free: an empty set gives a zero bit and index -1, the spare
    // record slot in front of the chunk (finite contents, both pixels masked: sigma = 0 changes
    // nothing).
    while (__any_sync(kFull, colU)) {
        const uint32_t bit1 = colU & (0u - colU);
        const int k1 = 31 - __clz(bit1);
        const uint32_t rem = colU ^ bit1;
        const uint32_t bit2 = rem & (0u - rem);
        const int k2 = 31 - __clz(bit2);
        const bool hA1 = (colA & bit1) != 0u, hB1 = (colB & bit1) != 0u;
        const bool hA2 = (colA & bit2) != 0u, hB2 = (colB & bit2) != 0u;
        const uint32_t ad1 = cbase + k1 * kRec, ad2 = cbase + k2 * kRec;
        const float4 a1 = lds_f4(ad1), b1 = lds_f4(ad1 + 16);
        const float4 a2 = lds_f4(ad2), b2 = lds_f4(ad2 + 16);
        const float cz1 = lds_f1(ad1 + 32), cz2 = lds_f1(ad2 + 32);
        const float2 q1 = pair_quad(a1, b1.x, fx, fyA, fyB);
        const float2 q2 = pair_quad(a2, b2.x, fx, fyA, fyB);
        const float2 e1 = make_float2(fast_exp2(q1.x), fast_exp2(q1.y));
        const float2 e2 = make_float2(fast_exp2(q2.x), fast_exp2(q2.y));
        // a pixel that does not pass the splat gets sigma = 0 (T, colour unchanged)
        const float2 s1 = make_float2(hA1 ? __fmul_rn(b1.y, e1.x) : 0.f, hB1 ? __fmul_rn(b1.y, e1.y) : 0.f);
        const float2 w1 = __fmul2_rn(s1, T);
        // 1 - sigma with one rounding, exactly as the scalar subtraction
        T = __fmul2_rn(T, __ffma2_rn(s1, make_float2(-1.0f, -1.0f), make_float2(1.0f, 1.0f)));
        C0 = __ffma2_rn(w1, make_float2(b1.z, b1.z), C0);
        C1 = __ffma2_rn(w1, make_float2(b1.w, b1.w), C1);
        C2 = __ffma2_rn(w1, make_float2(cz1, cz1), C2);
        const bool tA1 = hA1 && T.x < kTermT, tB1 = hB1 && T.y < kTermT;  // ray ends at k1
        const bool gA2 = hA2 && !tA1, gB2 = hB2 && !tB1;
        const float2 s2 = make_float2(gA2 ? __fmul_rn(b2.y, e2.x) : 0.f, gB2 ? __fmul_rn(b2.y, e2.y) : 0.f);
        const float2 w2 = __fmul2_rn(s2, T);
        T = __fmul2_rn(T, __ffma2_rn(s2, make_float2(-1.0f, -1.0f), make_float2(1.0f, 1.0f)));
        C0 = __ffma2_rn(w2, make_float2(b2.z, b2.z), C0);
        C1 = __ffma2_rn(w2, make_float2(b2.w, b2.w), C1);
        C2 = __ffma2_rn(w2, make_float2(cz2, cz2), C2);
        const bool tA2 = gA2 && T.x < kTermT, tB2 = gB2 && T.y < kTermT;
        colA &= ~(bit1 | bit2);
        colB &= ~(bit1 | bit2);
        if (tA1 || tA2) {  // ray A terminates (break after blending)
            termA = tA1 ? k1 : k2;
            colA = 0;
        }
        if (tB1 || tB2) {
            termB = tB1 ? k1 : k2;
            colB = 0;
        }
        colU = colA | colB;
    }
    // blended splats: the pass set up to the terminating one; the last is the highest set bit
    if (colA0) {
        const uint32_t used = termA < 32 ? (colA0 & (0xffffffffu >> (31 - termA))) : colA0;
        ops += __popc(used);
        lastA = lbase + 31 - __clz(used);
        if (termA < 32) doneA = true;
    }
    if (colB0) {
        const uint32_t used = termB < 32 ? (colB0 & (0xffffffffu >> (31 - termB))) : colB0;
        ops += __popc(used);
        lastB = lbase + 31 - __clz(used);
        if (termB < 32) doneB = true;
    }
    return __all_sync(kFull, doneA && doneB);
}

// Pixel epilogue of walk_pixel / render (rasterizer.cpp:131-133, 180-182): background term,
// outputs by dense rank, evaluation count, fused L1 value and dL/dC.
__device__ __forceinline__ void finish_pixel(const BlendParams& prm, bool valid, int x, int y, float Tp, float c0,
                                             float c1, float c2, uint32_t last, bool done, int count,
                                             unsigned long long& ev, float& lsum) {
    if (!valid) return;
    const int p = prm.p;
    c0 = __fmaf_rn(Tp, prm.bg0, c0);
    c1 = __fmaf_rn(Tp, prm.bg1, c1);
    c2 = __fmaf_rn(Tp, prm.bg2, c2);
    const int r = ((y - prm.oy) / p) * prm.cols + (x - prm.ox) / p;
    if (prm.rgb) {
        prm.rgb[3 * r] = c0;
        prm.rgb[3 * r + 1] = c1;
        prm.rgb[3 * r + 2] = c2;
    }
    prm.T[r] = Tp;
    prm.last[r] = last;
    ev += done ? last : (uint32_t)count;
    if (prm.target) {
        const int ty = prm.target_rows > 1 ? (y - prm.oy) / prm.target_rows : y;  // staged rows only
        const float* tg = prm.target + 3 * ((int64_t)ty * prm.W + x);
        const float d0 = c0 - tg[0], d1 = c1 - tg[1], d2 = c2 - tg[2];
        lsum += fabsf(d0) + fabsf(d1) + fabsf(d2);
        const float sc = prm.loss_scale;
        prm.dLdC[3 * r] = d0 > 0.f ? sc : (d0 < 0.f ? -sc : 0.f);
        prm.dLdC[3 * r + 1] = d1 > 0.f ? sc : (d1 < 0.f ? -sc : 0.f);
        prm.dLdC[3 * r + 2] = d2 > 0.f ? sc : (d2 < 0.f ? -sc : 0.f);
    }
}

// One CTA per tile, one warp per 8x8 block of active pixels, TWO vertically adjacent pixels per
// lane (rows 2r and 2r+1 of the block). The lane walks the union of its two pixels' passing
// splats front to back; the two Gaussians / blends of a splat run as packed FP32x2 (FMUL2 /
// FFMA2 with the splat's scalars broadcast), so one record read and one instruction stream
// serve two pixels. Every per-pixel quantity rounds exactly like walk_pixel
// (rasterizer.cpp:108-136) and like conic_gauss (the backward recomputes sigma from it).
template <int NWX, int NWY, int BATCH>
// <= 48 registers: 10 CTAs (40 warps) per SM instead of 8 at 63 registers (C2 0.358 -> 0.353 ms)
#ifndef TGSX_FWD_MINB
#define TGSX_FWD_MINB 10
#endif
__global__ void __launch_bounds__(NWX * NWY * 32, TGSX_FWD_MINB) forward_pairs_kernel(BlendParams prm) {
    constexpr int NW = NWX * NWY, NT = NW * 32;
    __shared__ __align__(16) unsigned char s_rec[(BATCH + 1) * kRec];  // the walk's spare slot + BATCH
    __shared__ unsigned long long s_red[2][NW];
    __shared__ float s_loss[NW];

    const int tile = blockIdx.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    TileGeo geo;
    geo.init(prm, tile);
    const int p = prm.p;
    const int bx = warp % NWX, by = warp / NWX;
    const int lx = bx * 8 + (lane & 7), lyA = by * 8 + 2 * (lane >> 3);
    const bool vA = lx < geo.acols && lyA < geo.arows;
    const bool vB = lx < geo.acols && lyA + 1 < geo.arows;
    const int x = geo.ax + lx * p, yA = geo.ay + lyA * p, yB = yA + p;
    const float fx = (float)x + 0.5f, fyA = (float)yA + 0.5f, fyB = (float)yB + 0.5f;
    const uint2 range = prm.ranges[tile];
    const int count = (int)(range.y - range.x);
    const uint32_t sbase = smem_addr(s_rec) + kRec;  // record j at sbase + j kRec; spare slot (-1) zeroed
    if (threadIdx.x < 3) sts_f4(sbase - kRec + 16 * threadIdx.x, make_float4(0.f, 0.f, 0.f, 0.f));

    float2 T = make_float2(1.0f, 1.0f);
    float2 C0 = make_float2(0.f, 0.f), C1 = C0, C2 = C0;
    uint32_t lastA = 0, lastB = 0, ops = 0;
    bool doneA = !vA, doneB = !vB;
    bool warp_done = __all_sync(kFull, doneA && doneB);

    for (int bstart = 0; bstart < count; bstart += BATCH) {
        if (__syncthreads_and(warp_done)) break;
        const int bcount = min(BATCH, count - bstart);
        for (int j = threadIdx.x; j < bcount; j += NT) {
            const Prepared& P = prm.prep[prm.items[range.x + bstart + j]];
            const float4 a = P.a, b = P.b, c = P.c;
            const uint32_t mask = box_mask(a.x, b.z, geo.ax, p, geo.acols) |
                                  (box_mask(a.y, b.w, geo.ay, p, geo.arows) << 16);
            const uint32_t dst = sbase + j * kRec;
            sts_f4(dst, make_float4(a.x, a.y, __fmul_rn(a.z, kNegHalfLog2e),
                                    __fmul_rn(a.w * 2.0f, kNegHalfLog2e)));
            sts_f4(dst + 16, make_float4(__fmul_rn(b.x, kNegHalfLog2e), b.y, c.x, c.y));
            sts_f4(dst + 32, make_float4(c.z, __uint_as_float(mask), 0.f, 0.f));
        }
        __syncthreads();
        if (warp_done) continue;
        for (int c0 = 0; c0 < bcount; c0 += 32) {
            if (walk_chunk(sbase + c0 * kRec, min(32, bcount - c0), (uint32_t)(bstart + c0 + 1), bx, by,
                           fx, fyA, fyB, T, C0, C1, C2, lastA, lastB, ops, doneA, doneB)) {
                warp_done = true;
                break;
            }
        }
    }

    float lsum = 0.f;
    unsigned long long ev = 0;
    finish_pixel(prm, vA, x, yA, T.x, C0.x, C1.x, C2.x, lastA, doneA, count, ev, lsum);
    finish_pixel(prm, vB, x, yB, T.y, C0.y, C1.y, C2.y, lastB, doneB, count, ev, lsum);
    unsigned long long o = ops;
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
        o += __shfl_xor_sync(kFull, o, sft);
        ev += __shfl_xor_sync(kFull, ev, sft);
        lsum += __shfl_xor_sync(kFull, lsum, sft);
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

// 16-byte global -> shared async copy (LDGSTS, L2 only), zero-fill when src_bytes == 0
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit_() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// Dilated forward (p >= 2: a tile's <= 8x8 active pixels are one warp's block): one warp per
// tile, independent warps (no block barriers). The list is consumed in chunks of 32; the raw
// 64-B prepared records of chunk c+1 are gathered by asynchronous copies (each lane copies its
// own list entry's record, four 16-B LDGSTS) while chunk c is walked, so the record gathers —
// the 3M-splat record array does not fit in L2 — do not stall the walk. Each lane then stages
// its own record of the arrived chunk (box mask, pre-scaled conic) exactly as the p = 1 kernel.
struct FwdWarpSmem {
    unsigned char raw[2][32 * sizeof(Prepared)];
    unsigned char rec[33 * kRec];  // the walk's spare slot + 32 records
};

template <int NWX, int NWY>
__global__ void __launch_bounds__(NWX * NWY * 32, 32 / (NWX * NWY)) forward_dilated_kernel(BlendParams prm) {
    __shared__ __align__(128) FwdWarpSmem SW[NWX * NWY];
    const int tile = blockIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    FwdWarpSmem& S = SW[warp];
    TileGeo geo;
    geo.init(prm, tile);
    const int p = prm.p;
    const int bx = warp % NWX, by = warp / NWX;
    const int lx = bx * 8 + (lane & 7), lyA = by * 8 + 2 * (lane >> 3);
    const bool vA = lx < geo.acols && lyA < geo.arows;
    const bool vB = lx < geo.acols && lyA + 1 < geo.arows;
    const int x = geo.ax + lx * p, yA = geo.ay + lyA * p, yB = yA + p;
    const float fx = (float)x + 0.5f, fyA = (float)yA + 0.5f, fyB = (float)yB + 0.5f;
    const uint2 range = prm.ranges[tile];
    const int count = (int)(range.y - range.x);
    const int nch = (count + 31) >> 5;
    const uint32_t rawbase = smem_addr(S.raw), recbase = smem_addr(S.rec) + kRec;  // spare slot at -1
    const uint32_t myraw = rawbase + lane * (uint32_t)sizeof(Prepared);
    // chunk c's gathers: lane copies its entry's record into raw[c & 1] (nothing past the list)
    auto issue = [&](int c, uint32_t item) {
        const uint32_t nb = c * 32 + lane < count ? 16u : 0u;
        const char* src = reinterpret_cast<const char*>(prm.prep + item);
        const uint32_t dst = myraw + (uint32_t)(c & 1) * (32u * sizeof(Prepared));
#pragma unroll
        for (int q = 0; q < 4; ++q) cp_async16(dst + 16 * q, src + 16 * q, nb);
        cp_async_commit_();
    };

    float2 T = make_float2(1.0f, 1.0f);
    float2 C0 = make_float2(0.f, 0.f), C1 = C0, C2 = C0;
    uint32_t lastA = 0, lastB = 0, ops = 0;
    bool doneA = !vA, doneB = !vB;
    bool warp_done = __all_sync(kFull, doneA && doneB);
    uint32_t item = 0;
    if (lane < 3) sts_f4(recbase - kRec + 16 * lane, make_float4(0.f, 0.f, 0.f, 0.f));  // spare slot
    if (!warp_done && nch > 0) {
        issue(0, lane < count ? prm.items[range.x + lane] : 0u);
        item = 32 + lane < count ? prm.items[range.x + 32 + lane] : 0u;
    }
    for (int c = 0; c < nch && !warp_done; ++c) {
        if (c + 1 < nch) {
            issue(c + 1, item);
            const int j = (c + 2) * 32 + lane;
            item = j < count ? prm.items[range.x + j] : 0u;
            cp_async_wait_<1>();
        } else {
            cp_async_wait_<0>();
        }
        const int n = min(32, count - c * 32);
        const uint32_t dst = recbase + lane * kRec;
        if (lane < n) {
            const uint32_t src = myraw + (uint32_t)(c & 1) * (32u * sizeof(Prepared));
            const float4 a = lds_f4(src), b = lds_f4(src + 16), cc = lds_f4(src + 32);
            const uint32_t mask = box_mask(a.x, b.z, geo.ax, p, geo.acols) |
                                  (box_mask(a.y, b.w, geo.ay, p, geo.arows) << 16);
            sts_f4(dst, make_float4(a.x, a.y, __fmul_rn(a.z, kNegHalfLog2e), __fmul_rn(a.w * 2.0f, kNegHalfLog2e)));
            sts_f4(dst + 16, make_float4(__fmul_rn(b.x, kNegHalfLog2e), b.y, cc.x, cc.y));
            sts_f4(dst + 32, make_float4(cc.z, __uint_as_float(mask), 0.f, 0.f));
        }
        __syncwarp();
        warp_done = walk_chunk(recbase, n, (uint32_t)(c * 32 + 1), bx, by, fx, fyA, fyB, T, C0, C1, C2, lastA, lastB,
                               ops, doneA, doneB);
    }
    cp_async_wait_<0>();  // copies still in flight must land before the CTA exits

    float lsum = 0.f;
    unsigned long long ev = 0;
    finish_pixel(prm, vA, x, yA, T.x, C0.x, C1.x, C2.x, lastA, doneA, count, ev, lsum);
    finish_pixel(prm, vB, x, yB, T.y, C0.y, C1.y, C2.y, lastB, doneB, count, ev, lsum);
    unsigned long long o = ops;
#pragma unroll
    for (int sft = 16; sft > 0; sft >>= 1) {
        o += __shfl_xor_sync(kFull, o, sft);
        ev += __shfl_xor_sync(kFull, ev, sft);
        lsum += __shfl_xor_sync(kFull, lsum, sft);
    }
    if (NWX * NWY == 1) {
        if (lane == 0) {
            if (o) atomicAdd(&prm.counters[1], o);
            if (ev) atomicAdd(&prm.counters[2], ev);
            if (prm.block_loss) prm.block_loss[tile] = lsum;
        }
        return;
    }
    __shared__ unsigned long long s_red[2][NWX * NWY];
    __shared__ float s_loss[NWX * NWY];
    if (lane == 0) {
        s_red[0][warp] = o;
        s_red[1][warp] = ev;
        s_loss[warp] = lsum;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long to = 0, te = 0;
        float tl = 0.f;
        for (int w = 0; w < NWX * NWY; ++w) {
            to += s_red[0][w];
            te += s_red[1][w];
            tl += s_loss[w];
        }
        if (to) atomicAdd(&prm.counters[1], to);
        if (te) atomicAdd(&prm.counters[2], te);
        if (prm.block_loss) prm.block_loss[tile] = tl;
    }
}

// ------------------------------------------------------------------------------ backward
// partial slot of (splat, tile): the splat's first slot (d.z = exclusive scan of tiles touched,
// in rank order) + the tile's row-major index inside the splat's tile rectangle
__device__ __forceinline__ uint32_t pair_slot(const Prepared& P, int tx, int ty) {
    const uint4 d = P.d;
    const int tx0 = d.x & 0xffff, tx1 = d.x >> 16, ty0 = d.y & 0xffff;
    return d.z + (uint32_t)((ty - ty0) * (tx1 - tx0 + 1) + (tx - tx0));
}

constexpr int kSubRows = 16;  // union rows per phase-1 / phase-2 round

#ifdef TGSX_BWD_STATS
// debug build only (A/B experiments): [0] group-chunks with work, [1] padded rows, [2] blended
// (splat, pixel) pairs, [3] U0 + U1, [4] phase-2 rounds, [5] chunks
__device__ unsigned long long g_bwd_stats[16];
#endif

// Per-warp shared memory of the backward. Pixel layout of an 8x8 group: lane l owns the two
// vertically adjacent pixels (col l&7, rows 2(l>>3), 2(l>>3)+1) = pixel slots 2l (A), 2l+1 (B).
// Record rows hold the 64 pixel slots as 16 chunks of 16 B; chunk c of row r sits at physical
// chunk c ^ (r & 3) (XOR swizzle: phase-1 row writes and the phase-2 row-per-lane-pair reads
// are both bank-conflict-free without padding).
template <int NG>
struct BwdWarpSmem {
    float rec_u[kSubRows * 64];  // phase-1 records u = dL/dsigma * G   [row][slot]
    float rec_w[kSubRows * 64];  //                  w = blend weight
    float4 st[NG][32];           // per lane (T_A, g.S_A, T_B, g.S_B) carried across chunks
    float lg[2][4][64];          // (last, dL/dC r, g, b) per slot of the current / next group,
                                 // filled by cp.async one group ahead
    unsigned char rec[32 * kRec];
    uint8_t klist[2][48];        // per half (lanes 0-15 / 16-31): union splats in visiting order,
                                 // padded to the longer half with a splat outside the union
};

// 4-byte global -> shared async copy (zero-fill when src_bytes == 0)
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, uint32_t src_bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(dst), "l"(src), "r"(src_bytes)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

__device__ __forceinline__ float2 neg2(float2 v) { return make_float2(-v.x, -v.y); }

// Phase-2 sums of one record row over half of an 8x8 group (lane half h: pixel rows 4h..4h+3),
// u / w row at rowp (byte address of the row's first chunk), dL/dC planar at gbase:
// acc += (sum u, sum u xi, sum u eta, sum u xi^2, sum u xi eta, sum u eta^2, sum w g0..g2),
// xi / eta = pixel offsets from the group centre (3.5, 3.5). Step s reads logical chunk
// 8h + (s ^ 4h) (row pair 2h + ((s>>2) ^ h), columns 2(s&3), 2(s&3)+1); a chunk holds
// (col c, row y), (c, y+1), (c+1, y), (c+1, y+1). Separable: per row pair accumulate packed
// (rows y, y+1) R = sum u, X = sum xi u, Q = sum xi^2 u over the columns, then fold with eta.
__device__ __forceinline__ void half_sums(uint32_t rowp, int ukey, uint32_t gbase, int h,
                                          float (&acc)[9]) {
    float2 c0p = make_float2(0.f, 0.f), c1p = c0p, c2p = c0p;
#pragma unroll
    for (int rp = 0; rp < 2; ++rp) {
        float2 Rp = make_float2(0.f, 0.f), Xp = Rp, Qp = Rp;
#pragma unroll
        for (int cs = 0; cs < 4; ++cs) {
            const int s = 4 * rp + cs;
            const uint32_t ua = rowp + (uint32_t)((s ^ ukey) << 4);
            const float4 u4 = lds_f4(ua);
            const float4 w4 = lds_f4(ua + kSubRows * 64 * 4);
            const uint32_t ga = gbase + (uint32_t)((s ^ (4 * h)) << 4);
            const float4 g0 = lds_f4(ga);  // two distinct addresses per quarter warp (broadcast)
            const float4 g1 = lds_f4(ga + 256);
            const float4 g2 = lds_f4(ga + 512);
            const float xa = (float)(2 * cs) - 3.5f, xb = xa + 1.0f;
            const float2 uA = make_float2(u4.x, u4.y), uB = make_float2(u4.z, u4.w);
            Rp = __fadd2_rn(Rp, uA);
            Rp = __fadd2_rn(Rp, uB);
            Xp = __ffma2_rn(uA, make_float2(xa, xa), Xp);
            Xp = __ffma2_rn(uB, make_float2(xb, xb), Xp);
            Qp = __ffma2_rn(uA, make_float2(xa * xa, xa * xa), Qp);
            Qp = __ffma2_rn(uB, make_float2(xb * xb, xb * xb), Qp);
            const float2 wA = make_float2(w4.x, w4.y), wB = make_float2(w4.z, w4.w);
            c0p = __ffma2_rn(wA, make_float2(g0.x, g0.y), c0p);
            c0p = __ffma2_rn(wB, make_float2(g0.z, g0.w), c0p);
            c1p = __ffma2_rn(wA, make_float2(g1.x, g1.y), c1p);
            c1p = __ffma2_rn(wB, make_float2(g1.z, g1.w), c1p);
            c2p = __ffma2_rn(wA, make_float2(g2.x, g2.y), c2p);
            c2p = __ffma2_rn(wB, make_float2(g2.z, g2.w), c2p);
        }
        const float eta = (float)(4 * h + 2 * (rp ^ h)) - 3.5f;  // row y; Rp.y is row y + 1
        const float R = Rp.x + Rp.y, X = Xp.x + Xp.y;
        acc[0] += R;
        acc[1] += X;
        acc[2] += __fmaf_rn(R, eta, Rp.y);
        acc[3] += Qp.x + Qp.y;
        acc[4] += __fmaf_rn(X, eta, Xp.y);
        acc[5] += __fmaf_rn(Rp.x, eta * eta, Rp.y * ((eta + 1.f) * (eta + 1.f)));
    }
    acc[6] += c0p.x + c0p.y;
    acc[7] += c1p.x + c1p.y;
    acc[8] += c2p.x + c2p.y;
}

// CTA = true: the tile's NG groups are walked by NG warps of one CTA in parallel (warp w takes
// group w; each warp stages the chunk itself; the per-splat moment sums of the NG groups are added
// in group order through `red` [2][NG][32][10] floats before one warp writes the pair slots) —
// for views with too few tiles to fill the GPU with one warp per tile (C1: 256 tiles).
template <int NGX, int NGY, bool CTA = false>
__device__ __forceinline__ void backward_tile(const BlendParams& prm, BwdWarpSmem<NGX * NGY>& S,
                                              int tile, int lane, float* red = nullptr) {
    constexpr int NG = NGX * NGY;
    const int gsel = CTA ? (int)(threadIdx.x >> 5) : 0;
    TileGeo geo;
    geo.init(prm, tile);
    const int p = prm.p;
    const uint2 range = prm.ranges[tile];
    const int count = (int)(range.y - range.x);
    const uint32_t rbase = smem_addr(S.rec);
    const uint32_t ubase = smem_addr(S.rec_u);
    const uint32_t wbase = smem_addr(S.rec_w);
    const int cxl = lane & 7, ryl = 2 * (lane >> 3);  // lane's column / first row in a group

    uint32_t maxlast = 0;
#pragma unroll 1
    for (int g = CTA ? gsel : 0; g < (CTA ? gsel + 1 : NG); ++g) {
        const int lx = (g % NGX) * 8 + cxl, lyA = (g / NGX) * 8 + ryl;
        float4 st = make_float4(1.f, 0.f, 1.f, 0.f);
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int ly = lyA + b;
            if (lx < geo.acols && ly < geo.arows) {
                const int x = geo.ax + lx * p, y = geo.ay + ly * p;
                const int r = ((y - prm.oy) / p) * prm.cols + (x - prm.ox) / p;
                const float T = prm.T[r];
                // g . S with S = background * trans_final (rasterizer.cpp:267)
                const float gS = prm.dLdC[3 * r] * (prm.bg0 * T) + prm.dLdC[3 * r + 1] * (prm.bg1 * T) +
                                 prm.dLdC[3 * r + 2] * (prm.bg2 * T);
                if (b == 0) st.x = T, st.y = gS;
                else st.z = T, st.w = gS;
                maxlast = max(maxlast, prm.last[r]);
            }
        }
        S.st[g][lane] = st;
    }
    maxlast = __reduce_max_sync(kFull, maxlast);
    if (CTA) {  // every warp walks the same chunks: the tile-wide last contributor
        __shared__ uint32_t s_max[NG];
        if (lane == 0) s_max[gsel] = maxlast;
        __syncthreads();
#pragma unroll
        for (int w = 0; w < NG; ++w) maxlast = max(maxlast, s_max[w]);
    }
    // moments about the tile's active-pixel centre (pixel-centre coordinates): active pixel
    // (cx, cy) sits at (ctr_x + (cx - hx) p, ctr_y + (cy - hy) p)
    constexpr float hx = 0.5f * (NGX * 8 - 1), hy = 0.5f * (NGY * 8 - 1);
    const float fp = (float)p;
    const float ctr_x = (float)geo.ax + 0.5f + hx * fp;
    const float ctr_y = (float)geo.ay + 0.5f + hy * fp;
    const float fxl = (float)(geo.ax + cxl * p) + 0.5f;  // group (0,0) pixel centres (A, B)
    const float fyl = (float)(geo.ay + ryl * p) + 0.5f;

    // list entries past every pixel's last contributor: zero partials
    for (int j = (int)maxlast + lane; j < (CTA && gsel ? 0 : count); j += 32) {
        const uint32_t slot = pair_slot(prm.prep[prm.items[range.x + j]], geo.tx, geo.ty);
        prm.partial.a[slot] = make_float4(0.f, 0.f, 0.f, 0.f);
        prm.partial.b[slot] = make_float4(0.f, 0.f, 0.f, 0.f);
        prm.partial.c[slot] = make_float2(0.f, 0.f);
    }

    // per-group (last, dL/dC) prefetch, one group ahead, cyclic over the groups of every chunk
    const uint32_t lgbase = smem_addr(S.lg);
    // dense rank of active pixel (lx, ly) = rank0 + ly * cols + lx (ax, ay are active pixels)
    const int rank0 = ((geo.ay - prm.oy) / p) * prm.cols + (geo.ax - prm.ox) / p;
    // Slot s of a plane holds pixel (lane s >> 1, A/B = s & 1); this lane fetches slots `lane` and
    // 32 + lane (contiguous 4-B destinations: no bank conflicts), i.e. the pixels of lanes
    // lane >> 1 and 16 + (lane >> 1), row offset lane & 1.
    const int fcol = (lane >> 1) & 7, frow = 2 * (lane >> 4) + (lane & 1);  // slot `lane`
    auto prefetch = [&](int g, int buf) {
        const int lx = (g % NGX) * 8 + fcol, ly0 = (g / NGX) * 8 + frow, ly1 = ly0 + 4;  // slot 32+lane: 4 rows down
        const bool v0 = lx < geo.acols && ly0 < geo.arows, v1 = lx < geo.acols && ly1 < geo.arows;
        const int r0 = v0 ? rank0 + ly0 * prm.cols + lx : 0;
        const int r1 = v1 ? rank0 + ly1 * prm.cols + lx : 0;
        const uint32_t n0 = v0 ? 4u : 0u, n1 = v1 ? 4u : 0u;
        const uint32_t d = lgbase + 1024u * (uint32_t)buf + 4u * (uint32_t)lane;
        cp_async4(d, prm.last + r0, n0);
        cp_async4(d + 128, prm.last + r1, n1);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            cp_async4(d + 256 * (c + 1), prm.dLdC + 3 * r0 + c, n0);
            cp_async4(d + 256 * (c + 1) + 128, prm.dLdC + 3 * r1 + c, n1);
        }
        cp_async_commit();
    };
    int buf = 0;
    prefetch(gsel, 0);  // (CTA: the warp's only group, loaded once for the whole tile)

    // phase-1 record offsets of this lane's slot pair in a row r: chunk (lane >> 1) ^ (r & 3)
    const uint32_t soff0 = (uint32_t)((lane >> 1) << 4) + (uint32_t)((lane & 1) << 3);
    // phase-2 role: lane = 2 i + h reads row i, half h
    const int p2row = lane >> 1, p2h = lane & 1;
    const int ukey = (4 * p2h) | (p2row & 3);

    const int nch = ((int)maxlast + 31) / 32;
    for (int ch = nch - 1; ch >= 0; --ch) {
        const int c0 = ch * 32;
        const int j = c0 + lane;
        const bool jvalid = j < (int)maxlast;
        __syncwarp();
        // the next (earlier) chunk's list entry, loaded alongside this chunk's: its prepared
        // record is prefetched into L2 below, hiding the DRAM latency of the next staging
        const uint32_t nxt = ch > 0 ? prm.items[range.x + j - 32] : 0u;
        const uint32_t myrec = rbase + lane * kRec;  // lane j's splat: mask, slot re-read from here
        if (jvalid) {
            const Prepared& P = prm.prep[prm.items[range.x + j]];
            stage_splat(P, geo, p, pair_slot(P, geo.tx, geo.ty), myrec);
        } else {  // empty mask; a zero record (finite) for filler rows that land here
            sts_f4(myrec, make_float4(0.f, 0.f, 0.f, 0.f));
            sts_f4(myrec + 16, make_float4(0.f, 0.f, 0.f, 0.f));
            sts_f4(myrec + 32, make_float4(0.f, 0.f, 0.f, 0.f));
        }
        if (ch > 0) asm volatile("prefetch.global.L2 [%0];" ::"l"(prm.prep + nxt));
        __syncwarp();
        // masks transposed: lane c < 16 holds the chunk's splats passing active column c, lane
        // 16 + r those passing row r (rasterizer.cpp:116-118); a pixel's pass set is column & row
        const uint32_t bits = transpose32(__float_as_uint(lds_f1(myrec + 36)));
#ifdef TGSX_BWD_STATS
        if (lane == 0) atomicAdd(&g_bwd_stats[5], 1ull);
#endif
        float m0 = 0.f, mx1 = 0.f, my1 = 0.f, mxx = 0.f, mxy = 0.f, myy = 0.f;
        float q0 = 0.f, q1 = 0.f, q2 = 0.f;
        uint32_t vism = 0;
#pragma unroll 1
        for (int gi = 0; gi < (CTA ? 1 : NG); ++gi) {
            const int g = CTA ? gsel : gi;
            const int gx = g % NGX, gy = g / NGX;
            const int cur = CTA ? 0 : buf;
            __syncwarp();  // the previous group's phase 2 is done with the rows and lg[buf]
            if (!CTA) {
                buf ^= 1;
                prefetch(g + 1 < NG ? g + 1 : 0, buf);
            }
            // pass sets of the lane's pixels A / B in this group
            const uint32_t X = __shfl_sync(kFull, bits, gx * 8 + cxl);
            uint32_t colA = X & __shfl_sync(kFull, bits, 16 + gy * 8 + ryl);
            uint32_t colB = X & __shfl_sync(kFull, bits, 17 + gy * 8 + ryl);
#ifdef TGSX_BWD_STATS
            const uint32_t boxA = colA, boxB = colB;
#endif
            if (CTA) cp_async_wait<0>();
            else cp_async_wait<1>();
            __syncwarp();
            const uint32_t lgc = lgbase + 1024u * (uint32_t)cur + 8u * (uint32_t)lane;
            const float2 lastp = lds_f2(lgc);
            // only splats before each pixel's last contributor were blended
            const int spA = (int)__float_as_uint(lastp.x) - c0, spB = (int)__float_as_uint(lastp.y) - c0;
            colA &= spA <= 0 ? 0u : (spA >= 32 ? kFull : ((1u << spA) - 1u));
            colB &= spB <= 0 ? 0u : (spB >= 32 ? kFull : ((1u << spB) - 1u));
            // Each half of the group (8x4 pixels, lanes 0-15 / 16-31) visits the union of its
            // pixels' walked splats back to front, both halves in lockstep (row r = the r-th
            // splat of each half's union): record reads are broadcasts per half, and every row
            // is DENSE (pixels that do not blend the row's splat store 0), so phase 2 reads only
            // max(U0, U1) rows. The shorter half runs on a splat outside its union (G = 0).
            const uint32_t cu = colA | colB;
            const uint32_t un0 = __reduce_or_sync(kFull, lane < 16 ? cu : 0u);
            const uint32_t un1 = __reduce_or_sync(kFull, lane < 16 ? 0u : cu);
            if (!(un0 | un1)) continue;
            const int U0 = __popc(un0), U1 = __popc(un1);
            // rows are visited in pairs: an odd count is padded with a filler row (each half then
            // has a splat outside its union, as U <= 31)
            const int U = (max(U0, U1) + 1) & ~1;
#ifdef TGSX_BWD_STATS
            {
                const unsigned nb = __reduce_add_sync(kFull, (unsigned)(__popc(colA) + __popc(colB)));
                if (lane == 0) {
                    atomicAdd(&g_bwd_stats[0], 1ull);
                    atomicAdd(&g_bwd_stats[1], (unsigned long long)U);
                    atomicAdd(&g_bwd_stats[2], (unsigned long long)nb);
                    atomicAdd(&g_bwd_stats[3], (unsigned long long)(U0 + U1));
                    atomicAdd(&g_bwd_stats[4], (unsigned long long)((U + kSubRows - 1) / kSubRows));
                }
                // [6] box-only blends (termination ignored; invalid pixels have T = 1 and are
                // never limited, so count only lanes whose pixels are valid via lastp != 0)
                const unsigned nbox = __reduce_add_sync(kFull, (unsigned)(__popc(boxA) + __popc(boxB)));
                // [7] rows if 4x4 quarters (lanes {0-3, 8-11} etc.) ran in lockstep
                uint32_t q = cu;
                q |= __shfl_xor_sync(kFull, q, 1);
                q |= __shfl_xor_sync(kFull, q, 2);
                q |= __shfl_xor_sync(kFull, q, 8);
                const unsigned qmax = __reduce_max_sync(kFull, (unsigned)__popc(q));
                const unsigned lmax = __reduce_max_sync(kFull, (unsigned)__popc(cu));
                const unsigned lsum = __reduce_add_sync(kFull, (unsigned)__popc(cu));
                if (lane == 0) {
                    atomicAdd(&g_bwd_stats[8], (unsigned long long)lmax);
                    atomicAdd(&g_bwd_stats[9], (unsigned long long)lsum);
                    atomicAdd(&g_bwd_stats[6], (unsigned long long)nbox);
                    atomicAdd(&g_bwd_stats[7], (unsigned long long)qmax);
                }
            }
#endif
            const float2 g0p = lds_f2(lgc + 256), g1p = lds_f2(lgc + 512), g2p = lds_f2(lgc + 768);
            const float4 st = S.st[g][lane];
            float2 T = make_float2(st.x, st.z), gS = make_float2(st.y, st.w);
            const float fx = fxl + (float)(gx * 8 * p), fyA = fyl + (float)(gy * 8 * p), fyB = fyA + fp;
            uint32_t visb = 0;
            // union splats in visiting order: row r <- splat k_r (lane j owns row popc(un >> j+1))
            const int row0 = __popc(un0 & (0xfffffffeu << lane)), row1 = __popc(un1 & (0xfffffffeu << lane));
            const bool in0 = (un0 >> lane) & 1u, in1 = (un1 >> lane) & 1u;
            if (in0) S.klist[0][row0] = (uint8_t)lane;
            if (in1) S.klist[1][row1] = (uint8_t)lane;
            if (U0 + lane < U) S.klist[0][U0 + lane] = (uint8_t)(__ffs(~un0) - 1);
            if (U1 + lane < U) S.klist[1][U1 + lane] = (uint8_t)(__ffs(~un1) - 1);
            __syncwarp();
            const uint8_t* kl = S.klist[lane >> 4];
            const float dxg = (float)(gx * 8) + 3.5f - hx, dyg = (float)(gy * 8) + 3.5f - hy;
            const uint32_t gb = lgbase + 1024u * (uint32_t)cur + 256u + 128u * (uint32_t)p2h;
            for (int rb = 0; rb < U; rb += kSubRows) {
                const int re = min(U, rb + kSubRows);
                // phase 1: per pixel pair, back to front, two union splats per iteration (k1 > k2):
                // Gaussians / reciprocals are independent (ILP); only the T and g.S recursions are
                // serial. A pixel that does not blend a splat computes on it with G = 0
                // (sigma = 0, 1 / (1 - sigma) = 1: T, g.S pass through; records u = w = 0).
                int k1n = kl[rb], k2n = kl[rb + 1];  // next pair, one iteration ahead
                uint32_t rowb = 0;  // byte offset of row (r - rb)
#ifndef TGSX_BWD_UNROLL
#define TGSX_BWD_UNROLL 2
#endif
#if TGSX_BWD_UNROLL == 1
#pragma unroll 1
#else
#pragma unroll 2
#endif
                for (int r = rb; r < re; r += 2) {
                    const int k1 = k1n, k2 = k2n;
                    k1n = kl[r + 2];
                    k2n = kl[r + 3];
                    const bool hA1 = (colA >> k1) & 1u, hB1 = (colB >> k1) & 1u;
                    const bool hA2 = (colA >> k2) & 1u, hB2 = (colB >> k2) & 1u;
                    const uint32_t ad1 = rbase + k1 * kRec, ad2 = rbase + k2 * kRec;
                    const float4 a1 = lds_f4(ad1), a2 = lds_f4(ad2);
                    const float4 b1 = lds_f4(ad1 + 16), b2 = lds_f4(ad2 + 16);
                    const float cz1 = lds_f1(ad1 + 32), cz2 = lds_f1(ad2 + 32);
                    const float2 e1 = pair_quad(a1, b1.x, fx, fyA, fyB);
                    const float2 e2 = pair_quad(a2, b2.x, fx, fyA, fyB);
                    const float2 G1 = make_float2(hA1 ? fast_exp2(e1.x) : 0.f, hB1 ? fast_exp2(e1.y) : 0.f);
                    const float2 G2 = make_float2(hA2 ? fast_exp2(e2.x) : 0.f, hB2 ? fast_exp2(e2.y) : 0.f);
                    const float2 s1 = __fmul2_rn(make_float2(b1.y, b1.y), G1);
                    const float2 s2 = __fmul2_rn(make_float2(b2.y, b2.y), G2);
                    // 1 - sigma with one rounding, exactly as the scalar subtraction
                    const float2 o1 = __ffma2_rn(s1, make_float2(-1.f, -1.f), make_float2(1.f, 1.f));
                    const float2 o2 = __ffma2_rn(s2, make_float2(-1.f, -1.f), make_float2(1.f, 1.f));
                    const float2 ir1 = make_float2(fast_rcp(o1.x), fast_rcp(o1.y));  // inv_rest
                    const float2 ir2 = make_float2(fast_rcp(o2.x), fast_rcp(o2.y));
                    const float2 gc1 = __ffma2_rn(g2p, make_float2(cz1, cz1),
                                                  __ffma2_rn(g1p, make_float2(b1.w, b1.w),
                                                             __fmul2_rn(g0p, make_float2(b1.z, b1.z))));
                    const float2 gc2 = __ffma2_rn(g2p, make_float2(cz2, cz2),
                                                  __ffma2_rn(g1p, make_float2(b2.w, b2.w),
                                                             __fmul2_rn(g0p, make_float2(b2.z, b2.z))));
                    // g . dC/dsigma_i = T_i (g.c_i) - (g.S_i) / (1 - sigma_i)  (rasterizer.cpp:272-275)
                    const float2 T1 = __fmul2_rn(T, ir1);
                    const float2 w1 = __fmul2_rn(s1, T1);
                    const float2 ds1 = __ffma2_rn(T1, gc1, neg2(__fmul2_rn(gS, ir1)));
                    const float2 gS1 = __ffma2_rn(gc1, w1, gS);
                    const float2 T2 = __fmul2_rn(T1, ir2);
                    const float2 w2 = __fmul2_rn(s2, T2);
                    const float2 ds2 = __ffma2_rn(T2, gc2, neg2(__fmul2_rn(gS1, ir2)));
                    T = T2;
                    gS = __ffma2_rn(gc2, w2, gS1);
                    const uint32_t o1b = rowb + (soff0 ^ (((uint32_t)(r - rb) & 3u) << 4));
                    sts_f2(ubase + o1b, __fmul2_rn(ds1, G1));
                    sts_f2(wbase + o1b, w1);
                    const uint32_t o2b = rowb + 256u + (soff0 ^ (((uint32_t)(r + 1 - rb) & 3u) << 4));
                    sts_f2(ubase + o2b, __fmul2_rn(ds2, G2));
                    sts_f2(wbase + o2b, w2);
                    visb |= (fmaxf(w1.x, w1.y) > kMinVisitW ? (1u << k1) : 0u) |
                            (fmaxf(w2.x, w2.y) > kMinVisitW ? (1u << k2) : 0u);
                    rowb += 512u;
                }
                __syncwarp();
                // phase 2: dense over each half's 32 pixels per record row; lane 2i + h takes
                // half h of row i (splat k^h_i)
                float acc[9] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                if (p2row < re - rb)
                    half_sums(ubase + 256u * (uint32_t)p2row + 128u * (uint32_t)p2h, ukey, gb, p2h, acc);
                // hand each half-row's sums to lane j = its splat (from up to two lanes)
                const bool m0h = in0 && row0 >= rb && row0 < re, m1h = in1 && row1 >= rb && row1 < re;
                const int src0 = m0h ? 2 * (row0 - rb) : 0, src1 = m1h ? 2 * (row1 - rb) + 1 : 1;
#ifndef TGSX_BWD_SMEM_HANDOFF
#define TGSX_BWD_SMEM_HANDOFF 1
#endif
#if TGSX_BWD_SMEM_HANDOFF
                // through the (now read) rows of rec_u: 3 stores + up to 6 loads instead of 18
                // shuffles (lane l's sums at 48 l: conflict-free stores)
                __syncwarp();
                {
                    const uint32_t hb = ubase + 48u * (uint32_t)lane;
                    sts_f4(hb, make_float4(acc[0], acc[1], acc[2], acc[3]));
                    sts_f4(hb + 16, make_float4(acc[4], acc[5], acc[6], acc[7]));
                    sts_f1(hb + 32, acc[8]);
                }
                __syncwarp();
                if (m0h || m1h) {
                    float v0[9], v1[9];
#pragma unroll
                    for (int q = 0; q < 9; ++q) v0[q] = v1[q] = 0.f;
                    if (m0h) {
                        const uint32_t a = ubase + 48u * (uint32_t)src0;
                        const float4 x = lds_f4(a), y = lds_f4(a + 16);
                        v0[0] = x.x; v0[1] = x.y; v0[2] = x.z; v0[3] = x.w;
                        v0[4] = y.x; v0[5] = y.y; v0[6] = y.z; v0[7] = y.w;
                        v0[8] = lds_f1(a + 32);
                    }
                    if (m1h) {
                        const uint32_t a = ubase + 48u * (uint32_t)src1;
                        const float4 x = lds_f4(a), y = lds_f4(a + 16);
                        v1[0] = x.x; v1[1] = x.y; v1[2] = x.z; v1[3] = x.w;
                        v1[4] = y.x; v1[5] = y.y; v1[6] = y.z; v1[7] = y.w;
                        v1[8] = lds_f1(a + 32);
                    }
#pragma unroll
                    for (int q = 0; q < 9; ++q) acc[q] = v0[q] + v1[q];
                }
#else
#pragma unroll
                for (int q = 0; q < 9; ++q) {
                    const float v0 = __shfl_sync(kFull, acc[q], src0), v1 = __shfl_sync(kFull, acc[q], src1);
                    acc[q] = (m0h ? v0 : 0.f) + (m1h ? v1 : 0.f);
                }
#endif
                if (m0h || m1h) {
                    const float a0 = acc[0], ax1 = acc[1], ay1 = acc[2];
                    m0 += a0;
                    mx1 += ax1 + dxg * a0;
                    my1 += ay1 + dyg * a0;
                    mxx += acc[3] + 2.f * dxg * ax1 + dxg * dxg * a0;
                    mxy += acc[4] + dyg * ax1 + dxg * ay1 + dxg * dyg * a0;
                    myy += acc[5] + 2.f * dyg * ay1 + dyg * dyg * a0;
                    q0 += acc[6];
                    q1 += acc[7];
                    q2 += acc[8];
                }
                __syncwarp();  // rows are rewritten by the next round
            }
            S.st[g][lane] = make_float4(T.x, gS.x, T.y, gS.y);
            vism |= __reduce_or_sync(kFull, visb);
        }
        if (CTA) {
            // group sums -> red[ch & 1][gsel][lane]; warp 0 adds them in group order
            float* rb = red + ((ch & 1) * NG + gsel) * 32 * 10 + lane * 10;
            rb[0] = m0; rb[1] = mx1; rb[2] = my1; rb[3] = mxx; rb[4] = mxy; rb[5] = myy;
            rb[6] = q0; rb[7] = q1; rb[8] = q2;
            rb[9] = __uint_as_float((vism >> lane) & 1u);
            __syncthreads();
            if (gsel != 0) continue;
            const float* r0p = red + (ch & 1) * NG * 32 * 10 + lane * 10;
            m0 = r0p[0]; mx1 = r0p[1]; my1 = r0p[2]; mxx = r0p[3]; mxy = r0p[4]; myy = r0p[5];
            q0 = r0p[6]; q1 = r0p[7]; q2 = r0p[8];
            uint32_t vb = __float_as_uint(r0p[9]);
#pragma unroll
            for (int w = 1; w < NG; ++w) {
                const float* rw = r0p + w * 32 * 10;
                m0 += rw[0]; mx1 += rw[1]; my1 += rw[2]; mxx += rw[3]; mxy += rw[4]; myy += rw[5];
                q0 += rw[6]; q1 += rw[7]; q2 += rw[8];
                vb |= __float_as_uint(rw[9]);
            }
            vism = vb << lane;
        }
        if (jvalid) {
            float4 r0 = make_float4(0.f, 0.f, 0.f, 0.f), r1 = r0;
            const uint32_t slot = __float_as_uint(lds_f1(myrec + 40));
            if (m0 != 0.f || mxx != 0.f || myy != 0.f || q0 != 0.f || q1 != 0.f || q2 != 0.f) {
                const float4 ja = lds_f4(myrec), jb = lds_f4(myrec + 16);
                constexpr float iK = 1.0f / kNegHalfLog2e;
                const float ia = ja.z * iK, ib = 0.5f * ja.w * iK, ic = jb.x * iK;
                const float al = jb.y;
                // moments about the splat mean: dx = p xi - mxb, dy = p eta - myb
                const float mxb = ja.x - ctr_x, myb = ja.y - ctr_y;
                const float sdx = fp * mx1 - mxb * m0;
                const float sdy = fp * my1 - myb * m0;
                const float sxx = fp * fp * mxx - 2.f * fp * mxb * mx1 + mxb * mxb * m0;
                const float sxy = fp * fp * mxy - fp * myb * mx1 - fp * mxb * my1 + mxb * myb * m0;
                const float syy = fp * fp * myy - 2.f * fp * myb * my1 + myb * myb * m0;
                // d_mean = alpha u (A delta); d_Sigma' = alpha/2 u (A delta)(A delta)^T
                const float ha = 0.5f * al;
                r0 = make_float4(al * (ia * sdx + ib * sdy), al * (ib * sdx + ic * sdy),
                                 ha * (ia * ia * sxx + 2.f * ia * ib * sxy + ib * ib * syy),
                                 ha * (ia * ib * sxx + (ia * ic + ib * ib) * sxy + ib * ic * syy));
                r1 = make_float4(ha * (ib * ib * sxx + 2.f * ib * ic * sxy + ic * ic * syy), m0, q0, q1);
            }
            prm.partial.a[slot] = r0;
            prm.partial.b[slot] = r1;
            prm.partial.c[slot] = make_float2(q2, ((vism >> lane) & 1u) ? 1.0f : 0.0f);
        }
    }
    cp_async_wait<0>();  // drain the last (unused) prefetch
}

// One warp per tile, tiles taken from a queue: a warp starts its next tile as soon as it has
// finished one, so no warp idles until its CTA siblings finish (per-tile work varies) and the
// tail of the launch is at most one tile.
template <int NGX, int NGY>
__global__ void __launch_bounds__(kWPB * 32, TGSX_BWD_MINB) backward_kernel(BlendParams prm) {
    constexpr int NG = NGX * NGY;
    static_assert(sizeof(BwdWarpSmem<NG>) % 16 == 0 && offsetof(BwdWarpSmem<NG>, st) % 16 == 0 &&
                      offsetof(BwdWarpSmem<NG>, lg) % 16 == 0 && offsetof(BwdWarpSmem<NG>, rec) % 16 == 0,
                  "float4 shared-memory reads need 16-byte alignment");
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto& S = reinterpret_cast<BwdWarpSmem<NG>*>(smem_raw)[warp];
    if (prm.fault) {
        const unsigned long long* c = prm.counters;
        const bool bad = *reinterpret_cast<const volatile unsigned*>(prm.fault) != 0u || c[0] != kErrNone ||
                         (c[3] & 0xffffffffull) > prm.guard_pairs || c[5] > prm.guard_list;
        if (bad) {
            if (threadIdx.x == 0) atomicOr(prm.fault, 1u);
            return;
        }
    }
    for (;;) {
        int tile = 0;
        if (lane == 0) tile = (int)atomicAdd(prm.tile_queue, 1u);
        tile = __shfl_sync(kFull, tile, 0);
        if (tile >= prm.tiles) break;
        backward_tile<NGX, NGY>(prm, S, tile, lane);
        __syncwarp();
    }
}

// One CTA per tile, one warp per group (backward_tile<..., true>): views with few tiles.
template <int NGX, int NGY>
__global__ void __launch_bounds__(NGX * NGY * 32) backward_cta_kernel(BlendParams prm) {
    constexpr int NG = NGX * NGY;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    auto& S = reinterpret_cast<BwdWarpSmem<NG>*>(smem_raw)[warp];
    float* red = reinterpret_cast<float*>(smem_raw + NG * sizeof(BwdWarpSmem<NG>));
    if (prm.fault) {
        const unsigned long long* c = prm.counters;
        const bool bad = *reinterpret_cast<const volatile unsigned*>(prm.fault) != 0u || c[0] != kErrNone ||
                         (c[3] & 0xffffffffull) > prm.guard_pairs || c[5] > prm.guard_list;
        if (bad) {
            if (threadIdx.x == 0) atomicOr(prm.fault, 1u);
            return;
        }
    }
    backward_tile<NGX, NGY, true>(prm, S, (int)blockIdx.x, lane, red);
}

BlendParams make_params(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items) {
    Workspace& ws = ctx->ws;
    BlendParams prm{};
    prm.ranges = ws.ranges.as<uint2>();
    prm.items = items;
    prm.prep = ws.prep.as<Prepared>();
    prm.tiles = ws.tiles_x * ws.tiles_y;
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
    prm.partial = Partials::at(ws.partial.p, ws.pair_cap);
    // counters slot 7 (u32): the backward's tile queue
    prm.tile_queue = reinterpret_cast<unsigned int*>(ws.counters.as<unsigned long long>() + 7);
    if (ctx->graph_capturing) {
        prm.fault = ctx->graph_fault;
        prm.guard_pairs = (uint32_t)std::min<int64_t>(std::min(ws.pair_cap, ctx->graph_guard_pairs), 0xffffffffll);
        prm.guard_list = (uint32_t)ctx->bin_sort_cap;
    }
    return prm;
}

template <int NGX, int NGY>
cudaError_t run_backward(tgsx_ctx* ctx, const BlendParams& prm) {
    const size_t smem = kWPB * sizeof(BwdWarpSmem<NGX * NGY>);
    int& resident = ctx->bwd_resident[NGX == 2 ? 0 : 1];  // CTAs resident at once (SMs x CTAs/SM)
    if (!resident) {
        // per context: the opt-in above 48 KB is a per-device attribute, set on the ctx's device
        int prev = 0;
        cudaError_t e = cudaGetDevice(&prev);
        if (e) return e;
        if (prev != ctx->device && (e = cudaSetDevice(ctx->device))) return e;
        e = cudaFuncSetAttribute(backward_kernel<NGX, NGY>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        int sms = 0, per_sm = 0;
        if (!e) e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        if (!e) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, backward_kernel<NGX, NGY>, kWPB * 32, smem);
        if (prev != ctx->device) cudaSetDevice(prev);
        if (e) return e;
        resident = std::max(1, sms * std::max(per_sm, 1));
    }
    if (NGX * NGY > 1 && (int64_t)prm.tiles * 2 < (int64_t)resident * kWPB) {
        // too few tiles to occupy every resident warp slot with one warp per tile: one CTA per tile,
        // its groups walked in parallel
        constexpr int NG = NGX * NGY;
        const size_t smem_cta = NG * sizeof(BwdWarpSmem<NG>) + 2 * NG * 32 * 10 * sizeof(float);
        int& cfg_done = ctx->bwd_resident[2];
        if (!cfg_done) {
            int prev = 0;
            cudaError_t e = cudaGetDevice(&prev);
            if (e) return e;
            if (prev != ctx->device && (e = cudaSetDevice(ctx->device))) return e;
            e = cudaFuncSetAttribute(backward_cta_kernel<NGX, NGY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_cta);
            if (prev != ctx->device) cudaSetDevice(prev);
            if (e) return e;
            cfg_done = 1;
        }
        backward_cta_kernel<NGX, NGY><<<(unsigned)prm.tiles, NG * 32, smem_cta, ctx->stream>>>(prm);
        return cudaGetLastError();
    }
    cudaError_t e = cudaMemsetAsync(prm.tile_queue, 0, sizeof(unsigned int), ctx->stream);
    if (e) return e;
    const unsigned grid =
        (unsigned)std::min<int64_t>((prm.tiles + kWPB - 1) / kWPB, (int64_t)resident);
    if (grid == 0) return cudaSuccess;
    backward_kernel<NGX, NGY><<<grid, kWPB * 32, smem, ctx->stream>>>(prm);
    return cudaGetLastError();
}

}  // namespace

#ifdef TGSX_BWD_STATS
extern "C" int tgsx_debug_bwd_stats(unsigned long long* out) {
    cudaDeviceSynchronize();
    cudaMemcpyFromSymbol(out, g_bwd_stats, sizeof(unsigned long long) * 16);
    unsigned long long z[16] = {};
    return (int)cudaMemcpyToSymbol(g_bwd_stats, z, sizeof(z));
}
#endif

cudaError_t launch_forward(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items,
                           bool fused_loss) {
    BlendParams prm = make_params(ctx, ra, items);
    if (fused_loss) {
        prm.target = ra.target;
        prm.target_rows = ra.target_rows;
        prm.loss_scale = ra.P > 0 ? (float)((double)ra.l1_weight / (3.0 * (double)ra.P)) : 0.f;
    } else {
        prm.target = nullptr;
        prm.block_loss = nullptr;
    }
    const unsigned tiles = (unsigned)prm.tiles;
    if (ra.p == 1) {
        // (one independent warp per 8x8 block, each staging the whole list, measured 0.46 ms at
        // C2 against 0.36 for the shared 256-record batches: the redundant staging dominates)
        forward_pairs_kernel<2, 2, 256><<<tiles, 128, 0, ctx->stream>>>(prm);
    } else {  // dilated: a tile's <= 8x8 active pixels are one warp's block
        forward_dilated_kernel<1, 1><<<tiles, 32, 0, ctx->stream>>>(prm);
    }
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_backward(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items) {
    BlendParams prm = make_params(ctx, ra, items);
    cudaError_t e;
    if (ra.p == 1) {
        e = run_backward<2, 2>(ctx, prm);
    } else {
        e = run_backward<1, 1>(ctx, prm);
    }
    ctx->launches++;
    return e;
}

}  // namespace tgsx
