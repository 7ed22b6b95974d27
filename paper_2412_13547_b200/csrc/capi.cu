// libtgsx C ABI (include/tgsx.h): contexts, device-resident models, and the host-side
// orchestration of the fit hot path. The product path is CUDA only: there is no CPU fallback —
// every entry point fails with TGSX_ECUDA if the device work cannot run.
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <utility>
#include <string>
#include <vector>

namespace tgsx {

// Buffers outgrown in the middle of a fit are not freed on the spot: cudaFree synchronises the
// whole device (the queued work of this and the next step drains) and unmapping can take tens of
// milliseconds, which showed up as 50-200 ms stalls of the first step after a densify event.
// They are retired here and freed at the next explicit synchronisation point (tgsx_synchronize,
// tgsx_destroy) — or at once when more than kGraveCap bytes are waiting.
static std::mutex g_grave_mu;
static std::vector<std::pair<int, void*>> g_grave;  // (device current at retirement, pointer)
static size_t g_grave_bytes = 0;
constexpr size_t kGraveCap = size_t(4) << 30;

static void drain_graveyard_locked() {
    int cur = 0;
    cudaGetDevice(&cur);
    for (const auto& q : g_grave) {
        if (q.first != cur) cudaSetDevice(q.first);
        cudaFree(q.second);
        if (q.first != cur) cudaSetDevice(cur);
    }
    g_grave.clear();
    g_grave_bytes = 0;
}

static void retire(void* q, size_t nb) {
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(g_grave_mu);
    g_grave.emplace_back(dev, q);
    g_grave_bytes += nb;
    if (g_grave_bytes > kGraveCap) drain_graveyard_locked();
}

void drain_graveyard() {
    std::lock_guard<std::mutex> lock(g_grave_mu);
    drain_graveyard_locked();
}

cudaError_t DevBuf::ensure(size_t need) {
    if (need <= bytes && p) return cudaSuccess;
    const bool growing = p != nullptr;
    if (p) retire(p, bytes);
    p = nullptr;
    bytes = 0;
    size_t nb = std::max<size_t>(need, 256);
    // headroom: K and P drift between iterations; a buffer that had to grow (a fit whose model
    // grows) gets more, so a growing fit reallocates rarely
    nb = growing ? nb + nb / 2 : nb + nb / 4;
    cudaError_t e = cudaMalloc(&p, nb);
    if (e) {
        p = nullptr;
        bytes = 0;
        return e;
    }
    bytes = nb;
    return cudaSuccess;
}

cudaError_t DevBuf::grow_keep(size_t need, size_t keep_bytes, cudaStream_t s) {
    if (need <= bytes && p) return cudaSuccess;
    void* np = nullptr;
    const size_t nb = std::max<size_t>(need, 256);
    cudaError_t e = cudaMalloc(&np, nb);
    if (e) return e;
    if (p && keep_bytes) {
        e = cudaMemcpyAsync(np, p, std::min(keep_bytes, bytes), cudaMemcpyDeviceToDevice, s);
        if (e) return e;
        cudaStreamSynchronize(s);
    }
    if (p) retire(p, bytes);
    p = np;
    bytes = nb;
    return cudaSuccess;
}

void DevBuf::release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
}

cudaEvent_t Profiler::get() {
    if (next >= pool.size()) {
        cudaEvent_t e;
        cudaEventCreate(&e);
        pool.push_back(e);
    }
    return pool[next++];
}

void Profiler::begin(int stage, cudaStream_t s, cudaEvent_t* out) {
    (void)stage;
    *out = get();
    cudaEventRecord(*out, s);
}

void Profiler::end(int stage, cudaStream_t s, cudaEvent_t start) {
    cudaEvent_t e = get();
    cudaEventRecord(e, s);
    pending.push_back({stage, {start, e}});
}

void Profiler::harvest() {
    for (auto& p : pending) {
        float ms_ = 0.f;
        if (cudaEventElapsedTime(&ms_, p.second.first, p.second.second) == cudaSuccess) {
            ms[p.first] += ms_;
            count[p.first] += 1;
        } else {
            cudaGetLastError();
        }
    }
    pending.clear();
    next = 0;
}

}  // namespace tgsx

using namespace tgsx;

namespace {

bool debug_checks() {
    static const bool on = [] {
        const char* e = std::getenv("TGSX_DEBUG_CHECKS");
        return e && e[0] == '1';
    }();
    return on;
}

int32_t fail(tgsx_ctx* ctx, int32_t code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

int32_t cuda_fail(tgsx_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, TGSX_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define CK(expr)                                              \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
    } while (0)

constexpr int kParamRows = 10;  // px py rot lsx lsy rop cr cg cb depth

int32_t check_pattern(tgsx_ctx* ctx, const tgsx_pattern* pat) {
    // DilationPattern constructor checks (dilation.hpp:18-22)
    if (!pat) return fail(ctx, TGSX_EINVAL, "pattern is null");
    if (pat->p < 1) return fail(ctx, TGSX_EINVAL, "dilation must be >= 1");
    if (pat->ox < 0 || pat->oy < 0 || pat->ox >= pat->p || pat->oy >= pat->p)
        return fail(ctx, TGSX_EINVAL, "dilation offsets must lie in [0, p)");
    if (pat->width < 1 || pat->height < 1)
        return fail(ctx, TGSX_EINVAL, "image dimensions must be >= 1");
    return TGSX_OK;
}

RenderArgs make_args(const tgsx_pattern* pat, const float bg[3], int lowpass_p) {
    RenderArgs ra{};
    ra.p = pat->p;
    ra.ox = pat->ox;
    ra.oy = pat->oy;
    ra.W = pat->width;
    ra.H = pat->height;
    ra.cols = pat->width > pat->ox ? (pat->width - pat->ox - 1) / pat->p + 1 : 0;
    ra.rows = pat->height > pat->oy ? (pat->height - pat->oy - 1) / pat->p + 1 : 0;
    ra.P = ra.cols * ra.rows;
    ra.bg[0] = bg ? bg[0] : 0.f;
    ra.bg[1] = bg ? bg[1] : 0.f;
    ra.bg[2] = bg ? bg[2] : 0.f;
    ra.lowpass_p = lowpass_p > 0 ? lowpass_p : pat->p;  // resolve_lowpass rasterizer.cpp:138
    ra.l1_weight = 1.0f;
    return ra;
}

// ---------------------------------------------------------------- model storage
cudaError_t model_reserve(tgsx_ctx* ctx, tgsx_model* m, int64_t cap) {
    if (cap <= m->cap) return cudaSuccess;
    cap = std::max<int64_t>(cap, 1);
    const int64_t n = m->n, oc = m->cap;
    cudaStream_t s = ctx->stream;
    auto regrow_rows = [&](DevBuf& b, int rows, size_t elt) -> cudaError_t {
        void* np = nullptr;
        cudaError_t e = cudaMalloc(&np, (size_t)rows * cap * elt);
        if (e) return e;
        if ((e = cudaMemsetAsync(np, 0, (size_t)rows * cap * elt, s))) return e;
        if (b.p && n > 0) {
            e = cudaMemcpy2DAsync(np, cap * elt, b.p, oc * elt, n * elt, rows, cudaMemcpyDeviceToDevice, s);
            if (e) return e;
        }
        cudaStreamSynchronize(s);
        b.release();
        b.p = np;
        b.bytes = (size_t)rows * cap * elt;
        return cudaSuccess;
    };
    cudaError_t e;
    if ((e = regrow_rows(m->params, kParamRows, 4))) return e;
    if ((e = regrow_rows(m->ids, 1, 8))) return e;
    if ((e = regrow_rows(m->pos_acc, 1, 4))) return e;
    if ((e = regrow_rows(m->col_acc, 1, 4))) return e;
    if ((e = regrow_rows(m->accum, 1, 4))) return e;
    if ((e = regrow_rows(m->visit, 1, 8))) return e;
    if ((e = regrow_rows(m->window, 1, 8))) return e;
    if ((e = regrow_rows(m->tau_v, 1, 8))) return e;
    if ((e = regrow_rows(m->m1, 9, 4))) return e;
    if ((e = regrow_rows(m->m2, 9, 4))) return e;
    if ((e = regrow_rows(m->step, 1, sizeof(StepRec)))) return e;  // AoS records
    if ((e = regrow_rows(m->screen, 10, 4))) return e;
    if ((e = regrow_rows(m->perm, 1, 4))) return e;
    if ((e = regrow_rows(m->rank_of, 1, 4))) return e;
    m->cap = cap;
    return cudaSuccess;
}

// ---------------------------------------------------------------- physical row order
// Between depth sorts the blend order is fixed (depth_key is not optimised), so the model rows
// are kept physically in blend (rank) order: preprocess, the partial merge and Adam then stream
// every per-Gaussian array contiguously instead of gathering through rank_of. Densify, download
// and the explicit-gradient APIs see the logical (creation) order; permute_model converts.
template <typename T>
__global__ void permute_rows_kernel(const T* __restrict__ src, T* __restrict__ dst, int64_t cap,
                                    int64_t n, int rows, const uint32_t* __restrict__ idx) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int64_t q = idx[p];
    for (int r = 0; r < rows; ++r) dst[(int64_t)r * cap + p] = src[(int64_t)r * cap + q];
}

// every row group: new[p] = old[idx[p]] (through the model's spare buffers, pointer swap)
cudaError_t permute_model(tgsx_ctx* ctx, tgsx_model* m, const uint32_t* idx) {
    ctx->bin_valid = false;
    const int64_t n = m->n, cap = m->cap;
    if (n == 0) return cudaSuccess;
    struct R { DevBuf* b; int rows; int elt; } rs[] = {
        {&m->params, kParamRows, 4}, {&m->ids, 1, 8}, {&m->pos_acc, 1, 4}, {&m->col_acc, 1, 4},
        {&m->accum, 1, 4}, {&m->visit, 1, 8}, {&m->window, 1, 8}, {&m->tau_v, 1, 8},
        {&m->m1, 9, 4}, {&m->m2, 9, 4}, {&m->step, 1, (int)sizeof(StepRec)}};
    static_assert(sizeof(rs) / sizeof(rs[0]) == sizeof(m->spare) / sizeof(m->spare[0]), "spares");
    cudaError_t e;
    for (int i = 0; i < 11; ++i) {
        const R& r = rs[i];
        DevBuf& sp = m->spare[i];
        const size_t bytes = (size_t)r.rows * cap * r.elt;
        if (sp.bytes < bytes) {
            if ((e = cudaStreamSynchronize(ctx->stream))) return e;
            sp.release();
            if ((e = cudaMalloc(&sp.p, bytes))) return e;
            sp.bytes = bytes;
        }
        const unsigned grid = (unsigned)((n + 255) / 256);
        if (r.elt == 4)
            permute_rows_kernel<uint32_t><<<grid, 256, 0, ctx->stream>>>(r.b->as<uint32_t>(), sp.as<uint32_t>(),
                                                                        cap, n, r.rows, idx);
        else if (r.elt == (int)sizeof(StepRec))
            permute_rows_kernel<StepRec><<<grid, 256, 0, ctx->stream>>>(r.b->as<StepRec>(), sp.as<StepRec>(),
                                                                       cap, n, 1, idx);
        else
            permute_rows_kernel<unsigned long long><<<grid, 256, 0, ctx->stream>>>(
                r.b->as<unsigned long long>(), sp.as<unsigned long long>(), cap, n, r.rows, idx);
        ctx->launches++;
        if ((e = cudaGetLastError())) return e;
        std::swap(r.b->p, sp.p);
        std::swap(r.b->bytes, sp.bytes);
    }
    return cudaSuccess;
}

}  // namespace

// Capacity growth (contents kept) with the spare row buffers sized alongside, so neither
// permutation nor prune compaction allocates later.
cudaError_t model_grow(tgsx_ctx* ctx, tgsx_model* m, int64_t cap) {
    if (cap <= m->cap) return cudaSuccess;
    cudaError_t e = model_reserve(ctx, m, cap);
    if (e) return e;
    const int rows[11] = {kParamRows, 1, 1, 1, 1, 1, 1, 1, 9, 9, 1};
    const int elt[11] = {4, 8, 4, 4, 4, 8, 8, 8, 4, 4, (int)sizeof(StepRec)};
    for (int i = 0; i < 11; ++i) {
        DevBuf& sp = m->spare[i];
        const size_t bytes = (size_t)rows[i] * m->cap * elt[i];
        if (sp.bytes >= bytes) continue;
        sp.release();
        if ((e = cudaMalloc(&sp.p, bytes))) return e;
        sp.bytes = bytes;
    }
    return cudaSuccess;
}

cudaError_t model_to_blend_order(tgsx_ctx* ctx, tgsx_model* m) {
    if (m->blend_phys || m->order_dirty) return cudaSuccess;
    cudaError_t e = permute_model(ctx, m, m->perm.as<uint32_t>());
    if (!e) m->blend_phys = true;
    return e;
}

cudaError_t model_to_logical_order(tgsx_ctx* ctx, tgsx_model* m) {
    if (!m->blend_phys) return cudaSuccess;
    cudaError_t e = permute_model(ctx, m, m->rank_of.as<uint32_t>());
    if (!e) m->blend_phys = false;
    return e;
}

namespace {

// ---------------------------------------------------------------- error word
int32_t check_kernel_error(tgsx_ctx* ctx, unsigned long long err) {
    if (err == kErrNone) return TGSX_OK;
    const uint32_t code = (uint32_t)(err & 3u);
    const unsigned long long rank = err >> 2;
    if (code == 1)
        return fail(ctx, TGSX_EINVAL,
                    "covariance_from_params: non-finite input (blend rank " + std::to_string(rank) + ")");
    return fail(ctx, TGSX_ERUNTIME,
                "covariance numerically degenerate (det <= 0) (blend rank " + std::to_string(rank) + ")");
}

// per-pair partial slots to reserve for K pairs of an n-splat model of capacity cap: scaled by
// cap / n (a fit growing its model towards a reserved budget keeps one allocation)
int64_t pair_capacity(int64_t K, int64_t n, int64_t cap) {
    const int64_t k = std::max<int64_t>(K, 1);
    if (n <= 0 || cap <= n) return k;
    return k + (int64_t)((double)k * (double)(cap - n) / (double)n);
}

cudaError_t reset_counters(tgsx_ctx* ctx) {
    Workspace& ws = ctx->ws;
    cudaError_t e = ws.counters.ensure(8 * sizeof(unsigned long long));
    if (e) return e;
    if ((e = cudaMemsetAsync(ws.counters.p, 0, 8 * sizeof(unsigned long long), ctx->stream))) return e;
    return cudaMemsetAsync(ws.counters.p, 0xff, sizeof(unsigned long long), ctx->stream);
}

// TGSX_BINNING=onesweep (process-wide) or tgsx_set_binning(ctx, 1): onesweep tile binning for
// 2-D views, the global depth sort + onesweep binning for 3-D views (the fallback paths)
bool force_onesweep(const tgsx_ctx* ctx) {
    static const bool v = [] {
        const char* s = std::getenv("TGSX_BINNING");
        return s && std::string(s) == "onesweep";
    }();
    return v || (ctx && ctx->binning_mode == 1);
}

// Per-tile sort of the slabs for lists up to `cap` entries (the template is chosen from it).
// Per-tile sort of the slabs for lists up to `cap` entries (the template is chosen from it). The
// records already carry their first pair slot (the preprocess runs the pair-offset scan fused).
int32_t slab_sort(tgsx_ctx* ctx, int tiles, uint64_t cap) {
    {
        StageTimer t(ctx, kStSort);
        CK(launch_seg_sort(ctx, ctx->ws.tile_slab.as<uint32_t>(), tiles, (int64_t)cap));
    }
    ctx->bin_sort_cap = cap <= 256 ? 256 : (cap <= 512 ? 512 : kSegCap);
    return TGSX_OK;
}

int32_t bin_onesweep(tgsx_ctx* ctx, tgsx_model* m, int64_t n, int W, int H, int64_t K, uint32_t** items,
                     uint32_t** sorted_keys);

// Sort (if dirty) -> preprocess (+ per-tile lengths) -> scans -> [read-back of K, errors, the
// longest list] -> per-tile sort of the slabs, or (a list longer than kSegCap, or
// TGSX_BINNING=onesweep) duplicate -> onesweep radix sort -> ranges.
// With `defer` (fused views) the read-back is not waited for here: the per-tile sort is
// launched speculatively for lists up to the previous binning's longest (x1.25), the caller
// queues its forward and then bin_settle() checks the counters (normally long complete),
// redoing the sort (or taking the onesweep path) when the guess was short.
// On return ws.K, ws.ranges and `items` (per-tile ranks in blend order) describe the lists.
int32_t bin_compute(tgsx_ctx* ctx, tgsx_model* m, int lowpass_p, int W, int H, uint32_t** items,
                    uint32_t** sorted_keys, bool defer = false) {
    Workspace& ws = ctx->ws;
    ws.have_forward = false;
    ctx->bin_pending = false;
    CK(reset_counters(ctx));
    if (m->order_dirty || !m->blend_phys) {
        StageTimer t(ctx, kStDepthSort);
        if (m->order_dirty) CK(launch_sort_depth(ctx, m));
        CK(model_to_blend_order(ctx, m));
    }
    unsigned long long* counters = ws.counters.as<unsigned long long>();
    uint32_t* d_total = reinterpret_cast<uint32_t*>(counters + 3);
    {
        // rows are in blend order here: the pair-offset scan is fused into the preprocess
        StageTimer t(ctx, kStPreprocess);
        CK(launch_preprocess(ctx, m, lowpass_p, W, H, d_total));
    }
    const int tiles = ws.tiles_x * ws.tiles_y;
    {
        StageTimer t(ctx, kStScan);
        CK(launch_slab_finalize(ctx, tiles));
    }
    CK(cudaMemcpyAsync(ws.h_scratch, counters, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    if (defer && !sorted_keys && !force_onesweep(ctx) && !debug_checks()) {
        if (!ctx->bin_event) CK(cudaEventCreateWithFlags(&ctx->bin_event, cudaEventDisableTiming));
        if (!ctx->graph_capturing) CK(cudaEventRecord(ctx->bin_event, ctx->stream));
        const uint64_t guess = std::min<uint64_t>(kSegCap, ctx->bin_max_hint + ctx->bin_max_hint / 4);
        int32_t rc = slab_sort(ctx, tiles, guess);
        if (rc) return rc;
        ctx->bin_pending = true;
        *items = ws.tile_slab.as<uint32_t>();
        if (sorted_keys) *sorted_keys = nullptr;
        return TGSX_OK;
    }
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->prof.enabled) ctx->prof.harvest();  // every event recorded so far has completed
    int32_t rc = check_kernel_error(ctx, ws.h_scratch[0]);
    if (rc) return rc;
    const int64_t K = (int64_t)(uint32_t)(ws.h_scratch[3] & 0xffffffffull);
    const uint64_t max_list = ws.h_scratch[5];
    ws.K = K;
    ctx->bin_max_hint = max_list;
    CK(ws.partial.ensure(pair_capacity(K, m->n, m->cap) * 40));
    ws.pair_cap = (int64_t)(ws.partial.bytes / 40);
    if (max_list <= (uint64_t)kSegCap && !force_onesweep(ctx)) {
        // slab binning: every tile's list was claimed by preprocess into its slab; sort each slab
        // back into blend order (one warp per tile)
        rc = slab_sort(ctx, tiles, max_list);
        if (rc) return rc;
        *items = ws.tile_slab.as<uint32_t>();
        if (sorted_keys) *sorted_keys = nullptr;
        return TGSX_OK;
    }
    return bin_onesweep(ctx, m, m->n, W, H, K, items, sorted_keys);
}

// Completes a deferred binning: waits for the counters, reports kernel errors, sizes the
// per-pair partials and, when the speculative per-tile sort was too short for the longest list
// (or a list overflowed its slab), redoes the lists; *redo tells the caller to rerun its forward.
int32_t bin_settle(tgsx_ctx* ctx, tgsx_model* m, int W, int H, uint32_t** items, bool* redo) {
    *redo = false;
    if (!ctx->bin_pending) return TGSX_OK;
    ctx->bin_pending = false;
    // a captured step never waits on the host: the backward checks the counters against the
    // capture-time capacities on the device (graph.cpp)
    if (ctx->graph_capturing) return TGSX_OK;
    Workspace& ws = ctx->ws;
    CK(cudaEventSynchronize(ctx->bin_event));
    int32_t rc = check_kernel_error(ctx, ws.h_scratch[0]);
    if (rc) {
        ctx->bin_valid = false;
        return rc;
    }
    const int64_t K = (int64_t)(uint32_t)(ws.h_scratch[3] & 0xffffffffull);
    const uint64_t max_list = ws.h_scratch[5];
    ws.K = K;
    ctx->bin_max_hint = max_list;
    CK(ws.partial.ensure(pair_capacity(K, m->n, m->cap) * 40));
    ws.pair_cap = (int64_t)(ws.partial.bytes / 40);
    if (max_list <= (uint64_t)ctx->bin_sort_cap) return TGSX_OK;
    *redo = true;
    if (max_list <= (uint64_t)kSegCap) {
        rc = slab_sort(ctx, ws.tiles_x * ws.tiles_y, max_list);
        if (rc) return rc;
        *items = ws.tile_slab.as<uint32_t>();
    } else {
        rc = bin_onesweep(ctx, m, m->n, W, H, K, items, nullptr);
        if (rc) return rc;
    }
    if (ctx->bin_valid) ctx->bin_items = *items;
    return TGSX_OK;
}

// Onesweep path (a list longer than the slab, or TGSX_BINNING=onesweep): duplicate keys,
// radix sort by tile (stable: blend order inside a tile), ranges.
// m may be null (3-D front end): the debug checks of the blend permutation are then skipped.
int32_t bin_onesweep(tgsx_ctx* ctx, tgsx_model* m, int64_t n_splats, int W, int H, int64_t K, uint32_t** items,
                     uint32_t** sorted_keys) {
    Workspace& ws = ctx->ws;
    const int tiles = ws.tiles_x * ws.tiles_y;
    for (int i = 0; i < 2; ++i) CK(ws.vals[i].ensure(std::max<int64_t>(K, 1) * 4));
    const int key_bits = key_bits_for(tiles);
    const int passes = (key_bits + 7) / 8;
    for (int i = 0; i < 2; ++i) CK(ws.keys[i].ensure(std::max<int64_t>(K, 1) * 4));
    // sized once here: duplicate writes the digit histograms at its head and sort_pairs must
    // not reallocate it afterwards
    CK(ws.sort_tmp.ensure(sort_scratch_bytes(K, key_bits)));
    {
        StageTimer t(ctx, kStDuplicate);
        CK(launch_duplicate(ctx, n_splats, key_bits));
    }
    const bool dbg = debug_checks() && m;
    if (dbg) {
        // host validation of every binning stage (TGSX_DEBUG_CHECKS=1)
        const int64_t n = m->n;
        std::vector<uint32_t> perm(n), rank_of(n), touched(n), off(n), keys(K), hist(4 * 256);
        CK(cudaStreamSynchronize(ctx->stream));
        if (n) {
            CK(cudaMemcpy(perm.data(), m->perm.p, n * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(rank_of.data(), m->rank_of.p, n * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(touched.data(), ws.touched.p, n * 4, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(off.data(), ws.pair_off.p, n * 4, cudaMemcpyDeviceToHost));
        }
        if (K) CK(cudaMemcpy(keys.data(), ws.keys[0].p, K * 4, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(hist.data(), ws.sort_tmp.p, 4 * 256 * 4, cudaMemcpyDeviceToHost));
        std::vector<char> seen(n, 0);
        for (int64_t r = 0; r < n; ++r) {
            if (perm[r] >= n || seen[perm[r]]) return fail(ctx, TGSX_ESTATE, "debug: perm not a permutation");
            seen[perm[r]] = 1;
            if (rank_of[perm[r]] != r) return fail(ctx, TGSX_ESTATE, "debug: rank_of != perm^-1");
        }
        uint64_t run = 0;
        for (int64_t r = 0; r < n; ++r) {
            if (off[r] != run)
                return fail(ctx, TGSX_ESTATE, "debug: scan wrong at rank " + std::to_string(r) + " of " +
                                                  std::to_string(n) + " got " + std::to_string(off[r]) +
                                                  " want " + std::to_string(run));
            run += touched[r];
        }
        if (run != (uint64_t)K) return fail(ctx, TGSX_ESTATE, "debug: scan total wrong");
        std::vector<uint32_t> h2(4 * 256, 0);
        for (int64_t s = 0; s < K; ++s) {
            if (keys[s] >= (uint32_t)tiles)
                return fail(ctx, TGSX_ESTATE, "debug: duplicate key out of range at " + std::to_string(s));
            for (int p = 0; p < passes; ++p) h2[p * 256 + ((keys[s] >> (8 * p)) & 0xff)]++;
        }
        for (int i = 0; i < passes * 256; ++i)
            if (h2[i] != hist[i]) return fail(ctx, TGSX_ESTATE, "debug: digit histogram wrong");
    }
    uint32_t* k = ws.keys[0].as<uint32_t>();
    uint32_t* v = ws.vals[0].as<uint32_t>();
    {
        StageTimer t(ctx, kStSort);
        CK(sort_pairs(ctx, k, v, ws.keys[1].as<uint32_t>(), ws.vals[1].as<uint32_t>(), K, key_bits,
                      ws.sort_tmp.as<uint32_t>()));
    }
    if (dbg && K) {
        std::vector<uint32_t> keys(K);
        // the context stream is non-blocking: order the legacy-stream copy after the sort
        CK(cudaStreamSynchronize(ctx->stream));
        CK(cudaMemcpy(keys.data(), k, K * 4, cudaMemcpyDeviceToHost));
        for (int64_t s = 1; s < K; ++s)
            if (keys[s] < keys[s - 1] || keys[s] >= (uint32_t)tiles)
                return fail(ctx, TGSX_ESTATE, "debug: onesweep output unsorted at " + std::to_string(s) +
                                                  " of " + std::to_string(K) + " passes " + std::to_string(passes));
    }
    {
        StageTimer t(ctx, kStRanges);
        CK(launch_ranges(ctx, k, K, tiles));
    }
    *items = v;
    if (sorted_keys) *sorted_keys = k;
    return TGSX_OK;
}

// Binning with reuse: a second view of the same, unchanged model at the same resolution and
// low-pass (every view of a batched step; render followed by backward) keeps the previous
// prepared records and tile lists — pixel_span works on the full-resolution image, so the lists
// do not depend on the dilation offset (rasterizer.cpp:74-100).
int32_t bin(tgsx_ctx* ctx, tgsx_model* m, int lowpass_p, int W, int H, uint32_t** items,
            uint32_t** sorted_keys, bool defer = false) {
    if (!sorted_keys && ctx->bin_valid && ctx->bin_model == m->uid && ctx->bin_lowpass == lowpass_p &&
        ctx->bin_W == W && ctx->bin_H == H && ctx->bin_n == m->n && !m->order_dirty && m->blend_phys) {
        ctx->ws.have_forward = false;
        CK(reset_counters(ctx));  // blend-op / evaluation counters are per render
        *items = ctx->bin_items;
        return TGSX_OK;
    }
    ctx->bin_valid = false;
    const int32_t rc = bin_compute(ctx, m, lowpass_p, W, H, items, sorted_keys, defer);
    if (rc) return rc;
    ctx->bin_valid = true;
    ctx->bin_model = m->uid;
    ctx->bin_lowpass = lowpass_p;
    ctx->bin_W = W;
    ctx->bin_H = H;
    ctx->bin_n = m->n;
    ctx->bin_items = *items;
    return TGSX_OK;
}

cudaError_t ensure_pixels(tgsx_ctx* ctx, const RenderArgs& ra) {
    Workspace& ws = ctx->ws;
    const size_t P = (size_t)std::max(ra.P, 1);
    cudaError_t e;
    if ((e = ws.rgb.ensure(P * 12))) return e;
    if ((e = ws.T.ensure(P * 4))) return e;
    if ((e = ws.last.ensure(P * 4))) return e;
    if ((e = ws.dLdC.ensure(P * 12))) return e;
    const int tiles = ws.tiles_x * ws.tiles_y;
    if ((e = ws.block_loss.ensure((size_t)std::max(tiles, 1) * 4))) return e;
    return cudaSuccess;
}

void fill_adam(AdamCfg& c, const tgsx_adam_args* a) {
    c.b1 = 0.9f;
    c.b2 = 0.999f;
    c.omb1 = 1.0f - c.b1;
    c.omb2 = 1.0f - c.b2;
    c.eps = 1e-15f;
    const double frac = a->total_steps > 0 ? (double)a->step / (double)a->total_steps : 0.0;
    const float lr_pos = (float)(1.6e-4 * a->image_diagonal * std::pow(0.01, frac));
    c.lr[0] = c.lr[1] = lr_pos;
    c.lr[2] = 1e-3f;
    c.lr[3] = c.lr[4] = 5e-3f;
    c.lr[5] = 5e-2f;
    c.lr[6] = c.lr[7] = c.lr[8] = 2.5e-3f;
    c.bc1 = (float)(1.0 - std::pow(0.9, (double)a->step));
    c.bc2 = (float)(1.0 - std::pow(0.999, (double)a->step));
    // clamp_parameters (gaussian.hpp:105-116) bounds, CR logf
    c.ls_lo = (float)std::log((double)(float)kMinScale);
    c.ls_hi = (float)std::log((double)(float)a->image_diagonal);
    c.raw_cap = (float)kRawCap;
    c.batch = 1.0f;
}

}  // namespace

void tgsx::adam_cfg_from_args(AdamCfg& c, const tgsx_adam_args* a) { fill_adam(c, a); }
bool tgsx::graph_eligible_binning(const tgsx_ctx* ctx) {
    return !force_onesweep(ctx) && !debug_checks() && ctx->bin_max_hint <= (uint64_t)kSegCap;
}

namespace {

// rows of a dilated view's target into the workspace (StageRowsArgs); 16-B vectors when every
// address allows (the source moves per graph replay, so the check is made per launch)
__global__ void __launch_bounds__(256) stage_rows_kernel(StageRowsArgs a) {
    const bool vec = ((reinterpret_cast<uintptr_t>(a.src) | reinterpret_cast<uintptr_t>(a.dst)) & 15u) == 0 &&
                     (a.row_floats & 3) == 0 && (a.pitch_floats & 3) == 0;
    const int64_t per_row = vec ? a.row_floats / 4 : a.row_floats;
    const int64_t total = per_row * a.rows;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = i / per_row, c = i - r * per_row;
        if (vec)
            reinterpret_cast<float4*>(a.dst + r * a.row_floats)[c] =
                __ldg(reinterpret_cast<const float4*>(a.src + r * a.pitch_floats) + c);
        else
            a.dst[r * a.row_floats + c] = __ldg(a.src + r * a.pitch_floats + c);
    }
}

bool is_device_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Host or device source into a device buffer (H2D copy inside the call for host memory).
int32_t stage_input(tgsx_ctx* ctx, DevBuf& dst, const float* src, size_t bytes, const float** out) {
    if (is_device_ptr(src)) {
        *out = src;
        return TGSX_OK;
    }
    CK(dst.ensure(bytes));
    CK(cudaMemcpyAsync(dst.p, src, bytes, cudaMemcpyDefault, ctx->stream));
    *out = dst.as<float>();
    return TGSX_OK;
}

bool is_pinned_host_ptr(const void* p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeHost;
}

// View target: device pointers are used in place; host targets go through two staging buffers
// filled on the copy stream, so the H2D of this view overlaps the previous view's kernels (the
// compute stream waits for the copy; the next copy into a buffer waits for the forward that
// read it, see mark_target_consumed).
// Host targets of a dilated view (p > 1) only stage the active rows y = oy, oy + p, ... (the fused
// L1 reads nothing else): a pitched copy of 1/p of the image, indexed by the kernel as row
// (y - oy) / p (ra->target_rows = p). Device targets are used in place (full image).
int32_t stage_target(tgsx_ctx* ctx, const float* src, size_t bytes, const float** out,
                     RenderArgs* ra = nullptr) {
    const bool rows_only = ra && ra->p > 1 && ra->rows > 0;
    const size_t row_bytes = ra ? (size_t)ra->W * 12 : 0;
    if (ctx->graph_capturing && (ctx->graph_stage_targets || !is_device_ptr(src))) {
        // a graph-replayed step copies its target (pinned host, or device once the fit uses more
        // than one target; a dilated view only its active rows) on the compute stream into the
        // workspace (sized before the capture): the copy is a node of the step's graph whose
        // source is set per replay, so one graph serves every target of the same pattern
        // (graph.cpp)
        if (rows_only) bytes = row_bytes * (size_t)ra->rows;
        DevBuf& b = ctx->ws.target;
        if (b.bytes < bytes) CK(b.ensure(bytes));
        const size_t off = rows_only ? (size_t)ra->oy * ra->W * 3 : 0;
        if (rows_only) {  // a kernel node (its source can be re-targeted in the exec, a 2-D copy's not)
            StageRowsArgs a{b.as<float>(), src + off, (int64_t)ra->W * 3, (int64_t)ra->W * 3 * ra->p, ra->rows};
            stage_rows_kernel<<<(unsigned)std::min<int64_t>(4 * 148, (int64_t)ra->rows * 8), 256, 0, ctx->stream>>>(a);
            ctx->launches++;
            CK(cudaGetLastError());
            ctx->graph_stage_args = a;
            ctx->graph_target_kind = 2;
            ra->target_rows = ra->p;
        } else {
            CK(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyDefault, ctx->stream));
            ctx->graph_target_kind = 1;
        }
        cudaStreamCaptureStatus st;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        CK(cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, nullptr, &deps, &nd));
        ctx->graph_target_node = nd == 1 ? (void*)deps[0] : nullptr;
        ctx->graph_target_off = (int64_t)off;
        *out = b.as<float>();
        return TGSX_OK;
    }
    if (is_device_ptr(src)) {
        *out = src;
        return TGSX_OK;
    }
    if (rows_only) bytes = row_bytes * (size_t)ra->rows;
    if (!ctx->copy_stream) {
        CK(cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CK(cudaEventCreateWithFlags(&ctx->staged[i], cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&ctx->consumed[i], cudaEventDisableTiming));
        }
    }
    const int k = ctx->stage_next;
    ctx->stage_next ^= 1;
    DevBuf& b = ctx->stage_buf[k];
    if (b.bytes < bytes) {
        CK(cudaStreamSynchronize(ctx->copy_stream));
        CK(cudaStreamSynchronize(ctx->stream));
        CK(b.ensure(bytes));
    }
    if (ctx->stage_used[k]) CK(cudaStreamWaitEvent(ctx->copy_stream, ctx->consumed[k], 0));
    if (rows_only) {
        CK(cudaMemcpy2DAsync(b.p, row_bytes, src + (size_t)ra->oy * ra->W * 3, row_bytes * (size_t)ra->p,
                             row_bytes, (size_t)ra->rows, cudaMemcpyHostToDevice, ctx->copy_stream));
        ra->target_rows = ra->p;
    } else {
        CK(cudaMemcpyAsync(b.p, src, bytes, cudaMemcpyHostToDevice, ctx->copy_stream));
    }
    CK(cudaEventRecord(ctx->staged[k], ctx->copy_stream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->staged[k], 0));
    ctx->stage_pending = k;
    *out = b.as<float>();
    return TGSX_OK;
}

int32_t mark_target_consumed(tgsx_ctx* ctx) {
    if (ctx->stage_pending >= 0) {
        CK(cudaEventRecord(ctx->consumed[ctx->stage_pending], ctx->stream));
        ctx->stage_used[ctx->stage_pending] = true;
        ctx->stage_pending = -1;
    }
    return TGSX_OK;
}

int32_t render_core(tgsx_ctx* ctx, tgsx_model* m, const RenderArgs& ra, bool fused_loss,
                    uint32_t** items_out, bool defer = false) {
    uint32_t* items = nullptr;
    int32_t rc = bin(ctx, m, ra.lowpass_p, ra.W, ra.H, &items, nullptr, defer);
    if (rc) return rc;
    CK(ensure_pixels(ctx, ra));
    {
        StageTimer t(ctx, kStForward);
        CK(launch_forward(ctx, ra, items, fused_loss));
    }
    bool redo = false;
    if ((rc = bin_settle(ctx, m, ra.W, ra.H, &items, &redo))) return rc;
    if (redo) {  // the speculative lists were short: forward again on the settled ones
        CK(reset_counters(ctx));
        StageTimer t(ctx, kStForward);
        CK(launch_forward(ctx, ra, items, fused_loss));
    }
    ctx->ws.have_forward = true;
    ctx->ws.last_P = ra.P;
    *items_out = items;
    return TGSX_OK;
}


// run_chain = false: everything up to (not including) the chain kernel; the caller launches the
// chain itself (tgsx_batched_step pipelines it over Gaussian buckets with the all-reduce)
int32_t fused_view(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                   const float* target, float* out_loss, ChainMode mode, const AdamCfg* cfg,
                   bool run_chain = true) {
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    if (!target) return fail(ctx, TGSX_EINVAL, "target is null");
    if (!ctx->graph_capturing && !ctx->graph_replaying && (rc = graph_flush(ctx))) return rc;
    RenderArgs ra = make_args(pat, bg, 0);
    // compute_loss: dense views add the SSIM term, dilated views are L1 only
    const float lam = (pat->p == 1 && ctx->ssim_weight > 0.f) ? ctx->ssim_weight : 0.f;
    ra.l1_weight = 1.0f - lam;
    Workspace& ws = ctx->ws;
    rc = stage_target(ctx, target, (size_t)ra.W * ra.H * 12, &ra.target, &ra);
    if (rc) return rc;
    uint32_t* items = nullptr;
    rc = render_core(ctx, m, ra, true, &items, true);  // forward + fused (1 - lam) L1
    if (rc) return rc;
    int nsb = 0;
    if (lam > 0.f && ra.P > 0) {
        StageTimer t(ctx, kStLoss);
        nsb = (int)ssim_blocks(ra.W, ra.H);
        CK(ws.ssim_abc.ensure((size_t)ra.P * 36));
        CK(ws.ssim_part.ensure((size_t)nsb * 4));
        CK(launch_ssim(ctx, ws.rgb.as<float>(), ra.target, ra.W, ra.H, lam, ws.ssim_abc.as<float>(),
                       ws.ssim_part.as<float>(), ws.dLdC.as<float>()));
    }
    if ((rc = mark_target_consumed(ctx))) return rc;  // the loss kernels are the target's readers
    {
        StageTimer t(ctx, kStBackward);
        CK(launch_backward(ctx, ra, items));
    }
    if (run_chain) {
        StageTimer t(ctx, kStChain);
        CK(launch_chain(ctx, m, mode, true, nullptr, reinterpret_cast<const float*>(cfg)));
        if (ctx->graph_capturing) {  // the chain node: its Adam arguments change per replay
            cudaStreamCaptureStatus st;
            const cudaGraphNode_t* deps = nullptr;
            size_t nd = 0;
            CK(cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, nullptr, &deps, &nd));
            ctx->graph_chain_node = nd == 1 ? (void*)deps[0] : nullptr;
        }
    }
    if (mode == ChainMode::kAdam) ctx->bin_valid = false;  // the parameters moved
    const int tiles = ws.tiles_x * ws.tiles_y;
    float* dloss = reinterpret_cast<float*>(ws.counters.as<unsigned long long>() + 4);
    {
        StageTimer t(ctx, kStLoss);
        const double inv = ra.P > 0 ? 1.0 / (3.0 * (double)ra.P) : 0.0;
        CK(launch_loss_finalize(ctx, ws.block_loss.as<float>(), tiles, (float)((1.0 - lam) * inv),
                                ws.ssim_part.as<float>(), nsb, lam, inv, dloss));
    }
    CK(cudaGetLastError());
    if (out_loss) {
        // device and pinned host destinations are written in stream order (read the pinned
        // value after tgsx_synchronize); pageable host memory is written before returning
        CK(cudaMemcpyAsync(out_loss, dloss, 4, cudaMemcpyDefault, ctx->stream));
        if (ctx->graph_capturing) {  // the loss copy node: its destination is set per replay
            cudaStreamCaptureStatus st;
            const cudaGraphNode_t* deps = nullptr;
            size_t nd = 0;
            CK(cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, nullptr, &deps, &nd));
            ctx->graph_loss_node = nd == 1 ? (void*)deps[0] : nullptr;
            ctx->graph_loss_src = dloss;
        } else if (!is_device_ptr(out_loss) && !is_pinned_host_ptr(out_loss)) {
            CK(cudaStreamSynchronize(ctx->stream));
        }
    }
    return TGSX_OK;
}

// ============================================================================ 3-D front end
// preprocess3d -> depth sort (onesweep, 32-bit keys) -> rank-order
// gather + slab claims -> the 2-D path's scan / per-tile sort / blend kernels -> chain3d.

int32_t make_cam3(tgsx_ctx* ctx, const tgsx_camera* c, const tgsx_pattern* pat, Cam3* out) {
    if (!c) return fail(ctx, TGSX_EINVAL, "camera is null");
    if (pat && (c->width != pat->width || c->height != pat->height))
        return fail(ctx, TGSX_EINVAL, "camera size does not match the pattern size");
    if (!(c->fx > 0.f) || !(c->fy > 0.f) || !(c->znear > 0.f) || !std::isfinite(c->fx) ||
        !std::isfinite(c->fy) || !std::isfinite(c->cx) || !std::isfinite(c->cy) || c->width < 1 ||
        c->height < 1)
        return fail(ctx, TGSX_EINVAL, "camera: fx, fy, znear must be positive and finite");
    Cam3 k{};
    for (int i = 0; i < 9; ++i) k.R[i] = c->R[i];
    for (int i = 0; i < 3; ++i) k.t[i] = c->t[i];
    k.fx = c->fx; k.fy = c->fy; k.cx = c->cx; k.cy = c->cy; k.znear = c->znear;
    k.limx = (float)(1.3 * 0.5 * (double)c->width / (double)c->fx);
    k.limy = (float)(1.3 * 0.5 * (double)c->height / (double)c->fy);
    for (int j = 0; j < 3; ++j)
        k.C[j] = (float)(-((double)c->R[j] * c->t[0] + (double)c->R[3 + j] * c->t[1] +
                           (double)c->R[6 + j] * c->t[2]));
    *out = k;
    return TGSX_OK;
}

int32_t check_kernel_error3d(tgsx_ctx* ctx, unsigned long long err) {
    if (err == kErrNone) return TGSX_OK;
    const uint32_t code = (uint32_t)(err & 3u);
    const unsigned long long row = err >> 2;
    if (code == 1)
        return fail(ctx, TGSX_EINVAL, "3-D Gaussian with non-finite parameters or a zero quaternion (row " +
                                          std::to_string(row) + ")");
    return fail(ctx, TGSX_ERUNTIME, "projected covariance numerically degenerate (row " + std::to_string(row) + ")");
}

// defer (fused 3-D views): as the 2-D bin_compute — the per-tile sort is launched for lists up to
// the previous 3-D binning's longest (x1.25) without waiting for the counters; the caller queues
// its forward and bin3d_settle() checks them, redoing the lists when the guess was short. The
// host then never stalls the stream between the preprocess and the blend kernels.
int32_t bin3d(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int W, int H,
              uint32_t** items, bool defer = false) {
    Workspace& ws = ctx->ws;
    ctx->bin_valid = false;  // the 2-D path's binning reuse never sees these buffers as its own
    ctx->bin_pending = false;
    ctx->bin3d_pending = false;
    ws.have_forward = false;
    const int64_t n = m->n;
    CK(reset_counters(ctx));
    unsigned long long* counters0 = ws.counters.as<unsigned long long>();
    const int ntiles = ((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile);
    if (!force_onesweep(ctx)) {
        // per-tile path: no global depth sort. Rows claim their tiles' slab slots, the per-tile
        // warp sort orders every list by (depth key, row) = the blend order inside the tile.
        {
            StageTimer t(ctx, kStPreprocess);
            CK(launch_preprocess3d_bin(ctx, m, cam, lowpass_p, W, H, reinterpret_cast<uint32_t*>(counters0 + 3)));
        }
        {
            StageTimer t(ctx, kStScan);
            CK(launch_slab_finalize(ctx, ntiles));
        }
        CK(cudaMemcpyAsync(ws.h_scratch, counters0, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                           ctx->stream));
        if (defer && ctx->bin3d_max_hint > 0 && !debug_checks()) {
            if (!ctx->bin_event) CK(cudaEventCreateWithFlags(&ctx->bin_event, cudaEventDisableTiming));
            CK(cudaEventRecord(ctx->bin_event, ctx->stream));
            const uint64_t guess = std::min<uint64_t>(kSegCap, ctx->bin3d_max_hint + ctx->bin3d_max_hint / 4);
            ctx->bin3d_sort_cap = guess <= 256 ? 256 : (guess <= 512 ? 512 : kSegCap);
            {
                StageTimer t(ctx, kStSort);
                CK(launch_seg_sort3d(ctx, ntiles, (int64_t)guess));
            }
            m->rank_ordered = false;
            ctx->bin3d_pending = true;
            *items = ws.tile_slab.as<uint32_t>();
            return TGSX_OK;
        }
        CK(cudaStreamSynchronize(ctx->stream));
        if (ctx->prof.enabled) ctx->prof.harvest();
        int32_t rc0 = check_kernel_error3d(ctx, ws.h_scratch[0]);
        if (rc0) return rc0;
        const uint64_t max_list = ws.h_scratch[5];
        ctx->bin3d_max_hint = max_list;
        if (max_list <= (uint64_t)kSegCap) {
            const int64_t K = (int64_t)(uint32_t)(ws.h_scratch[3] & 0xffffffffull);
            ws.K = K;
            CK(ws.partial.ensure(std::max<int64_t>(K, 1) * 40));
            ws.pair_cap = (int64_t)(ws.partial.bytes / 40);
            {
                StageTimer t(ctx, kStSort);
                CK(launch_seg_sort3d(ctx, ntiles, (int64_t)max_list));
            }
            m->rank_ordered = false;
            *items = ws.tile_slab.as<uint32_t>();
            return TGSX_OK;
        }
        // a list longer than a slab: the global-sort path below
        CK(reset_counters(ctx));
    }
    m->rank_ordered = true;
    {
        StageTimer t(ctx, kStPreprocess);
        CK(launch_preprocess3d(ctx, m, cam, lowpass_p, W, H));
    }
    uint32_t* k = ws.keys[0].as<uint32_t>();
    uint32_t* v = ws.vals[0].as<uint32_t>();
    unsigned long long* counters = ws.counters.as<unsigned long long>();
    uint32_t* d_total = reinterpret_cast<uint32_t*>(counters + 3);
    {
        // blend order of this view: ascending camera depth, ties by row (stable LSD passes)
        StageTimer t(ctx, kStDepthSort);
        CK(sort_pairs(ctx, k, v, ws.keys[1].as<uint32_t>(), ws.vals[1].as<uint32_t>(), n, 32, nullptr));
        CK(launch_bin3d(ctx, m, k, v, W, H, d_total));
        // the onesweep binning below reuses the key buffers: keep the sorted depth keys
        CK(m->skeys.ensure((size_t)std::max<int64_t>(n, 1) * 4));
        if (n) CK(cudaMemcpyAsync(m->skeys.p, k, (size_t)n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    const int tiles = ws.tiles_x * ws.tiles_y;
    {
        StageTimer t(ctx, kStScan);
        CK(launch_slab_finalize(ctx, tiles));
    }
    CK(cudaMemcpyAsync(ws.h_scratch, counters, 6 * sizeof(unsigned long long), cudaMemcpyDeviceToHost,
                       ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (ctx->prof.enabled) ctx->prof.harvest();
    int32_t rc = check_kernel_error3d(ctx, ws.h_scratch[0]);
    if (rc) return rc;
    const int64_t K = (int64_t)(uint32_t)(ws.h_scratch[3] & 0xffffffffull);
    const uint64_t max_list = ws.h_scratch[5];
    ws.K = K;
    CK(ws.partial.ensure(std::max<int64_t>(K, 1) * 40));
    ws.pair_cap = (int64_t)(ws.partial.bytes / 40);
    if (max_list <= (uint64_t)kSegCap && !force_onesweep(ctx)) {
        rc = slab_sort(ctx, tiles, max_list);
        if (rc) return rc;
        *items = ws.tile_slab.as<uint32_t>();
        return TGSX_OK;
    }
    return bin_onesweep(ctx, nullptr, n, W, H, K, items, nullptr);
}

// Completes a deferred 3-D binning (bin3d with defer): waits for the counters (normally long
// complete), reports kernel errors, sizes the per-pair partials and, when the speculative per-tile
// sort was too short (or a list outgrew its slab: the global-sort path), redoes the lists; *redo
// tells the caller to rerun its forward.
int32_t bin3d_settle(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int W, int H,
                     uint32_t** items, bool* redo) {
    *redo = false;
    if (!ctx->bin3d_pending) return TGSX_OK;
    ctx->bin3d_pending = false;
    Workspace& ws = ctx->ws;
    CK(cudaEventSynchronize(ctx->bin_event));
    int32_t rc = check_kernel_error3d(ctx, ws.h_scratch[0]);
    if (rc) return rc;
    const int64_t K = (int64_t)(uint32_t)(ws.h_scratch[3] & 0xffffffffull);
    const uint64_t max_list = ws.h_scratch[5];
    ctx->bin3d_max_hint = max_list;
    if (max_list > (uint64_t)kSegCap) {  // a list longer than a slab: bin again on the global-sort path
        *redo = true;
        return bin3d(ctx, m, cam, lowpass_p, W, H, items, false);
    }
    ws.K = K;
    CK(ws.partial.ensure(std::max<int64_t>(K, 1) * 40));
    ws.pair_cap = (int64_t)(ws.partial.bytes / 40);
    if (max_list <= (uint64_t)ctx->bin3d_sort_cap) return TGSX_OK;
    *redo = true;
    {
        StageTimer t(ctx, kStSort);
        CK(launch_seg_sort3d(ctx, ((W + kTile - 1) / kTile) * ((H + kTile - 1) / kTile), (int64_t)max_list));
    }
    *items = ws.tile_slab.as<uint32_t>();
    return TGSX_OK;
}

int32_t render3d_core(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, const RenderArgs& ra,
                      bool fused_loss, uint32_t** items_out, bool defer = false) {
    uint32_t* items = nullptr;
    int32_t rc = bin3d(ctx, m, cam, ra.lowpass_p, ra.W, ra.H, &items, defer);
    if (rc) return rc;
    CK(ensure_pixels(ctx, ra));
    {
        StageTimer t(ctx, kStForward);
        CK(launch_forward(ctx, ra, items, fused_loss));
    }
    bool redo = false;
    if ((rc = bin3d_settle(ctx, m, cam, ra.lowpass_p, ra.W, ra.H, &items, &redo))) return rc;
    if (redo) {  // the speculative lists were short: forward again on the settled ones
        CK(reset_counters(ctx));
        StageTimer t(ctx, kStForward);
        CK(launch_forward(ctx, ra, items, fused_loss));
    }
    ctx->ws.have_forward = true;
    ctx->ws.last_P = ra.P;
    *items_out = items;
    return TGSX_OK;
}

void fill_adam3d(Adam3dCfg& c, const tgsx_adam3d_args* a) {
    // or3d_adam_config (oracle/ewa3d.c): 3DGS learning rates, SPEC.md:258-267 update
    c.b1 = 0.9f;
    c.b2 = 0.999f;
    c.omb1 = 1.0f - c.b1;
    c.omb2 = 1.0f - c.b2;
    c.eps = 1e-15f;
    const double frac = a->total_steps > 0 ? (double)a->step / (double)a->total_steps : 0.0;
    c.lr[0] = (float)(1.6e-4 * a->scene_extent * std::pow(0.01, frac));
    c.lr[1] = 1e-3f;
    c.lr[2] = 5e-3f;
    c.lr[3] = 5e-2f;
    c.lr[4] = 2.5e-3f;
    c.lr[5] = 2.5e-3f / 20.0f;
    c.bc1 = (float)(1.0 - std::pow(0.9, (double)a->step));
    c.bc2 = (float)(1.0 - std::pow(0.999, (double)a->step));
    c.raw_cap = (float)kRawCap;
}

cudaError_t model3d_reserve(tgsx_ctx* ctx, tgsx_model3d* m, int64_t cap, bool keep) {
    if (cap <= m->cap && m->params.p) return cudaSuccess;
    const int64_t nc = std::max<int64_t>(cap, 1);
    cudaError_t e;
    auto regrow = [&](DevBuf& b, int rows, size_t elt) -> cudaError_t {
        DevBuf nb;
        cudaError_t er = nb.ensure((size_t)rows * nc * elt);
        if (er) return er;
        if (keep && b.p && m->n) {
            er = cudaMemcpy2DAsync(nb.p, nc * elt, b.p, m->cap * elt, m->n * elt, rows, cudaMemcpyDeviceToDevice,
                                   ctx->stream);
            if (er) return er;
            er = cudaStreamSynchronize(ctx->stream);
            if (er) return er;
        }
        b.release();
        b = nb;
        return cudaSuccess;
    };
    if ((e = regrow(m->params, k3dParams, 4))) return e;
    if ((e = regrow(m->m1, k3dParams, 4))) return e;
    if ((e = regrow(m->m2, k3dParams, 4))) return e;
    if ((e = regrow(m->pos_acc, 1, 4))) return e;
    if ((e = regrow(m->col_acc, 1, 4))) return e;
    if ((e = regrow(m->visit, 1, 4))) return e;
    if ((e = regrow(m->step, k3dStepRows, 4))) return e;
    if ((e = regrow(m->ids, 1, 8))) return e;
    if ((e = regrow(m->tau_v, 1, 8))) return e;
    if ((e = regrow(m->visit_evt, 1, 4))) return e;
    if ((e = regrow(m->visit_aud, 1, 4))) return e;
    if ((e = m->perm.ensure(nc * 4))) return e;
    if ((e = m->rank_of.ensure(nc * 4))) return e;
    if ((e = m->prep_row.ensure(nc * sizeof(Prepared)))) return e;
    m->cap = nc;
    return cudaSuccess;
}

}  // namespace

cudaError_t model3d_grow(tgsx_ctx* ctx, tgsx_model3d* m, int64_t cap) { return model3d_reserve(ctx, m, cap, true); }

// ============================================================================ C ABI
extern "C" {

int32_t tgsx_create(int32_t device, tgsx_ctx** out) {
    if (!out) return TGSX_EINVAL;
    *out = nullptr;
    tgsx_ctx* ctx = new tgsx_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (!e) e = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    if (!e) e = cudaMallocHost(&ctx->ws.h_scratch, 64 * sizeof(uint64_t));
    if (!e) e = ctx->ws.counters.ensure(8 * sizeof(unsigned long long));
    if (e) {
        delete ctx;
        return TGSX_ECUDA;
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return TGSX_OK;
}

void tgsx_destroy(tgsx_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    graph_release(ctx);
    Workspace& ws = ctx->ws;
    DevBuf* bufs[] = {&ws.prep, &ws.touched, &ws.pair_off, &ws.scan_tmp, &ws.keys[0], &ws.keys[1],
                      &ws.vals[0], &ws.vals[1], &ws.sort_tmp, &ws.ranges, &ws.partial, &ws.rgb,
                      &ws.T, &ws.last, &ws.dLdC, &ws.target, &ws.block_loss, &ws.counters,
                      &ws.generic, &ws.tile_fill, &ws.tile_slab, &ws.ssim_abc, &ws.ssim_part,
                      &ws.loss_grad, &ws.rect};
    for (DevBuf* b : bufs) b->release();
    drain_graveyard();
    if (ctx->copy_stream) {
        cudaStreamSynchronize(ctx->copy_stream);
        cudaStreamDestroy(ctx->copy_stream);
        for (int i = 0; i < 2; ++i) {
            ctx->stage_buf[i].release();
            cudaEventDestroy(ctx->staged[i]);
            cudaEventDestroy(ctx->consumed[i]);
        }
    }
    comm_release(ctx);
    if (ws.h_scratch) cudaFreeHost(ws.h_scratch);
    if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
    delete ctx;
}

int32_t tgsx_set_stream(tgsx_ctx* ctx, void* stream) {
    if (!ctx) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return TGSX_OK;
}

void* tgsx_get_stream(tgsx_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

const char* tgsx_last_error(const tgsx_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int32_t tgsx_host_alloc(size_t bytes, void** out) {
    if (!out) return TGSX_EINVAL;
    *out = nullptr;
    if (bytes == 0) return TGSX_OK;
    return cudaHostAlloc(out, bytes, cudaHostAllocDefault) == cudaSuccess ? TGSX_OK : TGSX_ENOMEM;
}

void tgsx_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int32_t tgsx_synchronize(tgsx_ctx* ctx) {
    if (int32_t rc = graph_flush(ctx)) return rc;
    CK(cudaStreamSynchronize(ctx->stream));
    drain_graveyard();  // outgrown buffers (the stream is idle here)
    return TGSX_OK;
}

uint64_t tgsx_launch_count(const tgsx_ctx* ctx) { return ctx ? ctx->launches : 0; }

int32_t tgsx_profile(tgsx_ctx* ctx, int32_t enable) {
    if (!ctx) return TGSX_EINVAL;
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->prof.harvest();
    for (int i = 0; i < kNumStages; ++i) {
        ctx->prof.ms[i] = 0;
        ctx->prof.count[i] = 0;
    }
    ctx->prof.enabled = enable != 0;
    return TGSX_OK;
}

int32_t tgsx_profile_read(tgsx_ctx* ctx, double* ms, int64_t* counts, int32_t n) {
    if (!ctx) return TGSX_EINVAL;
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->prof.harvest();
    for (int i = 0; i < n && i < kNumStages; ++i) {
        if (ms) ms[i] = ctx->prof.ms[i];
        if (counts) counts[i] = ctx->prof.count[i];
    }
    return TGSX_OK;
}

// ---------------------------------------------------------------- model
int32_t tgsx_model_create(tgsx_ctx* ctx, int64_t capacity, tgsx_model** out) {
    if (!ctx || !out) return TGSX_EINVAL;
    tgsx_model* m = new tgsx_model();
    static std::atomic<uint64_t> next_uid{1};
    m->uid = next_uid.fetch_add(1);
    cudaError_t e = model_reserve(ctx, m, std::max<int64_t>(capacity, 1));
    if (e) {
        delete m;
        return cuda_fail(ctx, e, "tgsx_model_create");
    }
    *out = m;
    return TGSX_OK;
}

void tgsx_model_destroy(tgsx_model* m) {
    if (!m) return;
    DevBuf* bufs[] = {&m->params, &m->ids, &m->pos_acc, &m->col_acc, &m->accum, &m->visit,
                      &m->window, &m->tau_v, &m->m1, &m->m2, &m->step, &m->perm, &m->rank_of,
                      &m->screen};
    for (DevBuf* b : bufs) b->release();
    for (DevBuf& b : m->spare) b.release();
    delete m;
}

int32_t tgsx_model_reserve(tgsx_ctx* ctx, tgsx_model* m, int64_t capacity) {
    if (!ctx || !m || capacity < 0) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    ctx->bin_valid = false;
    CK(model_grow(ctx, m, capacity));
    // per-Gaussian workspace (prepared records, counts, offsets, depth-sort and densify scratch)
    Workspace& ws = ctx->ws;
    const int64_t c = std::max<int64_t>(m->cap, 1);
    CK(ws.prep.ensure(c * sizeof(Prepared)));
    CK(ws.touched.ensure((c + 1) * 4));
    CK(ws.pair_off.ensure((c + 1) * 4));
    for (int i = 0; i < 2; ++i) CK(ws.keys[i].ensure(c * 4));
    CK(ws.generic.ensure((size_t)c * 4 * 7));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int64_t tgsx_model_size(const tgsx_model* m) { return m ? m->n : 0; }
uint64_t tgsx_model_next_id(const tgsx_model* m) { return m ? m->next_id : 0; }

int32_t tgsx_model_upload(tgsx_ctx* ctx, tgsx_model* m, const tgsx_host_scene* h) {
    if (!ctx || !m || !h || h->n < 0) return fail(ctx, TGSX_EINVAL, "bad upload arguments");
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    ctx->bin_valid = false;
    const int64_t n = h->n;
    CK(model_reserve(ctx, m, n));
    m->n = n;
    m->blend_phys = false;  // uploaded rows are in logical order
    cudaStream_t s = ctx->stream;
    const int64_t cap = m->cap;
    float* P = m->params.as<float>();
    const float* rows[kParamRows] = {h->px, h->py, h->rot, h->lsx, h->lsy, h->rop, h->cr, h->cg, h->cb, h->depth};
    for (int q = 0; q < kParamRows; ++q) {
        if (!rows[q] && n) return fail(ctx, TGSX_EINVAL, "null parameter array");
        if (n) CK(cudaMemcpyAsync(P + q * cap, rows[q], n * 4, cudaMemcpyDefault, s));
    }
    std::vector<uint64_t> ids;
    const uint64_t* idp = h->id;
    if (!idp) {
        ids.resize(n);
        for (int64_t i = 0; i < n; ++i) ids[i] = (uint64_t)i;
        idp = ids.data();
    }
    bool mono = true;
    uint64_t mx = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (i && idp[i] <= idp[i - 1]) mono = false;
        mx = std::max(mx, idp[i]);
    }
    m->ids_monotone = mono;
    m->next_id = h->id ? std::max<uint64_t>(h->next_id, n ? mx + 1 : 0) : (uint64_t)n;
    if (n) CK(cudaMemcpyAsync(m->ids.p, idp, n * 8, cudaMemcpyHostToDevice, s));
    // stats (zeros when absent), tau_v (5.0 when absent)
    auto up_or_zero = [&](DevBuf& b, const void* src, size_t elt) -> cudaError_t {
        if (!n) return cudaSuccess;
        if (src) return cudaMemcpyAsync(b.p, src, n * elt, cudaMemcpyDefault, s);
        return cudaMemsetAsync(b.p, 0, n * elt, s);
    };
    CK(up_or_zero(m->pos_acc, h->pos_acc, 4));
    CK(up_or_zero(m->col_acc, h->col_acc, 4));
    CK(up_or_zero(m->accum, h->accum, 4));
    CK(up_or_zero(m->visit, h->visit, 8));
    CK(up_or_zero(m->window, h->window, 8));
    if (h->tau_v) {
        if (n) CK(cudaMemcpyAsync(m->tau_v.p, h->tau_v, n * 8, cudaMemcpyDefault, s));
    } else if (n) {
        std::vector<double> tv(n, 5.0);
        CK(cudaMemcpyAsync(m->tau_v.p, tv.data(), n * 8, cudaMemcpyHostToDevice, s));
        CK(cudaStreamSynchronize(s));
    }
    CK(cudaMemsetAsync(m->m1.p, 0, m->m1.bytes, s));
    CK(cudaMemsetAsync(m->m2.p, 0, m->m2.bytes, s));
    CK(cudaMemsetAsync(m->step.p, 0, m->step.bytes, s));
    m->step_views = 0;
    m->order_dirty = true;
    CK(cudaStreamSynchronize(s));
    return TGSX_OK;
}

int32_t tgsx_model_download(tgsx_ctx* ctx, tgsx_model* m, tgsx_host_scene* h) {
    if (!ctx || !m || !h) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    CK(model_to_logical_order(ctx, m));
    const int64_t n = m->n, cap = m->cap;
    cudaStream_t s = ctx->stream;
    float* rows[kParamRows] = {h->px, h->py, h->rot, h->lsx, h->lsy, h->rop, h->cr, h->cg, h->cb, h->depth};
    const float* P = m->params.as<float>();
    for (int q = 0; q < kParamRows; ++q)
        if (rows[q] && n) CK(cudaMemcpyAsync(rows[q], P + q * cap, n * 4, cudaMemcpyDefault, s));
    if (h->id && n) CK(cudaMemcpyAsync(h->id, m->ids.p, n * 8, cudaMemcpyDefault, s));
    if (h->pos_acc && n) CK(cudaMemcpyAsync(h->pos_acc, m->pos_acc.p, n * 4, cudaMemcpyDefault, s));
    if (h->col_acc && n) CK(cudaMemcpyAsync(h->col_acc, m->col_acc.p, n * 4, cudaMemcpyDefault, s));
    if (h->accum && n) CK(cudaMemcpyAsync(h->accum, m->accum.p, n * 4, cudaMemcpyDefault, s));
    if (h->visit && n) CK(cudaMemcpyAsync(h->visit, m->visit.p, n * 8, cudaMemcpyDefault, s));
    if (h->window && n) CK(cudaMemcpyAsync(h->window, m->window.p, n * 8, cudaMemcpyDefault, s));
    if (h->tau_v && n) CK(cudaMemcpyAsync(h->tau_v, m->tau_v.p, n * 8, cudaMemcpyDefault, s));
    h->n = n;
    h->next_id = m->next_id;
    CK(cudaStreamSynchronize(s));
    return TGSX_OK;
}

int32_t tgsx_model_download_moments(tgsx_ctx* ctx, tgsx_model* m, float* m1, float* m2) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    CK(model_to_logical_order(ctx, m));
    const int64_t n = m->n, cap = m->cap;
    if (n) {
        if (m1) CK(cudaMemcpy2DAsync(m1, n * 4, m->m1.p, cap * 4, n * 4, 9, cudaMemcpyDefault, ctx->stream));
        if (m2) CK(cudaMemcpy2DAsync(m2, n * 4, m->m2.p, cap * 4, n * 4, 9, cudaMemcpyDefault, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_model_upload_moments(tgsx_ctx* ctx, tgsx_model* m, const float* m1, const float* m2) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    CK(model_to_logical_order(ctx, m));
    const int64_t n = m->n, cap = m->cap;
    if (n) {
        if (m1) CK(cudaMemcpy2DAsync(m->m1.p, cap * 4, m1, n * 4, n * 4, 9, cudaMemcpyDefault, ctx->stream));
        if (m2) CK(cudaMemcpy2DAsync(m->m2.p, cap * 4, m2, n * 4, n * 4, 9, cudaMemcpyDefault, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

// ---------------------------------------------------------------- render / backward
int32_t tgsx_render(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                    int32_t lowpass_p, float* out_rgb, float* out_T, uint64_t* out_blend_ops) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    RenderArgs ra = make_args(pat, bg, lowpass_p);
    uint32_t* items = nullptr;
    rc = render_core(ctx, m, ra, false, &items);
    if (rc) return rc;
    Workspace& ws = ctx->ws;
    if (out_rgb && ra.P) CK(cudaMemcpyAsync(out_rgb, ws.rgb.p, (size_t)ra.P * 12, cudaMemcpyDefault, ctx->stream));
    if (out_T && ra.P) CK(cudaMemcpyAsync(out_T, ws.T.p, (size_t)ra.P * 4, cudaMemcpyDefault, ctx->stream));
    if (out_blend_ops) {
        CK(cudaMemcpyAsync(ws.h_scratch + 8, ws.counters.as<unsigned long long>() + 1, 8,
                           cudaMemcpyDeviceToHost, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    if (out_blend_ops) *out_blend_ops = ws.h_scratch[8];
    return TGSX_OK;
}

int32_t tgsx_backward(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                      int32_t lowpass_p, const float* dLdC, int64_t dLdC_count, float* out_grads,
                      int32_t update_stats) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    RenderArgs ra = make_args(pat, bg, lowpass_p);
    if (dLdC_count != ra.P)
        return fail(ctx, TGSX_EINVAL, "backward: loss-gradient count does not match pattern ranks");
    // the reference recomputes the forward inside backward (rasterizer.cpp:227-263)
    uint32_t* items = nullptr;
    rc = render_core(ctx, m, ra, false, &items);
    if (rc) return rc;
    Workspace& ws = ctx->ws;
    if (ra.P) CK(cudaMemcpyAsync(ws.dLdC.p, dLdC, (size_t)ra.P * 12, cudaMemcpyDefault, ctx->stream));
    CK(launch_backward(ctx, ra, items));
    float* gout = nullptr;
    bool host_out = false;
    if (out_grads && m->n) {
        if (is_device_ptr(out_grads)) {
            gout = out_grads;
        } else {
            CK(ws.generic.ensure((size_t)m->n * 36));
            gout = ws.generic.as<float>();
            host_out = true;
        }
    } else if (m->n) {
        CK(ws.generic.ensure((size_t)m->n * 36));
        gout = ws.generic.as<float>();
    }
    CK(launch_chain(ctx, m, ChainMode::kGrads, update_stats != 0, gout, nullptr));
    if (host_out) CK(cudaMemcpyAsync(out_grads, gout, (size_t)m->n * 36, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

// ---------------------------------------------------------------- fit step
int32_t tgsx_adam_step(tgsx_ctx* ctx, tgsx_model* m, const float* grads, const tgsx_adam_args* a) {
    if (!ctx || !m || !grads || !a) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    ctx->bin_valid = false;
    AdamCfg c;
    fill_adam(c, a);
    CK(model_to_logical_order(ctx, m));  // explicit gradients are in logical order
    const float* g = nullptr;
    int32_t rc = stage_input(ctx, ctx->ws.generic, grads, (size_t)std::max<int64_t>(m->n, 1) * 36, &g);
    if (rc) return rc;
    CK(launch_adam(ctx, m, g, reinterpret_cast<const float*>(&c), 1));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_fit_step(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                      const float* target, const tgsx_adam_args* a, float* out_loss) {
    if (!ctx || !m || !a) return TGSX_EINVAL;
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    AdamCfg c;
    fill_adam(c, a);
    return fused_view(ctx, m, pat, bg, target, out_loss, ChainMode::kAdam, &c);
}

int32_t tgsx_view_accumulate(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat,
                             const float bg[3], const float* target, float* out_loss) {
    if (!ctx || !m) return TGSX_EINVAL;
    int32_t rc = fused_view(ctx, m, pat, bg, target, out_loss, ChainMode::kAccumulate, nullptr);
    if (!rc) m->step_views++;
    return rc;
}

float* tgsx_step_buffer(tgsx_model* m, int64_t* out_floats) {
    if (!m) return nullptr;
    if (out_floats) *out_floats = (int64_t)kStepFloats * m->n;  // AoS [n][12]: exactly 48 B/G
    return m->step.as<float>();
}

// Canonical row order of the step buffer shared by every rank of a view-sharded step: the blend
// order (identical on every rank: depth_key and ids are replicated). A rank that accumulated views
// is already there (fused views permute the rows into blend order); a rank with no view of the
// step must be brought there BEFORE the all-reduce — its buffer is still zero, so the
// permutation moves nothing but the model rows — or it would apply blend-ordered sums to
// logically ordered rows.
int32_t tgsx_step_layout(tgsx_ctx* ctx, tgsx_model* m) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (m->order_dirty) {
        ctx->bin_valid = false;
        CK(launch_sort_depth(ctx, m));
    }
    if (!m->blend_phys) CK(model_to_blend_order(ctx, m));
    return TGSX_OK;
}

// Sum of the step buffer over the attached communicator's ranks (48 B per Gaussian, in place),
// on the comm stream ordered after / before the compute stream.
int32_t tgsx_allreduce_step(tgsx_ctx* ctx, tgsx_model* m) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (!ctx->comm) return fail(ctx, TGSX_ESTATE, "no communicator attached (tgsx_comm_init)");
    int32_t rc = tgsx_step_layout(ctx, m);
    if (rc) return rc;
    if (ctx->pipe_events.size() < 2) {
        for (auto& e : ctx->pipe_events) cudaEventDestroy(e);
        ctx->pipe_events.assign(2, nullptr);
        for (auto& e : ctx->pipe_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->pipe_events[0], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->pipe_events[0], 0));
    if ((rc = comm_allreduce_sum(ctx, m->step.as<float>(), (size_t)kStepFloats * m->n, ctx->comm_stream))) return rc;
    CK(cudaEventRecord(ctx->pipe_events[1], ctx->comm_stream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->pipe_events[1], 0));
    return TGSX_OK;
}

// One view-sharded batched step of this rank: its n_views views accumulated into
// the step buffer, the buffer summed over the communicator's ranks, then the identical Adam +
// stats update over the global batch (rasterizer.cpp:350-358). The last view's
// chain kernel, the all-reduce and Adam are pipelined over `buckets` contiguous Gaussian ranges:
// chain(b) -> all-reduce(b) on the comm stream -> Adam(b), so the transfer of bucket b overlaps
// the chain of bucket b+1 and the Adam of bucket b-1.
int32_t tgsx_batched_step(tgsx_ctx* ctx, tgsx_model* m, int32_t n_views, const tgsx_pattern* pats,
                          const float bg[3], const float* const* targets, int32_t batch_views,
                          const tgsx_adam_args* a, float* out_losses, int32_t buckets) {
    if (!ctx || !m || !a || n_views < 0 || (n_views > 0 && (!pats || !targets)))
        return fail(ctx, TGSX_EINVAL, "batched_step: bad arguments");
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (batch_views < 1 || batch_views < n_views) return fail(ctx, TGSX_EINVAL, "batched_step: bad batch size");
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    AdamCfg c;
    fill_adam(c, a);
    c.batch = (float)batch_views;
    int32_t rc;
    for (int v = 0; v + 1 < n_views; ++v) {
        rc = fused_view(ctx, m, &pats[v], bg, targets[v], out_losses ? out_losses + v : nullptr,
                        ChainMode::kAccumulate, nullptr);
        if (rc) return rc;
    }
    const bool last_view = n_views > 0;
    if (last_view) {
        rc = fused_view(ctx, m, &pats[n_views - 1], bg, targets[n_views - 1],
                        out_losses ? out_losses + n_views - 1 : nullptr, ChainMode::kAccumulate, nullptr, false);
        if (rc) return rc;
    } else if ((rc = tgsx_step_layout(ctx, m))) {
        return rc;
    }
    const int64_t n = m->n;
    const bool comm = ctx->comm != nullptr;
    const int B = comm ? (int)std::max<int64_t>(1, std::min<int64_t>(std::max(buckets, 1), (n + 1023) / 1024)) : 1;
    // bucket bounds, aligned to 256 Gaussians (whole chain / Adam blocks, 12 KB NCCL chunks)
    std::vector<int64_t> lo(B + 1);
    for (int b = 0; b <= B; ++b) lo[b] = std::min<int64_t>(n, ((n * b / B) + 255) / 256 * 256);
    lo[B] = n;
    const size_t ne = 1 + 6 * (size_t)B;
    if (ctx->pipe_events.size() < ne) {
        for (auto& e : ctx->pipe_events) cudaEventDestroy(e);
        ctx->pipe_events.assign(ne, nullptr);
        for (auto& e : ctx->pipe_events) CK(cudaEventCreate(&e));  // timing: the pipeline timeline
    }
    cudaEvent_t* ev = ctx->pipe_events.data();  // [0] step start; per bucket 6: chain s/e, ar s/e, adam s/e
    CK(cudaEventRecord(ev[0], ctx->stream));
    for (int b = 0; b < B; ++b) {
        cudaEvent_t* e = ev + 1 + 6 * b;
        CK(cudaEventRecord(e[0], ctx->stream));
        if (last_view) {
            StageTimer t(ctx, kStChain);
            CK(launch_chain(ctx, m, ChainMode::kAccumulate, true, nullptr, nullptr, lo[b], lo[b + 1]));
        }
        CK(cudaEventRecord(e[1], ctx->stream));
        if (comm) {
            CK(cudaStreamWaitEvent(ctx->comm_stream, e[1], 0));
            CK(cudaEventRecord(e[2], ctx->comm_stream));
            rc = comm_allreduce_sum(ctx, m->step.as<float>() + (size_t)kStepFloats * lo[b],
                                    (size_t)kStepFloats * (lo[b + 1] - lo[b]), ctx->comm_stream);
            if (rc) return rc;
            CK(cudaEventRecord(e[3], ctx->comm_stream));
        }
    }
    for (int b = 0; b < B; ++b) {
        cudaEvent_t* e = ev + 1 + 6 * b;
        if (comm) CK(cudaStreamWaitEvent(ctx->stream, e[3], 0));
        CK(cudaEventRecord(e[4], ctx->stream));
        {
            StageTimer t(ctx, kStAdam);
            CK(launch_adam(ctx, m, nullptr, reinterpret_cast<const float*>(&c), batch_views, lo[b], lo[b + 1]));
        }
        CK(cudaEventRecord(e[5], ctx->stream));
    }
    m->step_views = 0;
    ctx->bin_valid = false;  // the parameters moved
    if (ctx->prof.enabled) {
        CK(cudaStreamSynchronize(ctx->stream));
        ctx->pipe_timeline.assign(6 * (size_t)B, 0.f);
        for (int b = 0; b < B; ++b)
            for (int k = 0; k < 6; ++k) {
                if (!comm && (k == 2 || k == 3)) continue;
                float ms = 0.f;
                CK(cudaEventElapsedTime(&ms, ev[0], ev[1 + 6 * b + k]));
                ctx->pipe_timeline[6 * b + k] = ms;
            }
    }
    return TGSX_OK;
}

int32_t tgsx_pipeline_timeline(tgsx_ctx* ctx, float* out, int32_t max_floats) {
    if (!ctx) return -1;
    const int32_t n = (int32_t)ctx->pipe_timeline.size();
    if (out)
        for (int32_t i = 0; i < std::min(n, max_floats); ++i) out[i] = ctx->pipe_timeline[i];
    return n;
}

int32_t tgsx_set_binning(tgsx_ctx* ctx, int32_t mode) {
    if (!ctx || mode < 0 || mode > 1) return TGSX_EINVAL;
    ctx->binning_mode = mode;
    ctx->bin_valid = false;
    return TGSX_OK;
}

int32_t tgsx_set_ssim_weight(tgsx_ctx* ctx, float ssim_weight) {
    if (!ctx) return TGSX_EINVAL;
    if (!(ssim_weight >= 0.f && ssim_weight <= 1.f)) return fail(ctx, TGSX_EINVAL, "ssim weight must lie in [0, 1]");
    ctx->ssim_weight = ssim_weight;
    return TGSX_OK;
}

int32_t tgsx_loss(tgsx_ctx* ctx, const tgsx_pattern* pat, const float* rgb, const float* target,
                  float ssim_weight, float* out_loss, float* out_dLdC) {
    if (!ctx || !rgb || !target) return fail(ctx, TGSX_EINVAL, "loss: null input");
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    if (!(ssim_weight >= 0.f && ssim_weight <= 1.f)) return fail(ctx, TGSX_EINVAL, "ssim weight must lie in [0, 1]");
    RenderArgs ra = make_args(pat, nullptr, 0);
    const float lam = pat->p == 1 ? ssim_weight : 0.f;  // dilated iterations: L1 only
    Workspace& ws = ctx->ws;
    ws.have_forward = false;
    const float* d_rgb = nullptr;
    if ((rc = stage_input(ctx, ws.rgb, rgb, (size_t)std::max(ra.P, 1) * 12, &d_rgb))) return rc;
    if ((rc = stage_input(ctx, ws.target, target, (size_t)ra.W * ra.H * 12, &ra.target))) return rc;
    CK(ws.loss_grad.ensure((size_t)std::max(ra.P, 1) * 12));
    float* grad = ws.loss_grad.as<float>();
    const double inv = ra.P > 0 ? 1.0 / (3.0 * (double)ra.P) : 0.0;
    int n1 = 0, n2 = 0;
    CK(ws.block_loss.ensure((size_t)std::max<int64_t>((ra.P + 255) / 256, 1) * 4));
    CK(launch_l1(ctx, ra, d_rgb, (float)((1.0 - lam) * inv), grad, ws.block_loss.as<float>(), &n1));
    if (lam > 0.f && ra.P > 0) {
        n2 = (int)ssim_blocks(ra.W, ra.H);
        CK(ws.ssim_abc.ensure((size_t)ra.P * 36));
        CK(ws.ssim_part.ensure((size_t)n2 * 4));
        CK(launch_ssim(ctx, d_rgb, ra.target, ra.W, ra.H, lam, ws.ssim_abc.as<float>(),
                       ws.ssim_part.as<float>(), grad));
    }
    float* dloss = reinterpret_cast<float*>(ws.counters.as<unsigned long long>() + 4);
    CK(launch_loss_finalize(ctx, ws.block_loss.as<float>(), n1, (float)((1.0 - lam) * inv),
                            ws.ssim_part.as<float>(), n2, lam, inv, dloss));
    if (out_loss) CK(cudaMemcpyAsync(out_loss, dloss, 4, cudaMemcpyDefault, ctx->stream));
    if (out_dLdC && ra.P) CK(cudaMemcpyAsync(out_dLdC, grad, (size_t)ra.P * 12, cudaMemcpyDefault, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_apply_step(tgsx_ctx* ctx, tgsx_model* m, int32_t batch_views, const tgsx_adam_args* a) {
    if (!ctx || !m || !a) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (batch_views < 1) return fail(ctx, TGSX_EINVAL, "accumulate: empty batch");
    ctx->bin_valid = false;  // parameters change
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    AdamCfg c;
    fill_adam(c, a);
    {
        StageTimer t(ctx, kStAdam);
        CK(launch_adam(ctx, m, nullptr, reinterpret_cast<const float*>(&c), batch_views));
    }
    m->step_views = 0;
    return TGSX_OK;
}

// ---------------------------------------------------------------- stage access
int32_t tgsx_stage_prepare(tgsx_ctx* ctx, tgsx_model* m, int32_t lowpass_p, float* out, uint32_t* orig) {
    if (!ctx || !m || lowpass_p < 1) return fail(ctx, TGSX_EINVAL, "bad arguments");
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    ctx->bin_valid = false;
    CK(reset_counters(ctx));
    if (m->order_dirty) CK(launch_sort_depth(ctx, m));
    CK(launch_preprocess(ctx, m, lowpass_p, 16, 16));
    CK(cudaMemcpyAsync(ctx->ws.h_scratch, ctx->ws.counters.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    int32_t rc = check_kernel_error(ctx, ctx->ws.h_scratch[0]);
    if (rc) return rc;
    const int64_t n = m->n;
    if (!n) return TGSX_OK;
    std::vector<Prepared> hp(n);
    CK(cudaMemcpy(hp.data(), ctx->ws.prep.p, n * sizeof(Prepared), cudaMemcpyDeviceToHost));
    std::vector<float> o(11 * n);
    std::vector<uint32_t> og(n);
    for (int64_t r = 0; r < n; ++r) {
        const Prepared& p = hp[r];
        const float v[11] = {p.a.x, p.a.y, p.a.z, p.a.w, p.b.x, p.b.y, p.c.x, p.c.y, p.c.z, p.b.z, p.b.w};
        for (int q = 0; q < 11; ++q) o[q * n + r] = v[q];
        std::memcpy(&og[r], &p.c.w, 4);
    }
    if (out) CK(cudaMemcpy(out, o.data(), o.size() * 4, cudaMemcpyDefault));
    if (orig) CK(cudaMemcpy(orig, og.data(), og.size() * 4, cudaMemcpyDefault));
    return TGSX_OK;
}

int32_t tgsx_stage_sorted_order(tgsx_ctx* ctx, tgsx_model* m, uint32_t* perm) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    ctx->bin_valid = false;
    if (m->order_dirty) CK(launch_sort_depth(ctx, m));
    if (m->n && perm) CK(cudaMemcpyAsync(perm, m->perm.p, m->n * 4, cudaMemcpyDefault, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_stage_tile_lists(tgsx_ctx* ctx, tgsx_model* m, int32_t lowpass_p, int32_t width,
                              int32_t height, uint32_t* offsets, uint32_t* items,
                              int64_t items_cap, int64_t* out_k) {
    if (!ctx || !m || lowpass_p < 1 || width < 1 || height < 1) return fail(ctx, TGSX_EINVAL, "bad arguments");
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    uint32_t* it = nullptr;
    uint32_t* keys = nullptr;
    int32_t rc = bin(ctx, m, lowpass_p, width, height, &it, &keys);
    if (rc) return rc;
    const int64_t K = ctx->ws.K;
    if (out_k) *out_k = K;
    const int tiles = ctx->ws.tiles_x * ctx->ws.tiles_y;
    std::vector<uint2> rg(tiles);
    // the context stream is non-blocking: order the legacy-stream copies after bin()'s kernels
    CK(cudaStreamSynchronize(ctx->stream));
    if (tiles) CK(cudaMemcpy(rg.data(), ctx->ws.ranges.p, (size_t)tiles * sizeof(uint2), cudaMemcpyDeviceToHost));
    // per-tile ranges index the items buffer (per-tile slabs, or one contiguous array for the
    // onesweep path): gather them in tile order, checking blend order inside every tile
    size_t span = 0;
    for (int t = 0; t < tiles; ++t) {
        if (rg[t].y < rg[t].x) return fail(ctx, TGSX_ESTATE, "bad tile range at tile " + std::to_string(t));
        if (rg[t].y > rg[t].x) span = std::max<size_t>(span, rg[t].y);
    }
    std::vector<uint32_t> hi(span), flat;
    flat.reserve(K);
    if (span) CK(cudaMemcpy(hi.data(), it, span * 4, cudaMemcpyDeviceToHost));
    std::vector<uint32_t> off(tiles + 1, 0);
    for (int t = 0; t < tiles; ++t) {
        for (uint32_t s = rg[t].x; s < rg[t].y; ++s) {
            if (s > rg[t].x && hi[s] <= hi[s - 1])
                return fail(ctx, TGSX_ESTATE, "tile list not in blend order at tile " + std::to_string(t));
            flat.push_back(hi[s]);
        }
        off[t + 1] = off[t] + (rg[t].y - rg[t].x);
    }
    if (off[tiles] != (uint64_t)K) return fail(ctx, TGSX_ESTATE, "tile ranges do not cover the pairs");
    if (offsets) CK(cudaMemcpy(offsets, off.data(), off.size() * 4, cudaMemcpyDefault));
    if (items && items_cap >= K && K) CK(cudaMemcpy(items, flat.data(), K * 4, cudaMemcpyDefault));
    return TGSX_OK;
}

int32_t tgsx_stage_screen_grads(tgsx_ctx* ctx, tgsx_model* m, float* out) {
    if (!ctx || !m || !out) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    if (m->n) CK(cudaMemcpy2DAsync(out, m->n * 4, m->screen.p, m->cap * 4, m->n * 4, 10, cudaMemcpyDefault, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_stage_counters(tgsx_ctx* ctx, uint64_t* out_blend_ops, uint64_t* out_evals, uint64_t* out_pairs) {
    if (!ctx) return TGSX_EINVAL;
    CK(cudaMemcpyAsync(ctx->ws.h_scratch + 16, ctx->ws.counters.p, 4 * 8, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (out_blend_ops) *out_blend_ops = ctx->ws.h_scratch[17];
    if (out_evals) *out_evals = ctx->ws.h_scratch[18];
    if (out_pairs) *out_pairs = (uint64_t)ctx->ws.K;
    return TGSX_OK;
}

int32_t tgsx_sort_pairs(tgsx_ctx* ctx, uint32_t* keys, uint32_t* vals, int64_t n, int32_t key_bits) {
    if (!ctx || n < 0 || key_bits < 0 || key_bits > 32) return TGSX_EINVAL;
    ctx->bin_valid = false;  // shares the binning scratch
    if (n <= 1) return TGSX_OK;
    DevBuf& a = ctx->ws.generic;
    CK(a.ensure((size_t)n * 8));
    uint32_t* k2 = a.as<uint32_t>();
    uint32_t* v2 = k2 + n;
    uint32_t* k = keys;
    uint32_t* v = vals;
    CK(sort_pairs(ctx, k, v, k2, v2, n, key_bits, nullptr));
    if (k != keys) {
        CK(cudaMemcpyAsync(keys, k, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
        CK(cudaMemcpyAsync(vals, v, n * 4, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_exclusive_scan(tgsx_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n, uint64_t* out_total) {
    if (!ctx || n < 0) return TGSX_EINVAL;
    ctx->bin_valid = false;  // shares the binning scratch
    uint32_t* d_total = reinterpret_cast<uint32_t*>(ctx->ws.counters.as<unsigned long long>() + 5);
    CK(launch_exclusive_scan(ctx, in, out, n, d_total));
    CK(cudaMemcpyAsync(ctx->ws.h_scratch + 24, d_total, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (out_total) *out_total = n ? (uint64_t)(uint32_t)ctx->ws.h_scratch[24] : 0;
    return TGSX_OK;
}

// ---------------------------------------------------------------- 3-D front end (A3b)
int32_t tgsx_model3d_create(tgsx_ctx* ctx, int64_t capacity, tgsx_model3d** out) {
    if (!ctx || !out || capacity < 0) return TGSX_EINVAL;
    tgsx_model3d* m = new tgsx_model3d();
    cudaError_t e = model3d_reserve(ctx, m, std::max<int64_t>(capacity, 1), false);
    if (e) {
        delete m;
        return cuda_fail(ctx, e, "tgsx_model3d_create");
    }
    *out = m;
    return TGSX_OK;
}

void tgsx_model3d_destroy(tgsx_model3d* m) {
    if (!m) return;
    DevBuf* bufs[] = {&m->params, &m->m1,    &m->m2,       &m->pos_acc,   &m->col_acc, &m->visit,
                      &m->perm,   &m->rank_of, &m->prep_row, &m->gbuf,      &m->step,    &m->skeys,
                      &m->ids,    &m->tau_v, &m->visit_evt, &m->visit_aud};
    for (DevBuf* b : bufs) b->release();
    for (DevBuf& b : m->spare) b.release();
    delete m;
}

int64_t tgsx_model3d_size(const tgsx_model3d* m) { return m ? m->n : 0; }

int32_t tgsx_model3d_reserve(tgsx_ctx* ctx, tgsx_model3d* m, int64_t capacity) {
    if (!ctx || !m || capacity < 0) return TGSX_EINVAL;
    if (int32_t rc_ = tgsx::graph_flush(ctx)) return rc_;
    ctx->bin_valid = false;
    CK(model3d_reserve(ctx, m, capacity, true));
    // the prune compaction's spare row buffers (densify3d.cu, same order and sizes), allocated now
    // instead of inside the first densify event (a GB-scale cudaMalloc in the middle of a fit)
    const int rows[10] = {k3dParams, k3dParams, k3dParams, 1, 1, 1, 1, 1, 1, 1};
    const int elt[10] = {4, 4, 4, 4, 4, 4, 4, 4, 8, 8};
    for (int i = 0; i < 10; ++i) {
        DevBuf& sp = m->spare[i];
        const size_t bytes = (size_t)rows[i] * m->cap * elt[i];
        if (sp.bytes < bytes) {
            CK(cudaStreamSynchronize(ctx->stream));
            sp.release();
            CK(cudaMalloc(&sp.p, bytes));
            sp.bytes = bytes;
        }
    }
    return TGSX_OK;
}

int32_t tgsx_model3d_upload(tgsx_ctx* ctx, tgsx_model3d* m, const float* params, int64_t n) {
    if (!ctx || !m || n < 0 || (n && !params)) return fail(ctx, TGSX_EINVAL, "bad 3-D upload arguments");
    ctx->bin_valid = false;
    CK(model3d_reserve(ctx, m, n, false));
    m->n = n;
    cudaStream_t s = ctx->stream;
    const int64_t cap = m->cap;
    if (n) CK(cudaMemcpy2DAsync(m->params.p, cap * 4, params, n * 4, n * 4, k3dParams, cudaMemcpyDefault, s));
    CK(cudaMemsetAsync(m->m1.p, 0, m->m1.bytes, s));
    CK(cudaMemsetAsync(m->m2.p, 0, m->m2.bytes, s));
    CK(cudaMemsetAsync(m->pos_acc.p, 0, m->pos_acc.bytes, s));
    CK(cudaMemsetAsync(m->col_acc.p, 0, m->col_acc.bytes, s));
    CK(cudaMemsetAsync(m->visit.p, 0, m->visit.bytes, s));
    CK(cudaMemsetAsync(m->step.p, 0, m->step.bytes, s));
    CK(cudaMemsetAsync(m->visit_evt.p, 0, m->visit_evt.bytes, s));
    CK(cudaMemsetAsync(m->visit_aud.p, 0, m->visit_aud.bytes, s));
    CK(densify3d_init_rows(ctx, m, 0, n));  // ids 0..n-1, tau_v = tau_v_init default
    m->next_id = (uint64_t)n;
    m->step_views = 0;
    CK(cudaStreamSynchronize(s));
    return TGSX_OK;
}

int32_t tgsx_model3d_download(tgsx_ctx* ctx, tgsx_model3d* m, float* params, float* pos_acc,
                              float* col_acc, int32_t* visits) {
    if (!ctx || !m) return TGSX_EINVAL;
    const int64_t n = m->n, cap = m->cap;
    cudaStream_t s = ctx->stream;
    if (n) {
        if (params) CK(cudaMemcpy2DAsync(params, n * 4, m->params.p, cap * 4, n * 4, k3dParams, cudaMemcpyDefault, s));
        if (pos_acc) CK(cudaMemcpyAsync(pos_acc, m->pos_acc.p, n * 4, cudaMemcpyDefault, s));
        if (col_acc) CK(cudaMemcpyAsync(col_acc, m->col_acc.p, n * 4, cudaMemcpyDefault, s));
        if (visits) CK(cudaMemcpyAsync(visits, m->visit.p, n * 4, cudaMemcpyDefault, s));
    }
    CK(cudaStreamSynchronize(s));
    return TGSX_OK;
}

int32_t tgsx_model3d_download_moments(tgsx_ctx* ctx, tgsx_model3d* m, float* m1, float* m2) {
    if (!ctx || !m) return TGSX_EINVAL;
    const int64_t n = m->n, cap = m->cap;
    if (n) {
        if (m1) CK(cudaMemcpy2DAsync(m1, n * 4, m->m1.p, cap * 4, n * 4, k3dParams, cudaMemcpyDefault, ctx->stream));
        if (m2) CK(cudaMemcpy2DAsync(m2, n * 4, m->m2.p, cap * 4, n * 4, k3dParams, cudaMemcpyDefault, ctx->stream));
    }
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_render3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                      const float bg[3], int32_t lowpass_p, float* out_rgb, float* out_T,
                      uint64_t* out_blend_ops) {
    if (!ctx || !m) return TGSX_EINVAL;
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    Cam3 c3;
    if ((rc = make_cam3(ctx, cam, pat, &c3))) return rc;
    RenderArgs ra = make_args(pat, bg, lowpass_p);
    uint32_t* items = nullptr;
    if ((rc = render3d_core(ctx, m, c3, ra, false, &items))) return rc;
    Workspace& ws = ctx->ws;
    if (out_rgb && ra.P) CK(cudaMemcpyAsync(out_rgb, ws.rgb.p, (size_t)ra.P * 12, cudaMemcpyDefault, ctx->stream));
    if (out_T && ra.P) CK(cudaMemcpyAsync(out_T, ws.T.p, (size_t)ra.P * 4, cudaMemcpyDefault, ctx->stream));
    if (out_blend_ops)
        CK(cudaMemcpyAsync(ws.h_scratch + 8, ws.counters.as<unsigned long long>() + 1, 8,
                           cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    if (out_blend_ops) *out_blend_ops = ws.h_scratch[8];
    return TGSX_OK;
}

int32_t tgsx_backward3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                        const float bg[3], int32_t lowpass_p, const float* dLdC, int64_t dLdC_count,
                        float* out_grads, float* out_screen, int32_t update_stats) {
    if (!ctx || !m || !dLdC) return TGSX_EINVAL;
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    Cam3 c3;
    if ((rc = make_cam3(ctx, cam, pat, &c3))) return rc;
    RenderArgs ra = make_args(pat, bg, lowpass_p);
    if (dLdC_count != ra.P)
        return fail(ctx, TGSX_EINVAL, "backward3d: loss-gradient count does not match pattern ranks");
    uint32_t* items = nullptr;
    if ((rc = render3d_core(ctx, m, c3, ra, false, &items))) return rc;
    Workspace& ws = ctx->ws;
    if (ra.P) CK(cudaMemcpyAsync(ws.dLdC.p, dLdC, (size_t)ra.P * 12, cudaMemcpyDefault, ctx->stream));
    {
        StageTimer t(ctx, kStBackward);
        CK(launch_backward(ctx, ra, items));
    }
    const int64_t n = m->n;
    const size_t gbytes = (size_t)std::max<int64_t>(n, 1) * k3dParams * 4;
    const size_t sbytes = (size_t)std::max<int64_t>(n, 1) * 10 * 4;
    CK(ws.generic.ensure(gbytes + sbytes));
    float* gdev = (out_grads && is_device_ptr(out_grads)) ? out_grads : ws.generic.as<float>();
    float* sdev = out_screen ? (is_device_ptr(out_screen) ? out_screen : ws.generic.as<float>() + gbytes / 4)
                             : nullptr;
    {
        StageTimer t(ctx, kStChain);
        CK(launch_chain3d(ctx, m, c3, ra.lowpass_p, 0, update_stats != 0, gdev, sdev, nullptr));
    }
    if (out_grads && gdev != out_grads && n)
        CK(cudaMemcpyAsync(out_grads, gdev, (size_t)n * k3dParams * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (out_screen && sdev != out_screen && n)
        CK(cudaMemcpyAsync(out_screen, sdev, (size_t)n * 40, cudaMemcpyDeviceToHost, ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

int32_t tgsx_adam3d_step(tgsx_ctx* ctx, tgsx_model3d* m, const float* grads, const tgsx_adam3d_args* a) {
    if (!ctx || !m || !grads || !a) return TGSX_EINVAL;
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    Adam3dCfg c;
    fill_adam3d(c, a);
    const float* g = nullptr;
    int32_t rc = stage_input(ctx, ctx->ws.generic, grads, (size_t)std::max<int64_t>(m->n, 1) * k3dParams * 4, &g);
    if (rc) return rc;
    CK(launch_adam3d(ctx, m, g, c));
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

static int32_t fused_view3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                            const float bg[3], const float* target, const tgsx_adam3d_args* a, float* out_loss,
                            int mode);

int32_t tgsx_fit_step3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                        const float bg[3], const float* target, const tgsx_adam3d_args* a, float* out_loss) {
    if (!ctx || !m || !a) return TGSX_EINVAL;
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    return fused_view3d(ctx, m, cam, pat, bg, target, a, out_loss, 1);
}

int32_t tgsx_view_accumulate3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                               const float bg[3], const float* target, float* out_loss) {
    if (!ctx || !m) return TGSX_EINVAL;
    const int32_t rc = fused_view3d(ctx, m, cam, pat, bg, target, nullptr, out_loss, 2);
    if (!rc) m->step_views++;
    return rc;
}

float* tgsx_step_buffer3d(tgsx_model3d* m, int64_t* out_floats) {
    if (!m) return nullptr;
    if (out_floats) *out_floats = (int64_t)k3dStepRows * m->n;  // packed [62][n]
    return m->step.as<float>();
}

// In-place sum of the packed [62][n] 3-D step buffer over the attached communicator (rows stay in
// creation order on every rank: no layout step is needed).
int32_t tgsx_allreduce_step3d(tgsx_ctx* ctx, tgsx_model3d* m) {
    if (!ctx || !m) return TGSX_EINVAL;
    if (!ctx->comm) return fail(ctx, TGSX_ESTATE, "no communicator attached (tgsx_comm_init)");
    if (ctx->pipe_events.size() < 2) {
        for (auto& e : ctx->pipe_events) cudaEventDestroy(e);
        ctx->pipe_events.assign(2, nullptr);
        for (auto& e : ctx->pipe_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->pipe_events[0], ctx->stream));
    CK(cudaStreamWaitEvent(ctx->comm_stream, ctx->pipe_events[0], 0));
    int32_t rc = comm_allreduce_sum(ctx, m->step.as<float>(), (size_t)k3dStepRows * m->n, ctx->comm_stream);
    if (rc) return rc;
    CK(cudaEventRecord(ctx->pipe_events[1], ctx->comm_stream));
    CK(cudaStreamWaitEvent(ctx->stream, ctx->pipe_events[1], 0));
    return TGSX_OK;
}

int32_t tgsx_apply_step3d(tgsx_ctx* ctx, tgsx_model3d* m, int32_t batch_views, const tgsx_adam3d_args* a) {
    if (!ctx || !m || !a) return TGSX_EINVAL;
    if (a->step < 1) return fail(ctx, TGSX_EINVAL, "adam step must be >= 1");
    if (batch_views < 1) return fail(ctx, TGSX_EINVAL, "batch_views must be >= 1");
    Adam3dCfg cfg;
    fill_adam3d(cfg, a);
    CK(launch_adam3d_step(ctx, m, batch_views, cfg));
    m->step_views = 0;
    return TGSX_OK;  // stream-ordered: no host sync per step
}

// One 3-D view: render + fused L1 (+ SSIM on dense views) + backward + chain3d in `mode`
// (1 fused Adam, 2 accumulate into the step buffer).
static int32_t fused_view3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, const tgsx_pattern* pat,
                            const float bg[3], const float* target, const tgsx_adam3d_args* a, float* out_loss,
                            int mode) {
    int32_t rc = check_pattern(ctx, pat);
    if (rc) return rc;
    if (!target) return fail(ctx, TGSX_EINVAL, "target is null");
    Cam3 c3;
    if ((rc = make_cam3(ctx, cam, pat, &c3))) return rc;
    Adam3dCfg cfg{};
    if (a) fill_adam3d(cfg, a);
    RenderArgs ra = make_args(pat, bg, 0);
    const float lam = (pat->p == 1 && ctx->ssim_weight > 0.f) ? ctx->ssim_weight : 0.f;
    ra.l1_weight = 1.0f - lam;
    Workspace& ws = ctx->ws;
    if ((rc = stage_target(ctx, target, (size_t)ra.W * ra.H * 12, &ra.target, &ra))) return rc;
    uint32_t* items = nullptr;
    if ((rc = render3d_core(ctx, m, c3, ra, true, &items, true))) return rc;
    int nsb = 0;
    if (lam > 0.f && ra.P > 0) {
        StageTimer t(ctx, kStLoss);
        nsb = (int)ssim_blocks(ra.W, ra.H);
        CK(ws.ssim_abc.ensure((size_t)ra.P * 36));
        CK(ws.ssim_part.ensure((size_t)nsb * 4));
        CK(launch_ssim(ctx, ws.rgb.as<float>(), ra.target, ra.W, ra.H, lam, ws.ssim_abc.as<float>(),
                       ws.ssim_part.as<float>(), ws.dLdC.as<float>()));
    }
    if ((rc = mark_target_consumed(ctx))) return rc;
    {
        StageTimer t(ctx, kStBackward);
        CK(launch_backward(ctx, ra, items));
    }
    {
        StageTimer t(ctx, kStChain);
        CK(launch_chain3d(ctx, m, c3, ra.lowpass_p, mode, true, nullptr, nullptr, &cfg));
    }
    const int tiles = ws.tiles_x * ws.tiles_y;
    float* dloss = reinterpret_cast<float*>(ws.counters.as<unsigned long long>() + 4);
    {
        StageTimer t(ctx, kStLoss);
        const double inv = ra.P > 0 ? 1.0 / (3.0 * (double)ra.P) : 0.0;
        CK(launch_loss_finalize(ctx, ws.block_loss.as<float>(), tiles, (float)((1.0 - lam) * inv),
                                ws.ssim_part.as<float>(), nsb, lam, inv, dloss));
    }
    if (out_loss) {
        CK(cudaMemcpyAsync(out_loss, dloss, 4, cudaMemcpyDefault, ctx->stream));
        if (!is_device_ptr(out_loss) && !is_pinned_host_ptr(out_loss)) CK(cudaStreamSynchronize(ctx->stream));
    }
    return TGSX_OK;
}

int32_t tgsx_stage_prepare3d(tgsx_ctx* ctx, tgsx_model3d* m, const tgsx_camera* cam, int32_t lowpass_p,
                             float* out_records, uint32_t* out_keys, int32_t* out_blend_ordered) {
    if (!ctx || !m || lowpass_p < 1) return TGSX_EINVAL;
    Cam3 c3;
    int32_t rc = make_cam3(ctx, cam, nullptr, &c3);
    if (rc) return rc;
    uint32_t* items = nullptr;
    if ((rc = bin3d(ctx, m, c3, lowpass_p, cam->width, cam->height, &items))) return rc;
    const int64_t n = m->n;
    if (n && out_records) CK(cudaMemcpyAsync(out_records, ctx->ws.prep.p, (size_t)n * sizeof(Prepared),
                                             cudaMemcpyDefault, ctx->stream));
    // depth keys in the records' order (culled rows: key 0xffffffff)
    if (n && out_keys)
        CK(cudaMemcpyAsync(out_keys, m->rank_ordered ? m->skeys.p : ctx->ws.keys[0].p, (size_t)n * 4,
                           cudaMemcpyDefault, ctx->stream));
    if (out_blend_ordered) *out_blend_ordered = m->rank_ordered ? 1 : 0;
    CK(cudaStreamSynchronize(ctx->stream));
    return TGSX_OK;
}

}  // extern "C"
