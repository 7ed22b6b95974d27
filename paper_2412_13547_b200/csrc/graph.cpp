// CUDA-graph replay of the fused fit step (tgsx_fit_graph_step).
//
// The eager step (tgsx_fit_step) is ~10 launches plus one host wait for the binning counters (the
// pair count K sizes the partials, the longest list picks the per-tile sort). For small views
// (C1: 10K Gaussians at 256², tens of microseconds of GPU work) the launches and that wait are
// the step. Here the step is captured once into a graph and replayed with one cudaGraphLaunch:
//
//  * The host decisions of the eager step are frozen at capture: the per-tile sort handles lists
//    up to the capture-time cap, the partial buffer holds 1.25x the capture-time K. The blend
//    backward checks the step's counters against them ON THE DEVICE (and the kernel error word);
//    a violation sets a sticky fault word that turns the backward and the chain + Adam of this
//    and every later replayed step into no-ops (the model is untouched).
//  * Replays are verified one step behind (at most two in flight): before slot s is reused, the
//    step that last used it is waited for and the fault word copied after it (a node of the
//    graph, one pinned word per slot) is read. The first faulted step and the one after it are
//    re-run eagerly in order, the fault cleared and the graph recaptured on the next call, so
//    the sequence of model updates is exactly that of eager steps.
//  * Per-step arguments: the Adam hyper-parameters (step count, learning-rate decay) are set on
//    the captured chain kernel node, the loss destination on the captured loss-copy node and the
//    target on the captured target-copy node (the graph stages the target — only the active
//    rows of a dilated view — into the workspace) of the exec before each launch; everything
//    else (pattern, background, SSIM weight, memory types, model and workspace buffers, sizes)
//    is part of the key the graph was captured for — a different key re-runs eagerly and
//    recaptures.
//
// Every other entry point that reads or changes the model first calls graph_flush, so callers
// observe the same state as after eager steps. Targets passed to replayed steps must stay
// unchanged until the step after next returns (a faulted step is re-run from them).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <utility>
#include <vector>

#include "tgsx_internal.h"

namespace tgsx {

namespace {

// One captured step (per key: a dilated fit cycling p x p offsets keeps p^2 of them).
struct Entry {
    std::vector<uintptr_t> key;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec[2] = {nullptr, nullptr};  // per slot: the fault copy goes to h_fault[slot]
    cudaGraphNode_t chain = nullptr;
    cudaGraphNode_t loss = nullptr;  // the out_loss copy (destination set per replay)
    const void* loss_src = nullptr;
    cudaGraphNode_t target = nullptr;  // the target staging into the workspace (source set per replay)
    int target_kind = 0;               // 1: 1-D memcpy node, 2: stage-rows kernel node
    cudaMemcpy3DParms target_parms{};
    cudaKernelNodeParams target_kernel{};
    StageRowsArgs target_args{};
    int64_t target_off = 0;
    uint64_t kernels = 0;  // kernel launches per replay (counted at capture)
    uint64_t used = 0;     // last use (LRU)
    void release() {
        for (auto& e : exec)
            if (e) cudaGraphExecDestroy(e), e = nullptr;
        if (graph) cudaGraphDestroy(graph), graph = nullptr;
    }
};
constexpr size_t kMaxEntries = 16;

struct FitGraph {
    std::vector<Entry> entries;
    cudaEvent_t done[2] = {nullptr, nullptr};
    struct Pending {
        bool live = false;
        uint64_t seq = 0;
        tgsx_model* m = nullptr;
        tgsx_pattern pat{};
        float bg[3] = {0, 0, 0};
        const float* target = nullptr;
        tgsx_adam_args a{};
        float* out_loss = nullptr;
        float ssim_weight = 0.f;
    } pend[2];
    uint64_t seq = 0;
    uint64_t captures = 0, replays = 0, reruns = 0;
    // per model (uid): the first device target replayed, and whether the model's fit has seen a
    // second one (its graphs then stage the target through a node with a per-replay source)
    struct TargetUse {
        uint64_t uid;
        const float* first;
        bool staging;
    };
    std::vector<TargetUse> targets;

    void drop_graphs() {
        for (auto& e : entries) e.release();
        entries.clear();
    }
};

FitGraph* get(tgsx_ctx* ctx) {
    if (!ctx->graph) ctx->graph = new FitGraph();
    return static_cast<FitGraph*>(ctx->graph);
}

int32_t cuda_err(tgsx_ctx* ctx, cudaError_t e, const char* where) {
    ctx->err = std::string(where) + ": " + cudaGetErrorString(e);
    return TGSX_ECUDA;
}
#define GK(expr)                                         \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) return cuda_err(ctx, _e, #expr); \
    } while (0)

cudaMemoryType mem_type(const void* p) {
    if (!p) return cudaMemoryTypeUnregistered;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return cudaMemoryTypeUnregistered;
    }
    return at.type;
}

template <typename T>
void put(std::vector<uintptr_t>& k, T v) {
    uintptr_t u = 0;
    static_assert(sizeof(T) <= sizeof(uintptr_t), "key field too wide");
    std::memcpy(&u, &v, sizeof(T));
    k.push_back(u);
}

// Everything the eager step's launch sequence depends on besides the device data.
bool device_or_pinned(cudaMemoryType t) {
    return t == cudaMemoryTypeDevice || t == cudaMemoryTypeManaged || t == cudaMemoryTypeHost;
}

// (target / loss memory types are looked up once per call by the caller)
std::vector<uintptr_t> make_key(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                                const float* target, float* out_loss, cudaMemoryType tt, cudaMemoryType lt) {
    std::vector<uintptr_t> k;
    put(k, m);
    put(k, m->uid);
    put(k, m->n);
    put(k, m->cap);
    put(k, (int)m->blend_phys + 2 * (int)m->order_dirty + 4 * (int)m->spatial_valid);
    put(k, m->spatial.p);
    for (const DevBuf* b : {&m->params, &m->ids, &m->pos_acc, &m->col_acc, &m->accum, &m->visit, &m->window,
                            &m->tau_v, &m->m1, &m->m2, &m->step, &m->perm, &m->rank_of, &m->screen})
        put(k, b->p);
    const Workspace& ws = ctx->ws;
    for (const DevBuf* b : {&ws.prep, &ws.touched, &ws.pair_off, &ws.rect, &ws.scan_tmp, &ws.ranges, &ws.tile_fill,
                            &ws.tile_slab, &ws.partial, &ws.rgb, &ws.T, &ws.last, &ws.dLdC, &ws.target,
                            &ws.block_loss, &ws.ssim_abc, &ws.ssim_part, &ws.counters})
        put(k, b->p);
    put(k, ws.pair_cap);
    put(k, ws.h_scratch);
    put(k, pat->p);
    put(k, pat->ox);
    put(k, pat->oy);
    put(k, pat->width);
    put(k, pat->height);
    for (int i = 0; i < 3; ++i) put(k, bg[i]);
    // a staged target (pinned host, or any target once several device targets were seen) is a
    // per-replay argument; a device target read in place is part of the key
    if (tt == cudaMemoryTypeDevice && !ctx->graph_stage_targets) put(k, target);
    else put(k, 1 + (int)tt);
    put(k, ctx->graph_stage_targets);
    // the loss destination is a per-replay argument; its memory type is fixed by the copy node
    put(k, out_loss ? 1 + (int)lt : 0);
    put(k, ctx->ssim_weight);
    put(k, ctx->binning_mode);
    put(k, ctx->stream);
    return k;
}

// Re-runs the live steps from slot s on (in sequence order) eagerly after a fault.
int32_t rerun_from(tgsx_ctx* ctx, FitGraph& G, int s) {
    GK(cudaStreamSynchronize(ctx->stream));
    std::vector<FitGraph::Pending> todo;
    for (int i = 0; i < 2; ++i)
        if (G.pend[i].live && G.pend[i].seq >= G.pend[s].seq) todo.push_back(G.pend[i]);
    if (todo.size() == 2 && todo[0].seq > todo[1].seq) std::swap(todo[0], todo[1]);
    for (auto& p : G.pend) p.live = false;
    GK(cudaMemsetAsync(ctx->graph_fault, 0, sizeof(unsigned), ctx->stream));
    G.drop_graphs();  // outgrown capacities (or a kernel error): recapture on the next call
    ctx->graph_replaying = true;
    const float w0 = ctx->ssim_weight;
    int32_t rc = TGSX_OK;
    for (auto& p : todo) {
        G.reruns++;
        ctx->ssim_weight = p.ssim_weight;  // the weight the replayed step was captured with
        rc = tgsx_fit_step(ctx, p.m, &p.pat, p.bg, p.target, &p.a, p.out_loss);
        if (rc) break;
    }
    ctx->ssim_weight = w0;
    ctx->graph_replaying = false;
    return rc;
}

// Verifies live replayed steps in order; keep_one: leave the newest in flight.
int32_t check(tgsx_ctx* ctx, FitGraph& G, bool keep_one) {
    for (;;) {
        int s = -1, live = 0;
        for (int i = 0; i < 2; ++i) {
            if (!G.pend[i].live) continue;
            ++live;
            if (s < 0 || G.pend[i].seq < G.pend[s].seq) s = i;
        }
        if (s < 0 || (keep_one && live < 2)) return TGSX_OK;
        GK(cudaEventSynchronize(G.done[s]));
        if (ctx->h_graph_fault[s] == 0u) {
            G.pend[s].live = false;
            continue;
        }
        return rerun_from(ctx, G, s);
    }
}

int32_t capture(tgsx_ctx* ctx, FitGraph& G, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                const float* target, const tgsx_adam_args* a, float* out_loss) {
    Workspace& ws = ctx->ws;
    // headroom over the capture-time pair count (the fit moves splats; the backward guards it).
    // TGSX_GRAPH_PAIR_SLACK overrides it (tests: a negative slack faults every replay)
    int64_t slack = ws.K / 4 + 1024;
    if (const char* e = std::getenv("TGSX_GRAPH_PAIR_SLACK")) slack = std::strtoll(e, nullptr, 10);
    const int64_t want = std::max<int64_t>(ws.K + slack, 1);
    if (ws.pair_cap < want) {
        GK(cudaStreamSynchronize(ctx->stream));
        GK(ws.partial.ensure((size_t)want * 40));
        ws.pair_cap = (int64_t)(ws.partial.bytes / 40);
        G.drop_graphs();  // the partial buffer moved
    }
    ctx->graph_guard_pairs = want;
    if (!ctx->graph_fault) {
        GK(cudaMalloc(&ctx->graph_fault, sizeof(unsigned)));
        GK(cudaHostAlloc(&ctx->h_graph_fault, 2 * sizeof(unsigned), cudaHostAllocDefault));
        ctx->h_graph_fault[0] = ctx->h_graph_fault[1] = 0u;
        GK(cudaMemsetAsync(ctx->graph_fault, 0, sizeof(unsigned), ctx->stream));
    }
    for (auto& e : G.done)
        if (!e) GK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    // the host target lands in ws.target inside the graph: size it outside the capture
    const size_t tbytes = (size_t)pat->width * pat->height * 12;
    if (ws.target.bytes < tbytes) {
        GK(cudaStreamSynchronize(ctx->stream));
        GK(ws.target.ensure(tbytes));
        G.drop_graphs();
    }
    GK(cudaStreamSynchronize(ctx->stream));

    const uint64_t launches0 = ctx->launches;
    GK(cudaStreamBeginCapture(ctx->stream, cudaStreamCaptureModeThreadLocal));
    ctx->graph_capturing = true;
    ctx->graph_chain_node = nullptr;
    ctx->graph_loss_node = nullptr;
    ctx->graph_target_node = nullptr;
    ctx->graph_target_kind = 0;
    int32_t rc = tgsx_fit_step(ctx, m, pat, bg, target, a, out_loss);
    cudaGraphNode_t fault_copy = nullptr;
    if (!rc) {
        cudaError_t e = cudaMemcpyAsync(ctx->h_graph_fault, ctx->graph_fault, sizeof(unsigned),
                                        cudaMemcpyDeviceToHost, ctx->stream);
        cudaStreamCaptureStatus st;
        const cudaGraphNode_t* deps = nullptr;
        size_t nd = 0;
        if (!e) e = cudaStreamGetCaptureInfo(ctx->stream, &st, nullptr, nullptr, &deps, &nd);
        if (!e && nd == 1) fault_copy = deps[0];
        if (e) rc = cuda_err(ctx, e, "graph capture");
    }
    ctx->graph_capturing = false;
    cudaGraph_t g = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(ctx->stream, &g);
    const uint64_t kernels = ctx->launches - launches0;
    ctx->launches = launches0;
    if (rc || ee || !g || !fault_copy || !ctx->graph_chain_node || (out_loss && !ctx->graph_loss_node)) {
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        return rc ? rc : (ee ? cuda_err(ctx, ee, "cudaStreamEndCapture") : TGSX_OK);
    }
    if (G.entries.size() >= kMaxEntries) {  // evict the least recently used
        size_t lru = 0;
        for (size_t i = 1; i < G.entries.size(); ++i)
            if (G.entries[i].used < G.entries[lru].used) lru = i;
        G.entries[lru].release();
        G.entries.erase(G.entries.begin() + (long)lru);
    }
    Entry en;
    en.graph = g;
    en.chain = static_cast<cudaGraphNode_t>(ctx->graph_chain_node);
    en.loss = out_loss ? static_cast<cudaGraphNode_t>(ctx->graph_loss_node) : nullptr;
    en.loss_src = ctx->graph_loss_src;
    en.target = static_cast<cudaGraphNode_t>(ctx->graph_target_node);
    en.target_off = ctx->graph_target_off;
    en.target_kind = en.target ? ctx->graph_target_kind : 0;
    en.target_args = ctx->graph_stage_args;
    cudaError_t e = cudaSuccess;
    if (en.target_kind == 1) e = cudaGraphMemcpyNodeGetParams(en.target, &en.target_parms);
    if (en.target_kind == 2) e = cudaGraphKernelNodeGetParams(en.target, &en.target_kernel);
    en.kernels = kernels;
    en.used = G.seq;
    if (!e) e = cudaGraphInstantiate(&en.exec[0], g, 0);
    if (!e) e = cudaGraphInstantiate(&en.exec[1], g, 0);
    if (!e)
        e = cudaGraphExecMemcpyNodeSetParams1D(en.exec[1], fault_copy, ctx->h_graph_fault + 1, ctx->graph_fault,
                                               sizeof(unsigned), cudaMemcpyDeviceToHost);
    if (!e) e = cudaGraphUpload(en.exec[0], ctx->stream);
    if (!e) e = cudaGraphUpload(en.exec[1], ctx->stream);
    if (e) {
        en.release();
        return cuda_err(ctx, e, "graph instantiate");
    }
    en.key = make_key(ctx, m, pat, bg, target, out_loss, mem_type(target), mem_type(out_loss));
    G.entries.push_back(std::move(en));
    G.captures++;
    return TGSX_OK;
}

}  // namespace

int32_t graph_flush(tgsx_ctx* ctx) {
    if (!ctx || !ctx->graph || ctx->graph_capturing || ctx->graph_replaying) return TGSX_OK;
    return check(ctx, *static_cast<FitGraph*>(ctx->graph), false);
}

void graph_release(tgsx_ctx* ctx) {
    if (!ctx) return;
    if (ctx->graph) {
        FitGraph* G = static_cast<FitGraph*>(ctx->graph);
        G->drop_graphs();
        for (auto& e : G->done)
            if (e) cudaEventDestroy(e);
        delete G;
        ctx->graph = nullptr;
    }
    if (ctx->graph_fault) cudaFree(ctx->graph_fault);
    if (ctx->h_graph_fault) cudaFreeHost(ctx->h_graph_fault);
    ctx->graph_fault = nullptr;
    ctx->h_graph_fault = nullptr;
}

}  // namespace tgsx

using namespace tgsx;

extern "C" {

int32_t tgsx_fit_graph_step(tgsx_ctx* ctx, tgsx_model* m, const tgsx_pattern* pat, const float bg[3],
                            const float* target, const tgsx_adam_args* a, float* out_loss) {
    if (!ctx || !m || !a || !pat || !bg) return TGSX_EINVAL;
    if (ctx->graph_capturing || ctx->graph_replaying) return TGSX_ESTATE;
    FitGraph& G = *get(ctx);
    const int slot = (int)(G.seq & 1);
    int32_t rc = check(ctx, G, true);  // retires the step that last used `slot`
    if (rc) return rc;
    const cudaMemoryType tt = mem_type(target), lt = mem_type(out_loss);
    const bool eligible = target && m->n > 0 && !ctx->prof.enabled && graph_eligible_binning(ctx) &&
                          device_or_pinned(tt) && (!out_loss || device_or_pinned(lt));
    if (!eligible) {
        if ((rc = check(ctx, G, false))) return rc;
        return tgsx_fit_step(ctx, m, pat, bg, target, a, out_loss);
    }
    // a model's second device target: from now on its targets are staged by a graph node
    // (per-replay source) instead of being part of the key, so a multi-view fit keeps one graph
    // per pattern (a single-target fit reads its target in place, no copy)
    FitGraph::TargetUse* tu = nullptr;
    for (auto& u : G.targets)
        if (u.uid == m->uid) tu = &u;
    if (!tu) {
        if (G.targets.size() >= 64) G.targets.erase(G.targets.begin());
        G.targets.push_back({m->uid, nullptr, false});
        tu = &G.targets.back();
    }
    if (!tu->staging && tt == cudaMemoryTypeDevice) {
        if (!tu->first) {
            tu->first = target;
        } else if (target != tu->first) {
            if ((rc = check(ctx, G, false))) return rc;
            tu->staging = true;
        }
    }
    ctx->graph_stage_targets = tu->staging;
    const std::vector<uintptr_t> key = make_key(ctx, m, pat, bg, target, out_loss, tt, lt);
    Entry* en = nullptr;
    for (auto& e : G.entries)
        if (e.key == key) en = &e;
    if (!en) {
        if ((rc = check(ctx, G, false))) return rc;
        // eager step (settles the binning sizes), then capture the step for the next calls
        if ((rc = tgsx_fit_step(ctx, m, pat, bg, target, a, out_loss))) return rc;
        if (!graph_eligible_binning(ctx)) return TGSX_OK;
        return capture(ctx, G, m, pat, bg, target, a, out_loss);
    }
    if (a->step < 1) {
        ctx->err = "adam step must be >= 1";
        return TGSX_EINVAL;
    }
    AdamCfg c;
    adam_cfg_from_args(c, a);
    GK(chain_node_set_adam(en->exec[slot], en->chain, c));
    if (en->loss)
        GK(cudaGraphExecMemcpyNodeSetParams1D(en->exec[slot], en->loss, out_loss, en->loss_src, 4,
                                              cudaMemcpyDefault));
    if (en->target_kind == 1) {
        cudaMemcpy3DParms tp = en->target_parms;
        tp.srcPtr.ptr = const_cast<float*>(target + en->target_off);
        GK(cudaGraphExecMemcpyNodeSetParams(en->exec[slot], en->target, &tp));
    } else if (en->target_kind == 2) {
        StageRowsArgs sa = en->target_args;
        sa.src = target + en->target_off;
        void* args[1] = {&sa};
        cudaKernelNodeParams kp = en->target_kernel;
        kp.kernelParams = args;
        kp.extra = nullptr;
        GK(cudaGraphExecKernelNodeSetParams(en->exec[slot], en->target, &kp));
    }
    GK(cudaGraphLaunch(en->exec[slot], ctx->stream));
    GK(cudaEventRecord(G.done[slot], ctx->stream));
    en->used = G.seq;
    ctx->launches += en->kernels;
    FitGraph::Pending& p = G.pend[slot];
    p.live = true;
    p.seq = G.seq++;
    p.m = m;
    p.pat = *pat;
    for (int i = 0; i < 3; ++i) p.bg[i] = bg[i];
    p.target = target;
    p.a = *a;
    p.out_loss = out_loss;
    p.ssim_weight = ctx->ssim_weight;
    G.replays++;
    return TGSX_OK;
}

int32_t tgsx_fit_graph_stats(const tgsx_ctx* ctx, uint64_t* out_captures, uint64_t* out_replays,
                             uint64_t* out_reruns) {
    if (!ctx) return TGSX_EINVAL;
    const FitGraph* G = static_cast<const FitGraph*>(ctx->graph);
    if (out_captures) *out_captures = G ? G->captures : 0;
    if (out_replays) *out_replays = G ? G->replays : 0;
    if (out_reruns) *out_reruns = G ? G->reruns : 0;
    return TGSX_OK;
}

}  // extern "C"
