// Host-side internals of libtgsx: context, device model, workspace, kernel launchers.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "../../include/tgsx.h"

namespace tgsx {

// Growable device allocation (never shrinks; contents are not preserved on growth unless
// grow_keep is used).
struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need);
    cudaError_t grow_keep(size_t need, size_t keep_bytes, cudaStream_t s);
    void release();
    template <typename T>
    T* as() const { return static_cast<T*>(p); }
};

// Arguments of the target-rows staging kernel of graph-captured dilated steps (capi.cu): rows
// r = 0..rows-1 of row_floats floats from src + r * pitch_floats to dst + r * row_floats. A graph
// replay re-targets src per step (graph.cpp: a 2-D memcpy node cannot be updated in an exec).
struct StageRowsArgs {
    float* dst;
    const float* src;
    int64_t row_floats, pitch_floats;
    int32_t rows;
};

// frees the buffers DevBuf::ensure / grow_keep retired while growing (capi.cu)
void drain_graveyard();

struct Status {
    int32_t code = TGSX_OK;
    std::string msg;
};

struct Workspace {
    // per-render, rank (blend) order
    DevBuf prep;        // Prepared[n]
    DevBuf touched;     // u32[n + 1] tiles touched per rank
    DevBuf pair_off;    // u32[n + 1] exclusive scan of touched
    DevBuf rect;        // uint2[n] tile rectangle per rank (tx0 | tx1 << 16, ty0 | ty1 << 16) for the claims
    DevBuf scan_tmp;    // look-back status
    // binning
    DevBuf keys[2], vals[2];  // u32[K] ping-pong
    DevBuf sort_tmp;          // histograms + block status + tickets
    DevBuf ranges;            // uint2[tiles]
    // slab binning: per-tile slot cursors (one per 128-B line) and kSegCap-entry slabs
    DevBuf tile_fill, tile_slab;
    DevBuf partial;           // per-(tile, splat) gradient partials, Partials SoA (40 B/pair)
    int64_t pair_cap = 0;     // pairs the partial buffer holds
    // per-pixel
    DevBuf rgb, T, last, dLdC, target;
    DevBuf block_loss;        // float[tiles]
    DevBuf ssim_abc, ssim_part, loss_grad;  // dense SSIM adjoint weights [P][3][3], block sums
    DevBuf counters;          // u64: [0] err, [1] blend ops, [2] evals, [3..] scratch
    DevBuf generic;           // misc scratch
    // pinned host scratch
    uint64_t* h_scratch = nullptr;
    int64_t K = 0;
    int tiles_x = 0, tiles_y = 0;
    int last_W = 0, last_H = 0, last_P = 0;
    bool have_forward = false;
};

}  // namespace tgsx

namespace tgsx {
// Live per-stage timing with CUDA events on the context stream (enabled by tgsx_profile).
enum Stage { kStDepthSort, kStPreprocess, kStScan, kStDuplicate, kStSort, kStRanges,
             kStForward, kStBackward, kStChain, kStLoss, kStDensify, kStAdam, kNumStages };
struct Profiler {
    bool enabled = false;
    std::vector<cudaEvent_t> pool;          // reusable events
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    double ms[kNumStages] = {};
    int64_t count[kNumStages] = {};
    size_t next = 0;
    cudaEvent_t get();
    void begin(int stage, cudaStream_t s, cudaEvent_t* out);
    void end(int stage, cudaStream_t s, cudaEvent_t start);
    void harvest();  // accumulates completed pairs (caller ensures completion)
};
}  // namespace tgsx

struct tgsx_ctx {
    int device = 0;
    cudaStream_t stream = nullptr;
    cudaStream_t own_stream = nullptr;
    std::string err;
    uint64_t launches = 0;
    tgsx::Workspace ws;
    tgsx::Profiler prof;
    // host-resident view targets: double-buffered H2D on a copy stream so the copy of view i+1
    // overlaps the kernels of view i (events order buffer reuse against the compute stream)
    cudaStream_t copy_stream = nullptr;
    tgsx::DevBuf stage_buf[2];
    cudaEvent_t staged[2] = {nullptr, nullptr}, consumed[2] = {nullptr, nullptr};
    bool stage_used[2] = {false, false};
    int stage_next = 0, stage_pending = -1;
    // binning reuse: views of an unchanged model with the same geometry share one binning (the
    // tile lists do not depend on the dilation offset). Any entry point that changes the
    // parameters, the row order or the binning workspace clears bin_valid.
    float ssim_weight = 0.f;  // lambda_ssim of dense fused views (tgsx_set_ssim_weight)
    int binning_mode = 0;     // 0 slab / per-tile binning with fallback, 1 force the onesweep paths
    bool bin_valid = false;
    uint64_t bin_model = 0;
    int bin_lowpass = 0, bin_W = 0, bin_H = 0;
    int64_t bin_n = -1;
    uint32_t* bin_items = nullptr;
    // deferred binning read-back (fused views): the counters copy is waited for after the
    // forward has been queued, so the GPU never idles on the host's decision
    cudaEvent_t bin_event = nullptr;
    bool bin_pending = false;
    int bin_sort_cap = 0;           // longest list the speculative per-tile sort handled
    uint64_t bin_max_hint = 0;      // longest list of the previous binning
    uint64_t bin3d_max_hint = 0;    // 3-D views: the previous binning's longest list
    int bin3d_sort_cap = 0;         // 3-D: longest list the speculative per-tile sort handled
    bool bin3d_pending = false;     // 3-D: a deferred binning awaits bin3d_settle
    // blend backward launch configuration, per context (= per device): the dynamic shared-memory
    // opt-in is a per-device function attribute and the resident-CTA count sizes the grid
    int bwd_resident[3] = {0, 0, 0};  // [0] / [1] resident CTAs of backward_kernel<2,2> / <1,1>; [2] CTA variant configured
    // NCCL communicator of a view-sharded fit (comm.cpp; null = single rank) and its stream;
    // events of the pipelined batched step (chain(b) -> all-reduce(b) -> Adam(b))
    void* comm = nullptr;
    int comm_ranks = 1, comm_rank = 0;
    cudaStream_t comm_stream = nullptr;
    std::vector<cudaEvent_t> pipe_events;
    // pipeline timeline of the last profiled batched step: per bucket (chain start, chain end,
    // all-reduce start, all-reduce end, Adam start, Adam end) in ms from the step's first event
    std::vector<float> pipe_timeline;
    // CUDA-graph replay of the fused fit step (graph.cpp, tgsx_fit_graph_step): while capturing,
    // the backward / chain kernels get the fault word and the capture-time capacities as guards
    bool graph_capturing = false, graph_replaying = false;
    unsigned* graph_fault = nullptr;    // device word, sticky until the host re-runs the steps
    unsigned* h_graph_fault = nullptr;  // pinned [2]: the fault word after each slot's last launch
    int64_t graph_guard_pairs = 0;      // pair count the captured step may produce (<= pair_cap)
    void* graph_chain_node = nullptr;   // cudaGraphNode_t of the captured chain kernel
    void* graph_loss_node = nullptr;    // cudaGraphNode_t of the captured loss copy (out_loss), if any
    const void* graph_loss_src = nullptr;  // its device source (the step's loss word)
    bool graph_stage_targets = false;   // this call's model has replayed steps for several device targets
    void* graph_target_node = nullptr;  // cudaGraphNode_t of the captured target staging
    int graph_target_kind = 0;          // 1: 1-D memcpy node, 2: stage-rows kernel node
    int64_t graph_target_off = 0;       // its source offset (floats) from the target's base
    tgsx::StageRowsArgs graph_stage_args{};  // kind 2: the kernel's captured arguments
    void* graph = nullptr;              // tgsx::FitGraph
};

// Scoped stage timer: no-op unless profiling is enabled.
namespace tgsx {
struct StageTimer {
    tgsx_ctx* ctx;
    int stage;
    cudaEvent_t start = nullptr;
    StageTimer(tgsx_ctx* c, int st) : ctx(c), stage(st) {
        if (ctx->prof.enabled) ctx->prof.begin(stage, ctx->stream, &start);
    }
    ~StageTimer() {
        if (ctx->prof.enabled && start) ctx->prof.end(stage, ctx->stream, start);
    }
};
}  // namespace tgsx

struct tgsx_model {
    uint64_t uid = 0;  // unique per created model (binning-reuse key)
    int64_t n = 0, cap = 0;
    uint64_t next_id = 0;
    bool order_dirty = true;
    bool ids_monotone = true;
    bool blend_phys = false;  // rows physically in blend (rank) order (perm maps rank -> logical)
    tgsx::DevBuf params;   // float[10][cap]: px py rot lsx lsy rop cr cg cb depth
    tgsx::DevBuf ids;      // u64[cap]
    tgsx::DevBuf pos_acc, col_acc, accum, visit, window, tau_v;
    tgsx::DevBuf m1, m2;   // float[9][cap] Adam moments
    tgsx::DevBuf step;     // StepRec[cap] (AoS, 48 B/G) batched-view step buffer
    tgsx::DevBuf perm;     // u32[cap] rank -> index
    tgsx::DevBuf rank_of;  // u32[cap] index -> rank
    tgsx::DevBuf screen;   // float[10][cap] screen-space grads of the last backward
    tgsx::DevBuf spare[11];  // prune compaction targets (swapped with the live rows; no per-event malloc)
    tgsx::DevBuf spatial;    // u32[cap] blend ranks in slot-claim (spatial) order (raster.cu launch_claims)
    bool spatial_valid = false;
    int spatial_age = 0;
    int64_t step_views = 0;
};

// 3-D front end model (scene3d.cu): params float[59][cap] = mean(3),
// quaternion wxyz(4), log-scales(3), raw opacity, SH coefficients [16][3]; row (creation) order.
struct tgsx_model3d {
    int64_t n = 0, cap = 0;
    tgsx::DevBuf params;            // float[59][cap]
    tgsx::DevBuf m1, m2;            // float[59][cap] Adam moments
    tgsx::DevBuf pos_acc, col_acc;  // float[cap] densify statistics
    tgsx::DevBuf visit;             // i32[cap]
    tgsx::DevBuf perm, rank_of;     // u32[cap] blend order of the last view
    tgsx::DevBuf prep_row;          // Prepared[cap] records in row order (before the depth sort)
    tgsx::DevBuf gbuf;              // float[17][n] chain-rule output of the fused step (scene3d.cu)
    tgsx::DevBuf step;              // float[62][cap] batched-view step buffer (all-reduced across ranks)
    int64_t step_views = 0;
    tgsx::DevBuf skeys;             // u32[cap] sorted depth keys of the global-sort path (parity stage)
    bool rank_ordered = false;      // last binning: records / pair slots by blend rank (global-sort
                                    // path) rather than by row (per-tile path)
    // densification state (densify3d.cu; the 2-D DensifyStats analogues):
    // stable ids, per-Gaussian visit threshold, and the visit count at the last densify event /
    // visit audit (accum = visit - visit_evt, window = visit - visit_aud: the fit kernels only
    // ever increment `visit`)
    tgsx::DevBuf ids;               // u64[cap]
    tgsx::DevBuf tau_v;             // f64[cap]
    tgsx::DevBuf visit_evt, visit_aud;  // i32[cap]
    uint64_t next_id = 0;
    tgsx::DevBuf spare[11];         // prune compaction targets (swapped with the live rows)
};

namespace tgsx {
// graph.cpp: verifies every in-flight graph-replayed fit step (re-running a faulted one and its
// successors eagerly); called by every entry point that reads or changes the model
int32_t graph_flush(tgsx_ctx* ctx);
void graph_release(tgsx_ctx* ctx);
}  // namespace tgsx

// physical row order of the model (capi.cu): blend order for the hot path, logical (creation)
// order for densify / download / explicit-gradient APIs
cudaError_t model_to_blend_order(tgsx_ctx* ctx, tgsx_model* m);
cudaError_t model3d_grow(tgsx_ctx* ctx, tgsx_model3d* m, int64_t cap);  // keeps the live rows
// ids = i, tau_v = SPEC default tau_v_init for rows [i0, i1) of a freshly uploaded 3-D model
cudaError_t densify3d_init_rows(tgsx_ctx* ctx, tgsx_model3d* m, int64_t i0, int64_t i1);
cudaError_t model_to_logical_order(tgsx_ctx* ctx, tgsx_model* m);
// capacity growth keeping contents, spare row buffers sized alongside (capi.cu)
cudaError_t model_grow(tgsx_ctx* ctx, tgsx_model* m, int64_t cap);

namespace tgsx {

// Adam hyper-parameters for one step, computed on the host.
struct AdamCfg {
    float lr[9];
    float b1, b2, omb1, omb2, eps, bc1, bc2;
    float ls_lo, ls_hi, raw_cap;
    float batch;  // divisor for the batched mean (1 = plain step)
};

// kernel launchers (defined in the .cu files); all enqueue on ctx->stream
struct RenderArgs {
    int p, ox, oy, W, H, cols, rows, P;
    float bg[3];
    int lowpass_p;
    const float* target;  // fused L1 target (device, W*H*3) or null
    float l1_weight;      // weight of the L1 term (1 - lambda_ssim on dense SSIM iterations)
    int target_rows = 1;  // > 1: the target holds only the active rows (row (y - oy) / p)
};

cudaError_t launch_sort_depth(tgsx_ctx* ctx, tgsx_model* m);
// NCCL (comm.cpp): in-place sum all-reduce of `count` floats on stream s; communicator teardown
int32_t comm_allreduce_sum(tgsx_ctx* ctx, float* buf, size_t count, cudaStream_t s);
void comm_release(tgsx_ctx* ctx);
// d_total non-null: the pair-offset scan is fused in (rows must be in blend order): pair_off,
// the records' first pair slot and the total pair count K are written by the same kernel
cudaError_t launch_preprocess(tgsx_ctx* ctx, tgsx_model* m, int lowpass_p, int W, int H,
                              uint32_t* d_total = nullptr);
cudaError_t launch_exclusive_scan(tgsx_ctx* ctx, const uint32_t* in, uint32_t* out, int64_t n,
                                  uint32_t* d_total);
cudaError_t launch_duplicate(tgsx_ctx* ctx, int64_t n, int key_bits);
size_t sort_scratch_bytes(int64_t n, int key_bits);
cudaError_t sort_pairs(tgsx_ctx* ctx, uint32_t*& keys, uint32_t*& vals, uint32_t* keys_alt,
                       uint32_t* vals_alt, int64_t n, int key_bits, const uint32_t* d_hist);
cudaError_t launch_ranges(tgsx_ctx* ctx, const uint32_t* keys, int64_t K, int tiles);
// slab binning: preprocess claims slots in per-tile slabs of kSegCap entries -> ranges ->
// per-tile warp register sort (lists up to kSegCap; longer lists take the onesweep path)
constexpr int kSegCap = 1024;
cudaError_t launch_slab_finalize(tgsx_ctx* ctx, int tiles);
cudaError_t launch_seg_sort(tgsx_ctx* ctx, uint32_t* items, int tiles, int64_t max_list);
cudaError_t launch_forward(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items,
                           bool fused_loss);
cudaError_t launch_backward(tgsx_ctx* ctx, const RenderArgs& ra, const uint32_t* items);
// compute_loss pieces (loss.cu): L1 over given colours, dense SSIM term, loss value
cudaError_t launch_l1(tgsx_ctx* ctx, const RenderArgs& ra, const float* rgb, float scale, float* dLdC,
                      float* block_sum, int* nblocks);
size_t ssim_blocks(int W, int H);
cudaError_t launch_ssim(tgsx_ctx* ctx, const float* rgb, const float* target, int W, int H, float lam,
                        float* abc, float* block_sum, float* dLdC);
cudaError_t launch_loss_finalize(tgsx_ctx* ctx, const float* l1_part, int n1, float w1, const float* s_part,
                                 int n2, float lam, double inv, float* out);
enum class ChainMode { kGrads, kAdam, kAccumulate };
// [i0, i1): the Gaussian rows of this launch (i1 < 0: up to n)
cudaError_t launch_chain(tgsx_ctx* ctx, tgsx_model* m, ChainMode mode, bool update_stats,
                         float* grads_out, const float* adam_cfg, int64_t i0 = 0, int64_t i1 = -1);
cudaError_t launch_adam(tgsx_ctx* ctx, tgsx_model* m, const float* grads, const float* adam_cfg,
                        int batch_views, int64_t i0 = 0, int64_t i1 = -1);
// graph.cpp helpers: the Adam hyper-parameters of a step (capi.cu fill_adam) and the per-launch
// update of a captured chain kernel node (optim.cu)
void adam_cfg_from_args(AdamCfg& c, const tgsx_adam_args* a);
cudaError_t chain_node_set_adam(cudaGraphExec_t exec, cudaGraphNode_t node, const AdamCfg& c);
bool graph_eligible_binning(const tgsx_ctx* ctx);

int key_bits_for(int tiles);

// 3-D front end (scene3d.cu)
struct Cam3 {
    float R[9], t[3];
    float fx, fy, cx, cy, znear;
    float limx, limy;  // 1.3 tan(fov / 2) clamp of the EWA Jacobian
    float C[3];        // camera centre -R^T t
};
struct Adam3dCfg {
    float lr[6];  // mean, rotation, log-scale, opacity, SH DC, SH rest
    float b1, b2, omb1, omb2, eps, bc1, bc2, raw_cap;
};
constexpr int k3dParams = 59;
cudaError_t launch_preprocess3d(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int W, int H);
// per-tile path: records by row, slab claims by row, fused pair-offset scan (K to d_total)
cudaError_t launch_preprocess3d_bin(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int W, int H,
                                    uint32_t* d_total);
// per-tile (depth key, row) sort of the slabs (keys = ws.keys[0] by row)
cudaError_t launch_seg_sort3d(tgsx_ctx* ctx, int tiles, int64_t max_list);
// gather into blend order + slot claims + the fused pair-offset scan (total K to d_total)
cudaError_t launch_bin3d(tgsx_ctx* ctx, tgsx_model3d* m, const uint32_t* skeys, const uint32_t* svals,
                         int W, int H, uint32_t* d_total);
// mode: 0 gradients out, 1 fused Adam, 2 accumulate into the batched step buffer
cudaError_t launch_chain3d(tgsx_ctx* ctx, tgsx_model3d* m, const Cam3& cam, int lowpass_p, int mode,
                           bool update_stats, float* grads, float* screen, const Adam3dCfg* cfg);
cudaError_t launch_adam3d_step(tgsx_ctx* ctx, tgsx_model3d* m, int batch_views, const Adam3dCfg& cfg);
constexpr int k3dStepRows = 62;  // 59 gradient sums, position-norm sum, colour-norm sum, visits
cudaError_t launch_adam3d(tgsx_ctx* ctx, tgsx_model3d* m, const float* grads, const Adam3dCfg& cfg);

}  // namespace tgsx
