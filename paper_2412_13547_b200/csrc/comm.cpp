// In-library NCCL for view-batch data parallelism (BASELINE north_star "NCCL
// allreduce over NVLink sums per-Gaussian gradients and densification statistics").
//
// The communicator lives in the tgsx_ctx, its collectives run on the context's own comm stream
// ordered against the compute stream with events, so the batched step can pipeline
// chain(b) -> all-reduce(b) -> Adam(b) over Gaussian buckets (capi.cu tgsx_batched_step).
//
// NCCL is loaded with dlopen("libnccl.so.2") on first use instead of being linked: inside a
// PyTorch process that resolves to the NCCL torch already loaded (one NCCL per process, no ABI
// mix; the Python front end imports torch before the first communicator call so that it is
// loaded), elsewhere to the system library. Only the stable core API is used (unique id, init,
// all-reduce, destroy, error string), declared here with their C types. NVLink SHARP (NVLS) is
// NCCL's own choice for all-reduce on NVSwitch systems (NCCL_NVLS_ENABLE, default on).
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>

#include "tgsx_internal.h"

namespace {

typedef int nccl_result_t;  // ncclResult_t
typedef struct ncclComm* nccl_comm_t;
struct NcclUniqueId {
    char internal[128];
};
constexpr int kNcclFloat32 = 7;  // ncclFloat32
constexpr int kNcclSum = 0;      // ncclSum

struct NcclApi {
    void* h = nullptr;
    nccl_result_t (*get_unique_id)(NcclUniqueId*) = nullptr;
    nccl_result_t (*comm_init_rank)(nccl_comm_t*, int, NcclUniqueId, int) = nullptr;
    nccl_result_t (*all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    nccl_result_t (*comm_destroy)(nccl_comm_t) = nullptr;
    const char* (*error_string)(nccl_result_t) = nullptr;
    std::string err;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        const char* names[] = {"libnccl.so.2", "libnccl.so"};
        for (const char* n : names) {
            a.h = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
            if (a.h) break;
        }
        if (!a.h) {
            a.err = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        a.get_unique_id = (decltype(a.get_unique_id))dlsym(a.h, "ncclGetUniqueId");
        a.comm_init_rank = (decltype(a.comm_init_rank))dlsym(a.h, "ncclCommInitRank");
        a.all_reduce = (decltype(a.all_reduce))dlsym(a.h, "ncclAllReduce");
        a.comm_destroy = (decltype(a.comm_destroy))dlsym(a.h, "ncclCommDestroy");
        a.error_string = (decltype(a.error_string))dlsym(a.h, "ncclGetErrorString");
        if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.comm_destroy || !a.error_string) {
            a.err = "NCCL library lacks the core API";
            a.h = nullptr;
        }
    });
    return a;
}

int32_t cfail(tgsx_ctx* ctx, int32_t code, const std::string& msg) {
    if (ctx) ctx->err = msg;
    return code;
}

}  // namespace

namespace tgsx {

int32_t comm_allreduce_sum(tgsx_ctx* ctx, float* buf, size_t count, cudaStream_t s) {
    if (!ctx->comm) return cfail(ctx, TGSX_ESTATE, "no communicator attached (tgsx_comm_init)");
    if (count == 0) return TGSX_OK;
    NcclApi& a = api();
    const nccl_result_t r = a.all_reduce(buf, buf, count, kNcclFloat32, kNcclSum, (nccl_comm_t)ctx->comm, s);
    if (r) return cfail(ctx, TGSX_ECUDA, std::string("ncclAllReduce: ") + a.error_string(r));
    return TGSX_OK;
}

void comm_release(tgsx_ctx* ctx) {
    if (ctx->comm) {
        api().comm_destroy((nccl_comm_t)ctx->comm);
        ctx->comm = nullptr;
    }
    if (ctx->comm_stream) {
        cudaStreamSynchronize(ctx->comm_stream);
        cudaStreamDestroy(ctx->comm_stream);
        ctx->comm_stream = nullptr;
    }
    for (auto& e : ctx->pipe_events)
        if (e) cudaEventDestroy(e);
    ctx->pipe_events.clear();
    ctx->comm_ranks = 1;
    ctx->comm_rank = 0;
}

}  // namespace tgsx

extern "C" {

int32_t tgsx_comm_unique_id(uint8_t out_id[128]) {
    if (!out_id) return TGSX_EINVAL;
    NcclApi& a = api();
    if (!a.h) return TGSX_ESTATE;
    NcclUniqueId id;
    if (a.get_unique_id(&id)) return TGSX_ECUDA;
    std::memcpy(out_id, id.internal, 128);
    return TGSX_OK;
}

int32_t tgsx_comm_init(tgsx_ctx* ctx, const uint8_t id[128], int32_t nranks, int32_t rank) {
    if (!ctx || !id || nranks < 1 || rank < 0 || rank >= nranks)
        return cfail(ctx, TGSX_EINVAL, "comm_init: bad rank / world size");
    NcclApi& a = api();
    if (!a.h) return cfail(ctx, TGSX_ESTATE, a.err);
    tgsx::comm_release(ctx);
    int prev = 0;
    cudaGetDevice(&prev);
    if (prev != ctx->device) cudaSetDevice(ctx->device);
    NcclUniqueId uid;
    std::memcpy(uid.internal, id, 128);
    nccl_comm_t c = nullptr;
    const nccl_result_t r = a.comm_init_rank(&c, nranks, uid, rank);
    cudaError_t e = cudaSuccess;
    if (!r) e = cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking);
    if (prev != ctx->device) cudaSetDevice(prev);
    if (r) return cfail(ctx, TGSX_ECUDA, std::string("ncclCommInitRank: ") + a.error_string(r));
    if (e) {
        a.comm_destroy(c);
        return cfail(ctx, TGSX_ECUDA, cudaGetErrorString(e));
    }
    ctx->comm = c;
    ctx->comm_ranks = nranks;
    ctx->comm_rank = rank;
    return TGSX_OK;
}

int32_t tgsx_comm_destroy(tgsx_ctx* ctx) {
    if (!ctx) return TGSX_EINVAL;
    tgsx::comm_release(ctx);
    return TGSX_OK;
}

int32_t tgsx_comm_size(const tgsx_ctx* ctx) { return ctx ? ctx->comm_ranks : 0; }

}  // extern "C"
