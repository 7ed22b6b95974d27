// Initializer on the device (the reference ships only the KD-tree header,
// kdtree.hpp:15-139): exact k-nearest neighbours of every point through a uniform grid hash.
//
//  grid_count / grid_scatter   points bucketed by cell (counting sort: count, scan, scatter)
//  knn_kernel                  one thread per query point: rings of cells around its own cell,
//                              keeping the k smallest (dist2, index) pairs (the ordering and
//                              exclusion rule of KdTree2::knn, kdtree.hpp:30-38,96-116) with
//                              dist2 = dx*dx + dy*dy in float, unfused (the reference is built
//                              with -ffp-contract=off); stops once every point outside the
//                              searched rings is provably farther than the k-th neighbour.
// Results equal the reference KD-tree's exactly (tests/test_gpu_init.py).
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <vector>

namespace tgsx {

namespace {

constexpr int kMaxK = 8;

struct Grid {
    float x0, y0, inv_h, h;
    int gx, gy;
};

__device__ __forceinline__ int cell_of(float v, float v0, float inv_h, int g) {
    int c = (int)floorf((v - v0) * inv_h);
    return c < 0 ? 0 : (c >= g ? g - 1 : c);
}

__global__ void grid_count(const float* __restrict__ xy, int64_t n, Grid G, uint32_t* __restrict__ cnt,
                           uint32_t* __restrict__ cell) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int cx = cell_of(xy[2 * i], G.x0, G.inv_h, G.gx), cy = cell_of(xy[2 * i + 1], G.y0, G.inv_h, G.gy);
    const uint32_t c = (uint32_t)(cy * G.gx + cx);
    cell[i] = c;
    atomicAdd(&cnt[c], 1u);
}

__global__ void grid_scatter(const uint32_t* __restrict__ cell, int64_t n, uint32_t* __restrict__ fill,
                             uint32_t* __restrict__ slots) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    slots[atomicAdd(&fill[cell[i]], 1u)] = (uint32_t)i;
}

__device__ __forceinline__ bool lex_less(float d, uint32_t i, float e, uint32_t j) {
    return d < e || (d == e && i < j);
}

template <int K>
__global__ void __launch_bounds__(128) knn_kernel(const float* __restrict__ xy, int64_t n, Grid G,
                                                  const uint32_t* __restrict__ start, const uint32_t* __restrict__ slots,
                                                  int k, uint32_t* __restrict__ out_idx, float* __restrict__ out_d2) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const float qx = xy[2 * q], qy = xy[2 * q + 1];
    const int cx = cell_of(qx, G.x0, G.inv_h, G.gx), cy = cell_of(qy, G.y0, G.inv_h, G.gy);
    float bd[K];
    uint32_t bi[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
        bd[j] = FLT_MAX;
        bi[j] = 0xffffffffu;
    }
    int found = 0;
    const int rmax = max(G.gx, G.gy);
    for (int r = 0; r <= rmax; ++r) {
        for (int yy = cy - r; yy <= cy + r; ++yy) {
            if (yy < 0 || yy >= G.gy) continue;
            const bool edge_row = (yy == cy - r) || (yy == cy + r);
            for (int xx = cx - r; xx <= cx + r; xx += (edge_row || r == 0) ? 1 : 2 * r) {
                if (xx < 0 || xx >= G.gx) continue;
                const uint32_t c = (uint32_t)(yy * G.gx + xx);
                for (uint32_t s = start[c]; s < start[c + 1]; ++s) {
                    const uint32_t p = slots[s];
                    if (p == (uint32_t)q) continue;
                    const float dx = __fsub_rn(qx, xy[2 * p]), dy = __fsub_rn(qy, xy[2 * p + 1]);
                    const float d2 = __fadd_rn(__fmul_rn(dx, dx), __fmul_rn(dy, dy));
                    if (found < k || lex_less(d2, p, bd[k - 1], bi[k - 1])) {
                        // insertion into the sorted k-list
                        float cd = d2;
                        uint32_t ci = p;
#pragma unroll
                        for (int j = 0; j < K; ++j) {
                            if (j < k && lex_less(cd, ci, bd[j], bi[j])) {
                                const float td = bd[j];
                                const uint32_t ti = bi[j];
                                bd[j] = cd;
                                bi[j] = ci;
                                cd = td;
                                ci = ti;
                            }
                        }
                        found = min(found + 1, k);
                    }
                }
            }
        }
        // every point beyond ring r lies at least r * h away along x or y (q is inside its cell);
        // 0.1 % margin for the rounding of the cell assignment
        if (found == k) {
            const float bound = (float)r * G.h * 0.999f;
            if (bd[k - 1] < bound * bound) break;
        }
    }
    for (int j = 0; j < k; ++j) {
        out_idx[q * k + j] = j < found ? bi[j] : 0xffffffffu;
        if (out_d2) out_d2[q * k + j] = j < found ? bd[j] : INFINITY;
    }
}

inline unsigned grid_for(int64_t n, int bt) { return (unsigned)((n + bt - 1) / bt); }

}  // namespace

// k nearest neighbours of every point (self excluded), ascending (dist2, index).
cudaError_t launch_knn(tgsx_ctx* ctx, const float* d_xy, int64_t n, int k, uint32_t* d_idx, float* d_d2,
                       const float bbox[4]) {
    if (n == 0) return cudaSuccess;
    Workspace& ws = ctx->ws;
    const float w = std::max(bbox[2] - bbox[0], 1e-6f), h = std::max(bbox[3] - bbox[1], 1e-6f);
    // about two points per cell
    const double cells = std::max<double>(1.0, (double)n / 2.0);
    float cell = (float)std::sqrt((double)w * (double)h / cells);
    cell = std::max(cell, std::max(w, h) / 4096.0f);
    Grid G;
    G.x0 = bbox[0];
    G.y0 = bbox[1];
    G.h = cell;
    G.inv_h = 1.0f / cell;
    G.gx = std::max(1, (int)std::ceil(w / cell) + 1);
    G.gy = std::max(1, (int)std::ceil(h / cell) + 1);
    const int64_t ncells = (int64_t)G.gx * G.gy;
    cudaError_t e;
    // scratch: cell[n], slots[n], count/start[ncells + 1], fill[ncells]
    if ((e = ws.generic.ensure((size_t)(2 * n + 2 * (ncells + 1)) * 4))) return e;
    uint32_t* cellv = ws.generic.as<uint32_t>();
    uint32_t* slots = cellv + n;
    uint32_t* cnt = slots + n;
    uint32_t* fill = cnt + (ncells + 1);
    if ((e = cudaMemsetAsync(cnt, 0, (size_t)(ncells + 1) * 4, ctx->stream))) return e;
    grid_count<<<grid_for(n, 256), 256, 0, ctx->stream>>>(d_xy, n, G, cnt, cellv);
    ctx->launches++;
    if ((e = launch_exclusive_scan(ctx, cnt, fill, ncells + 1, nullptr))) return e;
    // fill holds the exclusive scan (cell starts); keep a copy as the start array
    if ((e = cudaMemcpyAsync(cnt, fill, (size_t)(ncells + 1) * 4, cudaMemcpyDeviceToDevice, ctx->stream))) return e;
    grid_scatter<<<grid_for(n, 256), 256, 0, ctx->stream>>>(cellv, n, fill, slots);
    ctx->launches++;
    if (k <= 4)
        knn_kernel<4><<<grid_for(n, 128), 128, 0, ctx->stream>>>(d_xy, n, G, cnt, slots, k, d_idx, d_d2);
    else
        knn_kernel<kMaxK><<<grid_for(n, 128), 128, 0, ctx->stream>>>(d_xy, n, G, cnt, slots, k, d_idx, d_d2);
    ctx->launches++;
    return cudaGetLastError();
}

}  // namespace tgsx

// ============================================================================ C ABI
#include <cstring>
#include <string>
#include <unordered_set>

using namespace tgsx;

namespace {

struct PcgInit {
    uint64_t s[2];
    explicit PcgInit(uint64_t seed, uint64_t stream) { tgsx_pcg32_init(s, seed, stream); }
    double uniform() { return tgsx_pcg32_uniform(s); }
};

int32_t cuda_err(tgsx_ctx* ctx, cudaError_t e, const char* where) {
    ctx->err = std::string(where) + ": " + cudaGetErrorString(e);
    return TGSX_ECUDA;
}

int32_t knn_host(tgsx_ctx* ctx, const float* xy, int64_t n, int k, uint32_t* out_idx, float* out_d2) {
    if (n <= 0) return TGSX_OK;
    float bb[4] = {xy[0], xy[1], xy[0], xy[1]};
    for (int64_t i = 1; i < n; ++i) {
        bb[0] = std::min(bb[0], xy[2 * i]);
        bb[1] = std::min(bb[1], xy[2 * i + 1]);
        bb[2] = std::max(bb[2], xy[2 * i]);
        bb[3] = std::max(bb[3], xy[2 * i + 1]);
    }
    if (!std::isfinite(bb[0]) || !std::isfinite(bb[1]) || !std::isfinite(bb[2]) || !std::isfinite(bb[3]))
        return TGSX_EINVAL;
    ctx->bin_valid = false;  // the grid uses the binning scratch
    Workspace& ws = ctx->ws;
    cudaError_t e;
    // device buffers: points, indices, distances (the loss-gradient buffer is free here)
    const size_t pts = (size_t)n * 8, idx = (size_t)n * k * 4;
    if ((e = ws.loss_grad.ensure(pts + 2 * idx))) return cuda_err(ctx, e, "tgsx_knn: allocate");
    float* d_xy = ws.loss_grad.as<float>();
    uint32_t* d_idx = reinterpret_cast<uint32_t*>(ws.loss_grad.as<char>() + pts);
    float* d_d2 = reinterpret_cast<float*>(ws.loss_grad.as<char>() + pts + idx);
    if ((e = cudaMemcpyAsync(d_xy, xy, pts, cudaMemcpyHostToDevice, ctx->stream))) return cuda_err(ctx, e, "tgsx_knn: upload");
    if ((e = launch_knn(ctx, d_xy, n, k, d_idx, d_d2, bb))) return cuda_err(ctx, e, "tgsx_knn: kernels");
    if ((e = cudaMemcpyAsync(out_idx, d_idx, idx, cudaMemcpyDeviceToHost, ctx->stream))) return cuda_err(ctx, e, "tgsx_knn: download");
    if (out_d2 && (e = cudaMemcpyAsync(out_d2, d_d2, idx, cudaMemcpyDeviceToHost, ctx->stream))) return cuda_err(ctx, e, "tgsx_knn: download");
    if ((e = cudaStreamSynchronize(ctx->stream))) return cuda_err(ctx, e, "tgsx_knn: synchronize");
    return TGSX_OK;
}

}  // namespace

extern "C" {

int32_t tgsx_knn(tgsx_ctx* ctx, const float* xy, int64_t n, int32_t k, uint32_t* out_idx, float* out_d2) {
    if (!ctx || n < 0 || (n > 0 && (!xy || !out_idx)) || k < 1 || k > kMaxK) return TGSX_EINVAL;
    return knn_host(ctx, xy, n, k, out_idx, out_d2);
}

// sample_seed_points: count/2 uniform points, then count - count/2 drawn with
// probability proportional to the luminance-gradient magnitude (central differences, edge
// clamped; uniform when the image is flat), each jittered uniformly inside its pixel. PCG32
// (seed, stream 2), draws per point in order: uniform x, y; importance u, jitter x, jitter y.
// Colours are read at the point's pixel.
int32_t tgsx_seed_points(const float* image, int32_t W, int32_t H, int64_t count, uint64_t seed,
                         float* out_xy, float* out_rgb) {
    if (!image || !out_xy || W < 1 || H < 1 || count < 1 || count > (int64_t)W * H) return TGSX_EINVAL;
    PcgInit rng(seed, 2);
    const int64_t P = (int64_t)W * H;
    auto lum = [&](int x, int y) {
        x = std::min(std::max(x, 0), W - 1);
        y = std::min(std::max(y, 0), H - 1);
        const float* c = image + 3 * ((int64_t)y * W + x);
        return 0.299 * c[0] + 0.587 * c[1] + 0.114 * c[2];
    };
    std::vector<double> cdf((size_t)P);
    double total = 0.0;
    for (int y = 0; y < H; ++y)
        for (int x = 0; x < W; ++x) {
            const double gx = 0.5 * (lum(x + 1, y) - lum(x - 1, y)), gy = 0.5 * (lum(x, y + 1) - lum(x, y - 1));
            total += std::sqrt(gx * gx + gy * gy);
            cdf[(size_t)y * W + x] = total;
        }
    const int64_t nu = count / 2;
    for (int64_t i = 0; i < count; ++i) {
        double x, y;
        if (i < nu || !(total > 0.0)) {
            x = rng.uniform() * W;
            y = rng.uniform() * H;
        } else {
            const double u = rng.uniform() * total;
            const int64_t px = std::upper_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
            const int64_t pp = std::min<int64_t>(px, P - 1);
            x = (double)(pp % W) + rng.uniform();
            y = (double)(pp / W) + rng.uniform();
        }
        float fx = (float)x, fy = (float)y;
        fx = std::min(fx, std::nextafter((float)W, 0.f));  // keep rounding inside the image
        fy = std::min(fy, std::nextafter((float)H, 0.f));
        out_xy[2 * i] = fx;
        out_xy[2 * i + 1] = fy;
        if (out_rgb) {
            const int px = std::min((int)fx, W - 1), py = std::min((int)fy, H - 1);
            std::memcpy(out_rgb + 3 * i, image + 3 * ((int64_t)py * W + px), 12);
        }
    }
    return TGSX_OK;
}

// kdtree_upsample: per round, every point's nearest neighbour (self excluded,
// ties by lower index, as KdTree2::nearest_of); the midpoint (position and colour averaged in
// float) of each unique unordered pair {i, nn(i)} is appended in ascending (min, max) pair
// order unless its position equals an existing point's or an earlier midpoint's.
int32_t tgsx_upsample(tgsx_ctx* ctx, const float* xy, const float* rgb, int64_t n, int32_t rounds,
                      int64_t capacity, float* out_xy, float* out_rgb, int64_t* out_n) {
    if (!ctx || !xy || !rgb || !out_xy || !out_rgb || !out_n || n < 0 || rounds < 0 || capacity < n)
        return TGSX_EINVAL;
    std::vector<float> P(xy, xy + 2 * n), Cc(rgb, rgb + 3 * n);
    for (int32_t round = 0; round < rounds && P.size() / 2 >= 2; ++round) {
        const int64_t m = (int64_t)(P.size() / 2);
        std::vector<uint32_t> nn((size_t)m);
        int32_t rc = knn_host(ctx, P.data(), m, 1, nn.data(), nullptr);
        if (rc) return rc;
        std::vector<std::pair<uint32_t, uint32_t>> pairs;
        pairs.reserve((size_t)m);
        for (int64_t i = 0; i < m; ++i) {
            const uint32_t j = nn[(size_t)i];
            if (j == 0xffffffffu) continue;
            pairs.emplace_back(std::min((uint32_t)i, j), std::max((uint32_t)i, j));
        }
        std::sort(pairs.begin(), pairs.end());
        pairs.erase(std::unique(pairs.begin(), pairs.end()), pairs.end());
        std::unordered_set<uint64_t> seen;
        auto key = [](float x, float y) {
            uint32_t a, b;
            std::memcpy(&a, &x, 4);
            std::memcpy(&b, &y, 4);
            return ((uint64_t)a << 32) | b;
        };
        for (int64_t i = 0; i < m; ++i) seen.insert(key(P[2 * i], P[2 * i + 1]));
        for (const auto& pr : pairs) {
            const uint32_t a = pr.first, b = pr.second;
            const float mx = (P[2 * a] + P[2 * b]) * 0.5f, my = (P[2 * a + 1] + P[2 * b + 1]) * 0.5f;
            if (!seen.insert(key(mx, my)).second) continue;
            if ((int64_t)(P.size() / 2) >= capacity) return TGSX_EINVAL;
            P.push_back(mx);
            P.push_back(my);
            for (int c = 0; c < 3; ++c) Cc.push_back((Cc[3 * a + c] + Cc[3 * b + c]) * 0.5f);
        }
    }
    *out_n = (int64_t)(P.size() / 2);
    std::memcpy(out_xy, P.data(), P.size() * 4);
    std::memcpy(out_rgb, Cc.data(), Cc.size() * 4);
    return TGSX_OK;
}

// init_model: one Gaussian per point: position; activated colour = the
// sampled colour (logit, clamped to [1e-4, 1 - 1e-4]); isotropic log-scale = log of the mean
// distance to the 3 nearest neighbours (double from the exact float dist2; image diagonal / 16
// for fewer than 4 points; floor ln 1e-4); activated opacity 0.1; rotation 0; depth keys
// uniform from PCG32 (seed, stream 3); ids 0..n-1; fresh stats (tau_v 5).
int32_t tgsx_init_model(tgsx_ctx* ctx, tgsx_model* m, const float* xy, const float* rgb, int64_t n,
                        int32_t W, int32_t H, uint64_t seed) {
    if (!ctx || !m || !xy || !rgb || n < 1 || W < 1 || H < 1) return TGSX_EINVAL;
    std::vector<double> scale((size_t)n, std::hypot((double)W, (double)H) / 16.0);
    if (n >= 4) {
        std::vector<uint32_t> idx((size_t)n * 3);
        std::vector<float> d2((size_t)n * 3);
        int32_t rc = knn_host(ctx, xy, n, 3, idx.data(), d2.data());
        if (rc) return rc;
        for (int64_t i = 0; i < n; ++i)
            scale[(size_t)i] = (std::sqrt((double)d2[3 * i]) + std::sqrt((double)d2[3 * i + 1]) +
                                std::sqrt((double)d2[3 * i + 2])) / 3.0;
    }
    std::vector<float> px(n), py(n), rot(n, 0.f), ls(n), rop(n), cr(n), cg(n), cb(n), depth(n);
    const float ls_floor = (float)std::log((double)1e-4f);
    const float rop0 = (float)std::log(0.1 / 0.9);
    PcgInit rng(seed, 3);
    auto logit = [](float c) {
        const double v = std::min(std::max((double)c, 1e-4), 1.0 - 1e-4);
        return (float)std::log(v / (1.0 - v));
    };
    for (int64_t i = 0; i < n; ++i) {
        px[i] = xy[2 * i];
        py[i] = xy[2 * i + 1];
        const float l = scale[(size_t)i] > 0.0 ? (float)std::log(scale[(size_t)i]) : ls_floor;
        ls[i] = std::max(l, ls_floor);
        rop[i] = rop0;
        cr[i] = logit(rgb[3 * i]);
        cg[i] = logit(rgb[3 * i + 1]);
        cb[i] = logit(rgb[3 * i + 2]);
        depth[i] = (float)rng.uniform();
    }
    tgsx_host_scene s{};
    s.n = n;
    s.px = px.data(); s.py = py.data(); s.rot = rot.data(); s.lsx = ls.data(); s.lsy = ls.data();
    s.rop = rop.data(); s.cr = cr.data(); s.cg = cg.data(); s.cb = cb.data(); s.depth = depth.data();
    return tgsx_model_upload(ctx, m, &s);
}

}  // extern "C"
