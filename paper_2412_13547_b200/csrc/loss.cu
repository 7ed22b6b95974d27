// compute_loss on the device (loss.cpp is missing from the reference, the
// restatement is oracle/tgs_oracle.c or_loss): dense iterations (p = 1) use
// L = (1 - lam) L1 + lam (1 - SSIM) with the 11x11 Gaussian-window (sigma 1.5) SSIM, zero
// padding, C1 = 0.01^2, C2 = 0.03^2; dilated iterations L1 only.
//
//  l1_kernel          L1 over the active pixels of given colours (the fit step fuses this into
//                     the forward epilogue instead): sign gradient * scale, per-block |d| sums.
//  ssim_stats_kernel  per 32x16 output tile and channel: the five windowed moments of x, y
//                     (separable 11-tap passes over a haloed shared-memory tile), the SSIM map
//                     S and the per-pixel adjoint weights a = dS/dmu_x - 2 mu_x dS/dsxx -
//                     mu_y dS/dsxy, b = dS/dsxx, c = dS/dsxy; per-block sums of S.
//  ssim_grad_kernel   dL/dx += -lam/(3P) [(G*a) + 2 x (G*b) + y (G*c)] (the window is symmetric,
//                     so the adjoint of the zero-padded convolution is the same convolution).
// Block partial sums are reduced in a fixed order: the loss value is deterministic.
#include "tgsx_device.cuh"
#include "tgsx_internal.h"

#include <algorithm>
#include <cmath>

namespace tgsx {

namespace {

constexpr int kR = 5;                 // window radius (11 taps)
constexpr int kTW = 32, kTH = 16;     // output tile
constexpr int kHW = kTW + 2 * kR, kHH = kTH + 2 * kR;

__constant__ float c_win[2 * kR + 1];

__global__ void __launch_bounds__(256) l1_kernel(const float* __restrict__ rgb, const float* __restrict__ target,
                                                 int p, int ox, int oy, int W, int cols, int64_t P,
                                                 float scale, float* __restrict__ dLdC,
                                                 float* __restrict__ block_sum) {
    __shared__ float s[8];
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    float acc = 0.f;
    if (r < P) {
        const int x = ox + (int)(r % cols) * p, y = oy + (int)(r / cols) * p;
        const float* t = target + 3 * ((int64_t)y * W + x);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float d = rgb[3 * r + c] - t[c];
            acc += fabsf(d);
            dLdC[3 * r + c] = d > 0.f ? scale : (d < 0.f ? -scale : 0.f);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += s[w];
        block_sum[blockIdx.x] = t;
    }
}

// Separable windowed sums of NM maps over a haloed tile: in[m][kHH][kHW] -> out[m][kTH][kTW].
// Register blocking: a horizontal work item produces 4 consecutive outputs from 14 loads, a
// thread's vertical pass produces 2 consecutive rows from 12 loads (the shared-memory pipe, not
// the FMA pipe, bounds the naive one-load-per-tap form).
template <int NM>
__device__ __forceinline__ void window_sums(const float (*in)[kHH][kHW], float (*hs)[kHH][kTW],
                                            int tid, float (&out)[2][NM]) {
    constexpr int kQ = kTW / 4;  // 4-wide column groups per row
    for (int i = tid; i < kHH * kQ; i += 256) {
        const int yy = i / kQ, x0 = 4 * (i % kQ);
#pragma unroll
        for (int m = 0; m < NM; ++m) {
            float v[4 + 2 * kR];
#pragma unroll
            for (int j = 0; j < 4 + 2 * kR; ++j) v[j] = in[m][yy][x0 + j];
#pragma unroll
            for (int o = 0; o < 4; ++o) {
                float acc = 0.f;
#pragma unroll
                for (int k = 0; k <= 2 * kR; ++k) acc = fmaf(c_win[k], v[o + k], acc);
                hs[m][yy][x0 + o] = acc;
            }
        }
    }
    __syncthreads();
    // each thread: two vertically consecutive output pixels (rows 2 ty, 2 ty + 1)
    const int tx = tid % kTW, ty = tid / kTW;
#pragma unroll
    for (int m = 0; m < NM; ++m) {
        float v[2 + 2 * kR];
#pragma unroll
        for (int j = 0; j < 2 + 2 * kR; ++j) v[j] = hs[m][2 * ty + j][tx];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k <= 2 * kR; ++k) acc = fmaf(c_win[k], v[h + k], acc);
            out[h][m] = acc;
        }
    }
}

__global__ void __launch_bounds__(256) ssim_stats_kernel(const float* __restrict__ rgb,
                                                         const float* __restrict__ target, int W, int H,
                                                         float* __restrict__ abc, float* __restrict__ block_sum) {
    __shared__ float in[5][kHH][kHW];  // x, y, x^2, y^2, x y
    __shared__ float hs[5][kHH][kTW];
    __shared__ float red[8];
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * kTW - kR, y0 = blockIdx.y * kTH - kR;
    const float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;
    float ssum = 0.f;
    for (int ch = 0; ch < 3; ++ch) {
        for (int i = tid; i < kHH * kHW; i += 256) {
            const int yy = i / kHW, xx = i % kHW, gx = x0 + xx, gy = y0 + yy;
            float a = 0.f, b = 0.f;
            if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
                const int64_t q = 3 * ((int64_t)gy * W + gx) + ch;
                a = rgb[q];
                b = target[q];
            }
            in[0][yy][xx] = a;
            in[1][yy][xx] = b;
            in[2][yy][xx] = a * a;
            in[3][yy][xx] = b * b;
            in[4][yy][xx] = a * b;
        }
        __syncthreads();
        float st[2][5];
        window_sums<5>(in, hs, tid, st);
        const int tx = tid % kTW, ty = tid / kTW;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gx = blockIdx.x * kTW + tx, gy = blockIdx.y * kTH + 2 * ty + h;
            if (gx >= W || gy >= H) continue;
            const float mx = st[h][0], my = st[h][1];
            const float sxx = st[h][2] - mx * mx, syy = st[h][3] - my * my, sxy = st[h][4] - mx * my;
            const float A1 = 2.f * mx * my + C1, A2 = 2.f * sxy + C2;
            const float B1 = mx * mx + my * my + C1, B2 = sxx + syy + C2;
            const float iB = 1.f / (B1 * B2);
            const float S = A1 * A2 * iB;
            ssum += S;
            const float dmu = 2.f * my * A2 * iB - 2.f * mx * S / B1;
            const float dsxx = -S / B2, dsxy = 2.f * A1 * iB;
            float* o = abc + 9 * ((int64_t)gy * W + gx) + 3 * ch;
            o[0] = dmu - 2.f * mx * dsxx - my * dsxy;
            o[1] = dsxx;
            o[2] = dsxy;
        }
        __syncthreads();
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) ssum += __shfl_xor_sync(0xffffffffu, ssum, o);
    if ((tid & 31) == 0) red[tid >> 5] = ssum;
    __syncthreads();
    if (tid == 0) {
        float t = 0.f;
        for (int w = 0; w < 8; ++w) t += red[w];
        block_sum[blockIdx.y * gridDim.x + blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(256) ssim_grad_kernel(const float* __restrict__ rgb,
                                                        const float* __restrict__ target, int W, int H,
                                                        const float* __restrict__ abc, float scale,
                                                        float* __restrict__ dLdC) {
    __shared__ float in[3][kHH][kHW];
    __shared__ float hs[3][kHH][kTW];
    const int tid = threadIdx.x;
    const int x0 = blockIdx.x * kTW - kR, y0 = blockIdx.y * kTH - kR;
    for (int ch = 0; ch < 3; ++ch) {
        for (int i = tid; i < kHH * kHW; i += 256) {
            const int yy = i / kHW, xx = i % kHW, gx = x0 + xx, gy = y0 + yy;
            float a = 0.f, b = 0.f, c = 0.f;
            if (gx >= 0 && gx < W && gy >= 0 && gy < H) {
                const float* s = abc + 9 * ((int64_t)gy * W + gx) + 3 * ch;
                a = s[0];
                b = s[1];
                c = s[2];
            }
            in[0][yy][xx] = a;
            in[1][yy][xx] = b;
            in[2][yy][xx] = c;
        }
        __syncthreads();
        float g[2][3];
        window_sums<3>(in, hs, tid, g);
        const int tx = tid % kTW, ty = tid / kTW;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int gx = blockIdx.x * kTW + tx, gy = blockIdx.y * kTH + 2 * ty + h;
            if (gx >= W || gy >= H) continue;
            const int64_t q = 3 * ((int64_t)gy * W + gx) + ch;
            dLdC[q] -= scale * (g[h][0] + 2.f * rgb[q] * g[h][1] + target[q] * g[h][2]);
        }
        __syncthreads();
    }
}

// loss = w1 * sum(|d|) + lam * (1 - inv * sum(S)), sums in a fixed order (double)
__global__ void loss_finalize_kernel(const float* __restrict__ l1_part, int n1, float w1,
                                     const float* __restrict__ s_part, int n2, float lam, double inv,
                                     float* __restrict__ out) {
    __shared__ double sa[256], sb[256];
    double a = 0.0, b = 0.0;
    for (int i = threadIdx.x; i < n1; i += 256) a += (double)l1_part[i];
    for (int i = threadIdx.x; i < n2; i += 256) b += (double)s_part[i];
    sa[threadIdx.x] = a;
    sb[threadIdx.x] = b;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            sa[threadIdx.x] += sa[threadIdx.x + w];
            sb[threadIdx.x] += sb[threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        double l = (double)w1 * sa[0];
        if (n2 > 0) l += (double)lam * (1.0 - inv * sb[0]);
        out[0] = (float)l;
    }
}

bool g_window_ready = false;

cudaError_t upload_window() {
    if (g_window_ready) return cudaSuccess;
    float w[2 * kR + 1];
    double g[2 * kR + 1], s = 0.0;
    for (int i = -kR; i <= kR; ++i) {
        g[i + kR] = std::exp(-(double)(i * i) / (2.0 * 1.5 * 1.5));
        s += g[i + kR];
    }
    for (int i = 0; i <= 2 * kR; ++i) w[i] = (float)(g[i] / s);
    cudaError_t e = cudaMemcpyToSymbol(c_win, w, sizeof(w));
    if (!e) g_window_ready = true;
    return e;
}

}  // namespace

cudaError_t launch_l1(tgsx_ctx* ctx, const RenderArgs& ra, const float* rgb, float scale, float* dLdC,
                      float* block_sum, int* nblocks) {
    const int64_t P = ra.P;
    *nblocks = (int)((P + 255) / 256);
    if (P == 0) return cudaSuccess;
    l1_kernel<<<(unsigned)*nblocks, 256, 0, ctx->stream>>>(rgb, ra.target, ra.p, ra.ox, ra.oy, ra.W, ra.cols,
                                                           P, scale, dLdC, block_sum);
    ctx->launches++;
    return cudaGetLastError();
}

size_t ssim_blocks(int W, int H) {
    return (size_t)((W + kTW - 1) / kTW) * (size_t)((H + kTH - 1) / kTH);
}

cudaError_t launch_ssim(tgsx_ctx* ctx, const float* rgb, const float* target, int W, int H, float lam,
                        float* abc, float* block_sum, float* dLdC) {
    cudaError_t e = upload_window();
    if (e) return e;
    const dim3 grid((W + kTW - 1) / kTW, (H + kTH - 1) / kTH);
    ssim_stats_kernel<<<grid, 256, 0, ctx->stream>>>(rgb, target, W, H, abc, block_sum);
    ctx->launches++;
    if ((e = cudaGetLastError())) return e;
    const float scale = (float)((double)lam / (3.0 * (double)W * (double)H));
    ssim_grad_kernel<<<grid, 256, 0, ctx->stream>>>(rgb, target, W, H, abc, scale, dLdC);
    ctx->launches++;
    return cudaGetLastError();
}

cudaError_t launch_loss_finalize(tgsx_ctx* ctx, const float* l1_part, int n1, float w1, const float* s_part,
                                 int n2, float lam, double inv, float* out) {
    loss_finalize_kernel<<<1, 256, 0, ctx->stream>>>(l1_part, n1, w1, s_part, n2, lam, inv, out);
    ctx->launches++;
    return cudaGetLastError();
}

}  // namespace tgsx

// ---------------------------------------------------------------- FP32 peak microbenchmark
// Roofline denominator for the blend kernels ("add a measured FFMA
// microbenchmark peak"): 8 independent FMA chains per thread, scalar FFMA or packed FFMA2,
// grid = 8 CTAs x 256 threads per SM; timed with CUDA events on the context stream.
namespace tgsx {
namespace {
template <bool PACKED>
__global__ void __launch_bounds__(256) fp32_peak_kernel(float* out, int iters, float a, float b) {
    float2 x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = make_float2((float)(threadIdx.x + j), (float)(blockIdx.x - j));
    const float2 av = make_float2(a, a), bv = make_float2(b, b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (PACKED) {
                x[j] = __ffma2_rn(x[j], av, bv);
            } else {
                x[j].x = __fmaf_rn(x[j].x, a, b);
                x[j].y = __fmaf_rn(x[j].y, a, b);
            }
        }
    }
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) s += x[j].x + x[j].y;
    if (s == 1234.5f) out[0] = s;  // never true: keeps the chains live
}
}  // namespace
}  // namespace tgsx

extern "C" int32_t tgsx_measure_fp32_peak(tgsx_ctx* ctx, double* out_ffma_tflops, double* out_ffma2_tflops) {
    using namespace tgsx;
    if (!ctx) return TGSX_EINVAL;
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        return TGSX_ECUDA;
    if (ctx->ws.generic.ensure(64) != cudaSuccess) return TGSX_ECUDA;
    float* out = ctx->ws.generic.as<float>();
    const unsigned blocks = (unsigned)sms * 8u;
    const int iters = 4096;
    const double flops = 2.0 * 16.0 * iters * (double)blocks * 256.0;  // 16 FMAs per iteration
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double res[2] = {0.0, 0.0};
    for (int packed = 0; packed < 2; ++packed) {
        for (int rep = 0; rep < 3; ++rep) {  // first repetition warms up
            cudaEventRecord(e0, ctx->stream);
            if (packed) fp32_peak_kernel<true><<<blocks, 256, 0, ctx->stream>>>(out, iters, 0.999f, 1e-3f);
            else fp32_peak_kernel<false><<<blocks, 256, 0, ctx->stream>>>(out, iters, 0.999f, 1e-3f);
            cudaEventRecord(e1, ctx->stream);
            ctx->launches++;
            if (cudaEventSynchronize(e1) != cudaSuccess) return TGSX_ECUDA;
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (rep) res[packed] = std::max(res[packed], flops / (ms * 1e-3) / 1e12);
        }
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (out_ffma_tflops) *out_ffma_tflops = res[0];
    if (out_ffma2_tflops) *out_ffma2_tflops = res[1];
    return cudaGetLastError() == cudaSuccess ? TGSX_OK : TGSX_ECUDA;
}
