// TEST INFRASTRUCTURE: exhaustive-style check of the product's interval box mask
// (paper_2412_13547_b200/csrc/tgsx_device.cuh box_mask) against the per-column box test of
// rasterizer.cpp:116-118 restated literally (box_column_loop below), on hashed random splats
// including boxes whose edges fall exactly on (or one ulp beside) active pixel centres.
// Usage: box_mask_check <log2 cases>; prints "tested N mismatches M".
#include <cstdio>
#include <cstdlib>
#include "tgsx_device.cuh"

using namespace tgsx;

__device__ uint32_t box_column_loop(float m, float r, int a0, int p, int count) {
    uint32_t mask = 0;
    for (int c = 0; c < 16; ++c) {
        const float d = __fsub_rn(__fadd_rn((float)(a0 + c * p), 0.5f), m);  // (px + 0.5) - mean
        mask |= (c < count && fabsf(d) <= r) ? (1u << c) : 0u;
    }
    return mask;
}

__device__ uint32_t mix(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
    return x;
}

__global__ void check(unsigned long long* bad, unsigned long long n) {
    for (unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; i < n;
         i += gridDim.x * (unsigned long long)blockDim.x) {
        const uint32_t h1 = mix((uint32_t)i * 3u + 1u), h2 = mix((uint32_t)i * 3u + 2u), h3 = mix((uint32_t)i * 3u + 3u);
        const int p = 1 + (int)(h1 % 4u);
        const int a0 = (int)((h1 >> 4) % 300u) * 16 + (int)((h1 >> 12) % (uint32_t)p);
        const int count = (int)((h1 >> 20) % 17u);
        const float u = (float)(h2 >> 8) / 16777216.0f, v = (float)h3 / 4294967296.0f;
        float m, r;
        switch (h2 % 4u) {
        case 0:  // generic
            m = (float)a0 - 30.f + u * 100.f;
            r = v * 40.f;
            break;
        case 1: {  // both edges exactly on active pixel centres
            const int c1 = (int)(u * 20.f) - 2, c2 = c1 + (int)(v * 8.f);
            const float x1 = (float)(a0 + c1 * p) + 0.5f, x2 = (float)(a0 + c2 * p) + 0.5f;
            m = 0.5f * (x1 + x2);
            r = 0.5f * (x2 - x1);
            break;
        }
        case 2:  // radius one ulp around a value
            m = (float)a0 + u * 16.f * (float)p;
            r = __uint_as_float(__float_as_uint(v * 8.f) + (h3 & 3u) - 1u);
            break;
        default:  // mean within 1e-5 of a centre, integral radius +- 1e-6
            m = (float)(a0 + (int)(u * 16.f) * p) + 0.5f + (v - 0.5f) * 1e-5f;
            r = fmaxf(0.f, (float)((h3 >> 3) % 5u) * (float)p + ((h3 & 1u) ? 1e-6f : -1e-6f));
        }
        if (box_mask(m, r, a0, p, count) != box_column_loop(m, r, a0, p, count)) atomicAdd(bad, 1ull);
    }
}

int main(int argc, char** argv) {
    const int lg = argc > 1 ? atoi(argv[1]) : 28;
    unsigned long long* d = nullptr;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    const unsigned long long n = 1ull << lg;
    check<<<148 * 16, 256>>>(d, n);
    unsigned long long h = ~0ull;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const cudaError_t e = cudaGetLastError();
    printf("tested %llu mismatches %llu\n", n, h);
    return (e == cudaSuccess && h == 0) ? 0 : 1;
}
