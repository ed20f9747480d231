// Microbenchmark: L2 reduction (RED) throughput on B200 for the encoder
// scatter design.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a red_bench.cu -o red_bench
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int V>
__global__ void red_random(float *g, uint32_t mask, int64_t n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = hash32((uint32_t)i) & mask;
        if (V == 1) atomicAdd(g + s, 1.0f);
        if (V == 2) atomicAdd(reinterpret_cast<float2 *>(g) + s, make_float2(1.f, 1.f));
        if (V == 4) atomicAdd(reinterpret_cast<float4 *>(g) + s, make_float4(1.f, 1.f, 1.f, 1.f));
    }
}

template <int V>
__global__ void ld_random(const float *g, uint32_t mask, int64_t n, float *out) {
    float acc = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        uint32_t s = hash32((uint32_t)i) & mask;
        if (V == 2) { float2 v = __ldg(reinterpret_cast<const float2 *>(g) + s); acc += v.x + v.y; }
        if (V == 4) { float4 v = __ldg(reinterpret_cast<const float4 *>(g) + s); acc += v.x + v.w; }
    }
    if (acc == 12345.f) out[0] = acc;
}

// every CTA adds `per` float4 into the same `per` addresses (the per-CTA flush pattern)
__global__ void red_contended(float *g, int per) {
    for (int q = threadIdx.x; q < per; q += blockDim.x)
        atomicAdd(reinterpret_cast<float4 *>(g) + q, make_float4(1.f, 1.f, 1.f, 1.f));
}
__global__ void red_contended1(float *g, int per) {
    for (int q = threadIdx.x; q < per * 4; q += blockDim.x) atomicAdd(g + q, 1.f);
}

int main() {
    float *g, *o;
    cudaMalloc(&g, 256 << 20);
    cudaMalloc(&o, 64);
    cudaMemset(g, 0, 256 << 20);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int64_t n = 8 << 20;
    auto time = [&](const char *name, auto fn, double ops) {
        fn();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int r = 0; r < 10; ++r) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        ms /= 10;
        printf("%-48s %8.2f us  %7.1f Gop/s\n", name, ms * 1e3, ops / (ms * 1e-3) / 1e9);
    };
    for (uint32_t region_mb : {4u, 48u}) {
        uint32_t m1 = (region_mb << 20) / 4 - 1, m2 = (region_mb << 20) / 8 - 1, m4 = (region_mb << 20) / 16 - 1;
        char nm[128];
        snprintf(nm, sizeof nm, "RED f32  random, %u MB region", region_mb);
        time(nm, [&] { red_random<1><<<148 * 8, 256>>>(g, m1, n); }, n);
        snprintf(nm, sizeof nm, "RED f32x2 random, %u MB region", region_mb);
        time(nm, [&] { red_random<2><<<148 * 8, 256>>>(g, m2, n); }, n);
        snprintf(nm, sizeof nm, "RED f32x4 random, %u MB region", region_mb);
        time(nm, [&] { red_random<4><<<148 * 8, 256>>>(g, m4, n); }, n);
        snprintf(nm, sizeof nm, "LD f32x2 random, %u MB region", region_mb);
        time(nm, [&] { ld_random<2><<<148 * 8, 256>>>(g, m2, n, o); }, n);
        snprintf(nm, sizeof nm, "LD f32x4 random, %u MB region", region_mb);
        time(nm, [&] { ld_random<4><<<148 * 8, 256>>>(g, m4, n, o); }, n);
    }
    time("RED f32x4 148 CTAs x 3600 same addresses", [&] { red_contended<<<148, 256>>>(g, 3600); }, 148.0 * 3600);
    time("RED f32 148 CTAs x 14400 same addresses", [&] { red_contended1<<<148, 256>>>(g, 3600); }, 148.0 * 14400);
    time("RED f32x4 148 CTAs x 2900 same addresses", [&] { red_contended<<<148, 1024>>>(g, 2900); }, 148.0 * 2900);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
}
