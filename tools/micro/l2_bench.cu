// L2 peaks for the encoder / scatter rooflines (MEASURED_PEAKS.json has HBM and
// tensor peaks only): streaming float4 reads of an L2-resident buffer, random
// 8-byte gathers and random float2 REDs into a 48 MB (cfg2 table-sized) region.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a l2_bench.cu -o l2_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}
__global__ void stream_rd(const float4 *a, int64_t n4, int reps, float *out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
            float4 v = __ldcg(a + j);
            acc += v.x + v.w;
        }
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void gather8(const float2 *a, uint32_t mask, int64_t n, float *out) {
    float acc = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        float2 v = __ldg(a + (hash32((uint32_t)i) & mask));
        acc += v.x;
    }
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void red8(float2 *a, uint32_t mask, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(a + (hash32((uint32_t)i) & mask), make_float2(1.f, 1.f));
}

int main() {
    const int64_t bytes = 48ll << 20;  // 48 MB: L2-resident, the cfg2 hash-table size
    float4 *a; float *o;
    cudaMalloc(&a, bytes); cudaMalloc(&o, 64); cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    auto time = [&](auto fn) {
        fn(); cudaDeviceSynchronize();
        float best = 1e30f;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0); fn(); cudaEventRecord(e1); cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1); best = ms < best ? ms : best;
        }
        return best;
    };
    const int reps = 20;
    float ms = time([&] { stream_rd<<<148 * 8, 256>>>(a, bytes / 16, reps, o); });
    printf("{\"l2_stream_read_gbs\": %.0f, ", (double)bytes * reps / (ms * 1e-3) / 1e9);
    const int64_t n = 64ll << 20;
    const uint32_t mask = (uint32_t)(bytes / 8 - 1) & 0x7fffff;  // 8M float2 entries
    ms = time([&] { gather8<<<148 * 8, 256>>>((const float2 *)a, mask, n, o); });
    printf("\"l2_gather8_gops\": %.1f, \"l2_gather8_sector_gbs\": %.0f, ", n / (ms * 1e-3) / 1e9, n * 32.0 / (ms * 1e-3) / 1e9);
    ms = time([&] { red8<<<148 * 8, 256>>>((float2 *)a, mask, n); });
    printf("\"l2_red8_gops\": %.1f, \"status\": \"%s\"}\n", n / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaDeviceSynchronize()));
}
