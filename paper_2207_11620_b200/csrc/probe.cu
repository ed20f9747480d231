// L2 peaks for the encoder / scatter rooflines (MEASURED_PEAKS.json carries the
// HBM copy and tensor peaks only): streaming float4 reads of an L2-resident
// buffer, random 8-byte gathers and random float2 REDs into a 48 MB region (the
// cfg2 hash-table size).  Diagnostic only — bench.py calls it once to put a
// measured denominator under the L2-bound kernels.
#include "common.cuh"

namespace nvol {

__device__ __forceinline__ uint32_t probe_hash(uint32_t x) {
    x ^= x >> 16;
    x *= 0x7feb352dU;
    x ^= x >> 15;
    x *= 0x846ca68bU;
    x ^= x >> 16;
    return x;
}
__global__ void probe_stream(const float4 *a, int64_t n4, int reps, float *out) {
    float acc = 0.f;
    for (int r = 0; r < reps; ++r)
        for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
            const float4 v = __ldcg(a + j);
            acc += v.x + v.w;
        }
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void probe_gather(const float2 *a, uint32_t mask, int64_t n, float *out) {
    float acc = 0.f;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        acc += __ldg(a + (probe_hash((uint32_t)i) & mask)).x;
    if (acc == 1234.5f) out[0] = acc;
}
__global__ void probe_red(float2 *a, uint32_t mask, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(a + (probe_hash((uint32_t)i) & mask), make_float2(0.f, 0.f));
}

}  // namespace nvol

using namespace nvol;

// out[0] = L2 streaming read GB/s, out[1] = random 8-byte gathers G/s,
// out[2] = random float2 REDs G/s (best of 5, CUDA events).  Synchronous.
extern "C" int nvol_l2_probe(double *out) {
    NVOL_REQUIRE(out, "null pointer");
    const int64_t bytes = 48ll << 20, n = 32ll << 20;
    float4 *a = nullptr;
    float *o = nullptr;
    if (cudaMalloc(&a, bytes) != cudaSuccess || cudaMalloc(&o, 64) != cudaSuccess) {
        set_error("cudaMalloc failed");
        return NVOL_ECUDA;
    }
    cudaMemset(a, 0, bytes);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const uint32_t mask = (uint32_t)(bytes / 8 - 1);
    auto best = [&](int which) {
        float b = 1e30f;
        for (int r = 0; r < 6; ++r) {
            cudaEventRecord(e0);
            if (which == 0) probe_stream<<<sms * 8, 256>>>(a, bytes / 16, 10, o);
            if (which == 1) probe_gather<<<sms * 8, 256>>>(reinterpret_cast<const float2 *>(a), mask, n, o);
            if (which == 2) probe_red<<<sms * 8, 256>>>(reinterpret_cast<float2 *>(a), mask, n);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0.f;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 0 && ms < b) b = ms;  // first run warms L2
        }
        return (double)b * 1e-3;
    };
    out[0] = (double)bytes * 10 / best(0) / 1e9;
    out[1] = (double)n / best(1) / 1e9;
    out[2] = (double)n / best(2) / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(a);
    cudaFree(o);
    return check_launch("l2_probe");
}
