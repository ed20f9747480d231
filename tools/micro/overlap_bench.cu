// Microbenchmark: can the step's L2-operation-bound work (scatter REDs, encoder gathers) run
// beside its HBM-bound work (the Adam stream) without slowing either?  One kernel, warps split
// by role (HBM stream | L2 RED storm | L2 gather storm), each role's work fixed; the time of a
// role alone (same warps) against both together says whether the two resources are independent.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a overlap_bench.cu -o overlap_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

struct Args {
    float4 *p, *g, *m, *v;  // Adam-like stream: read 4, write 4 (n4 float4 each)
    int64_t n4;
    float *red;             // 48 MB RED region
    uint32_t red_mask;      // float2 slots
    int64_t n_red;
    const float *tab;       // 48 MB gather region
    uint32_t tab_mask;
    int64_t n_gat;
    float *sink;
};

// role: 0 = stream warps, 1 = RED warps, 2 = gather warps.  wsplit[r] = warps per CTA of role r
__global__ void mixed(Args a, int ws0, int ws1, int ws2) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int role, rw, nw;
    if (warp < ws0) { role = 0; rw = warp; nw = ws0; }
    else if (warp < ws0 + ws1) { role = 1; rw = warp - ws0; nw = ws1; }
    else { role = 2; rw = warp - ws0 - ws1; nw = ws2; }
    const int64_t tid = ((int64_t)blockIdx.x * nw + rw) * 32 + lane, nth = (int64_t)gridDim.x * nw * 32;
    if (role == 0) {
        for (int64_t i = tid; i < a.n4; i += nth) {
            float4 P = a.p[i], G = a.g[i], M = a.m[i], V = a.v[i];
            M.x = 0.9f * M.x + 0.1f * G.x; M.y = 0.9f * M.y + 0.1f * G.y; M.z = 0.9f * M.z + 0.1f * G.z; M.w = 0.9f * M.w + 0.1f * G.w;
            V.x = 0.999f * V.x + 0.001f * G.x * G.x; V.y = 0.999f * V.y + 0.001f * G.y * G.y;
            V.z = 0.999f * V.z + 0.001f * G.z * G.z; V.w = 0.999f * V.w + 0.001f * G.w * G.w;
            P.x -= M.x; P.y -= M.y; P.z -= M.z; P.w -= M.w;
            a.p[i] = P; a.m[i] = M; a.v[i] = V; a.g[i] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
    } else if (role == 1) {
        for (int64_t i = tid; i < a.n_red; i += nth) {
            const uint32_t s = hash32((uint32_t)i) & a.red_mask;
            atomicAdd(reinterpret_cast<float2 *>(a.red) + s, make_float2(1.f, 1.f));
        }
    } else {
        float acc = 0.f;
        for (int64_t i = tid; i < a.n_gat; i += nth) {
            const uint32_t s = hash32((uint32_t)i * 7u + 1u) & a.tab_mask;
            const float2 x = __ldg(reinterpret_cast<const float2 *>(a.tab) + s);
            acc += x.x + x.y;
        }
        if (acc == 1234.5f) a.sink[0] = acc;
    }
}

int main() {
    Args a;
    const int64_t nflat = 12181396;  // cfg2 flat parameters
    a.n4 = nflat / 4;
    cudaMalloc(&a.p, nflat * 4); cudaMalloc(&a.g, nflat * 4); cudaMalloc(&a.m, nflat * 4); cudaMalloc(&a.v, nflat * 4);
    cudaMemset(a.p, 0, nflat * 4); cudaMemset(a.g, 0, nflat * 4); cudaMemset(a.m, 0, nflat * 4); cudaMemset(a.v, 0, nflat * 4);
    cudaMalloc(&a.red, 64 << 20); cudaMemset(a.red, 0, 64 << 20);
    cudaMalloc((void **)&a.tab, 64 << 20); cudaMemset((void *)a.tab, 0, 64 << 20);
    cudaMalloc(&a.sink, 64);
    a.red_mask = (1u << 22) - 1;  // 4 M float2 = 32 MB
    a.tab_mask = (1u << 22) - 1;
    a.n_red = 65536LL * 13 * 8;   // the cfg2 scatter's global corner updates
    a.n_gat = 65536LL * 16 * 8;   // the cfg2 encoder's corner gathers
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    auto run = [&](const char *name, int w0, int w1, int w2, int ctas_per_sm) {
        Args b = a;
        if (!w0) b.n4 = 0;
        if (!w1) b.n_red = 0;
        if (!w2) b.n_gat = 0;
        const int th = 32 * (w0 + w1 + w2);
        const int grid = sms * ctas_per_sm;
        for (int r = 0; r < 2; ++r) mixed<<<grid, th>>>(b, w0, w1, w2);
        cudaDeviceSynchronize();
        float best = 1e9;
        for (int r = 0; r < 5; ++r) {
            cudaEventRecord(e0);
            mixed<<<grid, th>>>(b, w0, w1, w2);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            best = ms < best ? ms : best;
        }
        printf("%-44s warps %2d/%2d/%2d x %d CTA/SM  %8.1f us\n", name, w0, w1, w2, ctas_per_sm, best * 1e3);
    };
    for (int cps : {1, 2}) {
        run("stream only (Adam-like, 390 MB)", 16, 0, 0, cps);
        run("RED only (6.8 M float2 REDs, 32 MB)", 0, 16, 0, cps);
        run("gather only (8.4 M float2 loads, 32 MB)", 0, 0, 16, cps);
        run("stream 8 warps only", 8, 0, 0, cps);
        run("RED 8 warps only", 0, 8, 0, cps);
        run("gather 8 warps only", 0, 0, 8, cps);
        run("stream 8 + RED 8", 8, 8, 0, cps);
        run("stream 8 + gather 8", 8, 0, 8, cps);
        run("stream 4 only", 4, 0, 0, cps);
        run("RED 12 only", 0, 12, 0, cps);
        run("stream 4 + RED 12", 4, 12, 0, cps);
        run("gather 12 only", 0, 0, 12, cps);
        run("stream 4 + gather 12", 4, 0, 12, cps);
    }
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
