// Microbenchmark: streaming Adam-like kernels over 4 x 12.2M floats (the cfg2 flat
// buffers), L2 flushed between reps.  nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void upd(float &p, float &g, float &m, float &v) {
    float ge = g + 1e-6f * p;
    m = 0.9f * m + 0.1f * ge;
    v = 0.99f * v + 0.01f * ge * ge;
    p = p - 0.005f * (m / 0.9f) / (sqrtf(v / 0.99f) + 1e-15f);
    g = 0.f;
}

template <int UNR>
__global__ void __launch_bounds__(256) adam_gs(float4 *p, float4 *g, float4 *m, float4 *v, int64_t n4) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += stride * UNR) {
        float4 P[UNR], G[UNR], M[UNR], V[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            int64_t k = j + u * stride;
            if (k < n4) { P[u] = __ldcs(p + k); G[u] = __ldcg(g + k); M[u] = __ldcs(m + k); V[u] = __ldcs(v + k); }
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            int64_t k = j + u * stride;
            if (k < n4) {
                upd(P[u].x, G[u].x, M[u].x, V[u].x); upd(P[u].y, G[u].y, M[u].y, V[u].y);
                upd(P[u].z, G[u].z, M[u].z, V[u].z); upd(P[u].w, G[u].w, M[u].w, V[u].w);
                __stcs(p + k, P[u]); __stcg(g + k, G[u]); __stcs(m + k, M[u]); __stcs(v + k, V[u]);
            }
        }
    }
}

// block-contiguous: each block owns a contiguous range and walks it
__global__ void __launch_bounds__(256) adam_blk(float4 *p, float4 *g, float4 *m, float4 *v, int64_t n4, int64_t per) {
    const int64_t b0 = (int64_t)blockIdx.x * per, b1 = min(n4, b0 + per);
    for (int64_t j = b0 + threadIdx.x; j < b1; j += blockDim.x) {
        float4 P = __ldcs(p + j), G = __ldcg(g + j), M = __ldcs(m + j), V = __ldcs(v + j);
        upd(P.x, G.x, M.x, V.x); upd(P.y, G.y, M.y, V.y); upd(P.z, G.z, M.z, V.z); upd(P.w, G.w, M.w, V.w);
        __stcs(p + j, P); __stcg(g + j, G); __stcs(m + j, M); __stcs(v + j, V);
    }
}

__global__ void copy4(const float4 *a, float4 *b, int64_t n4) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x)
        b[j] = a[j];
}
__global__ void flush(float4 *a, int64_t n4) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x)
        a[j] = make_float4(1, 2, 3, (float)j);
}

int main() {
    const int64_t n = 12181396, n4 = n / 4;
    float4 *p, *g, *m, *v, *fl;
    cudaMalloc(&p, n * 4); cudaMalloc(&g, n * 4); cudaMalloc(&m, n * 4); cudaMalloc(&v, n * 4);
    cudaMalloc(&fl, 512ll << 20);
    cudaMemset(p, 0, n * 4); cudaMemset(g, 0, n * 4); cudaMemset(m, 0, n * 4); cudaMemset(v, 0, n * 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto time = [&](const char *name, auto fn, double bytes) {
        float best = 1e9;
        for (int r = 0; r < 6; ++r) {
            flush<<<148 * 8, 256>>>(fl, (512ll << 20) / 16);
            cudaEventRecord(a); fn(); cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b); if (r > 0 && ms < best) best = ms;
        }
        printf("%-40s %8.2f us  %7.0f GB/s\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    const double adam_bytes = 32.0 * n;
    for (int blocks : {148 * 2, 148 * 4, 148 * 8, 148 * 16}) {
        char nm[64]; snprintf(nm, sizeof nm, "grid-stride x1, %d blocks", blocks);
        time(nm, [&] { adam_gs<1><<<blocks, 256>>>(p, g, m, v, n4); }, adam_bytes);
        snprintf(nm, sizeof nm, "grid-stride x2, %d blocks", blocks);
        time(nm, [&] { adam_gs<2><<<blocks, 256>>>(p, g, m, v, n4); }, adam_bytes);
    }
    for (int blocks : {148 * 4, 148 * 8, 148 * 32}) {
        char nm[64]; snprintf(nm, sizeof nm, "block-contiguous, %d blocks", blocks);
        int64_t per = (n4 + blocks - 1) / blocks;
        time(nm, [&] { adam_blk<<<blocks, 256>>>(p, g, m, v, n4, per); }, adam_bytes);
    }
    time("copy 195 MB -> 195 MB (2 of the buffers)", [&] { copy4<<<148 * 8, 256>>>(p, m, n4); copy4<<<148 * 8, 256>>>(g, v, n4); }, 16.0 * n);
    printf("status %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
