// Microbenchmark: tcgen05.mma (kind::f16, cta_group::1, M = 128) issue rate for the MLP's
// operand shapes: SWIZZLE_NONE (core-matrix interleaved) vs SWIZZLE_128B K-major smem
// operands, N in {32, 64, 128, 256}, and A from TMEM.  One CTA per SM, one thread issues.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_bench.cu -o mma_bench
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)layout << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

template <int MODE>  // 0: SS no swizzle, 1: SS 128B swizzle, 2: A in TMEM (TS)
__global__ void __launch_bounds__(128, 1) bench(int n, int iters, unsigned long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t id = idesc(128, n);
        unsigned long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int k = i & 3;
            uint64_t ad, bd;
            if (MODE == 1) {  // K-major SW128: 8-row atoms of 1024 B, K step = 32 B inside the 128-B row
                ad = desc(a + k * 32, 16, 1024, 2);
                bd = desc(b + k * 32, 16, 1024, 2);
            } else {          // interleaved 8x8 core matrices: LBO = 128 (next K core matrix), SBO = rows of 8
                ad = desc(a + k * 256, 128, 1024, 0);
                bd = desc(b + k * 256, 128, 1024, 0);
            }
            const uint32_t acc = (i > 0) ? 1u : 0u;
            if (MODE == 2) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tm),
                    "r"(tm + 256 + k * 8), "l"(bd), "r"(id), "r"(acc));
            } else {
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm),
                    "l"(ad), "l"(bd), "r"(id), "r"(acc));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile(
            "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}\n" ::"r"(
                smem_u32(&bar)));
        unsigned long long t1 = clock64();
        if (blockIdx.x == 0) *cycles = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    unsigned long long *c;
    cudaMalloc(&c, 8);
    const int iters = 4096;
    for (int mode = 0; mode < 3; ++mode) {
        for (int n : {32, 64, 128, 256}) {
            if (mode == 2 && n > 256) continue;
            auto k = mode == 0 ? bench<0> : (mode == 1 ? bench<1> : bench<2>);
            cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
            k<<<148, 128, 96 * 1024>>>(n, iters, c);
            k<<<148, 128, 96 * 1024>>>(n, iters, c);
            cudaError_t e = cudaDeviceSynchronize();
            unsigned long long h = 0;
            cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
            const double cyc = (double)h / iters;
            const double macs = 128.0 * n * 16;
            printf("%-12s N=%3d: %6.1f cycles/MMA  %6.0f MAC/cycle/SM  (%s)\n",
                   mode == 0 ? "SS-noswz" : (mode == 1 ? "SS-sw128" : "TS(A tmem)"), n, cyc, macs / cyc,
                   cudaGetErrorString(e));
        }
    }
}
