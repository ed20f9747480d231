// Microbenchmark: do tcgen05.mma chains issued by DIFFERENT warps of one CTA overlap in the
// tensor pipe?  W warps each issue C chains of k MMAs (M = 128, N = 64, K = 16, SS, no swizzle,
// distinct accumulators, distinct A operands) + one commit per chain, then wait for them; the
// CTA's total time against W = 1.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_par.cu -o mma_par
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

__global__ void __launch_bounds__(256, 1) par(int k, int chains, int warps, int reps, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[8][8];
    __shared__ uint32_t tbase;
    __shared__ unsigned long long tmax;
    for (int i = threadIdx.x; i < 160 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int w = 0; w < 8; ++w)
            for (int c = 0; c < 8; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][c])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    const uint32_t id = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    unsigned long long total = 0;
    uint32_t par = 0;
    for (int r = 0; r < reps; ++r) {
        __syncthreads();
        unsigned long long t0 = clock64();
        if (warp < warps) {
            for (int c = 0; c < chains; ++c) {
                const int slot = warp * chains + c;  // distinct accumulator + A operand per chain
                const uint32_t a = smem_u32(smem) + slot * 16384, b = smem_u32(smem + 131072);
                for (int i = 0; i < k; ++i) {
                    const uint64_t ad = desc(a + (i & 3) * 256, 128, 1024), bd = desc(b + (i & 3) * 256, 128, 1024);
                    asm volatile(
                        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + slot * 64),
                        "l"(ad), "l"(bd), "r"(id), "r"(i > 0 ? 1u : 0u));
                }
                asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                             "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                                 smem_u32(&bar[warp][c])));
            }
            for (int c = 0; c < chains; ++c)
                asm volatile(
                    "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(
                        smem_u32(&bar[warp][c])), "r"(par));
        }
        par ^= 1u;
        __syncthreads();
        unsigned long long t1 = clock64();
        if (r > 0) total += t1 - t0;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *out = total / (reps - 1);
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    unsigned long long *d, h;
    cudaMalloc(&d, 8);
    cudaFuncSetAttribute(par, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
    for (int k : {4, 12}) {
        for (int warps : {1, 2, 4}) {
            for (int chains : {1, 2}) {
                par<<<148, 256, 160 * 1024>>>(k, chains, warps, 20, d);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                printf("k=%2d MMAs/chain, %d warps x %d chains: %6llu clk total (%6.1f clk/chain) %s\n", k, warps, chains, h,
                       (double)h / (warps * chains), e ? cudaGetErrorString(e) : "");
            }
        }
    }
}
