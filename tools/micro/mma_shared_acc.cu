// Correctness probe: W warps of one CTA issue tcgen05.mma chains (accumulate = 1) into the SAME
// TMEM accumulator concurrently.  A = B = fp16 1.0, so every MMA adds K = 16 to each element of
// the M128 x N64 accumulator; after W x C x k MMAs every element must equal 16 W C k exactly
// (integers below 2^24).  A lost or torn read-modify-write shows up as a smaller value.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_shared_acc.cu -o mma_shared_acc
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
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

__global__ void __launch_bounds__(256, 1) probe(int k, int chains, int warps, unsigned *bad, float *sample) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[8];
    __shared__ uint32_t tbase;
    const __half one = __float2half(1.0f);
    for (int i = threadIdx.x; i < 48 * 1024 / 2; i += blockDim.x) reinterpret_cast<__half *>(smem)[i] = one;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        for (int c = 0; c < 8; ++c) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[c])));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tbase;
    // zero the accumulator: warps 0-3 store zeros into their lane quarter (64 columns)
    if (warp < 4) {
        const uint32_t z = 0;
        for (int c = 0; c < 64; c += 8)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                             tm + ((uint32_t)(warp * 32) << 16) + c), "r"(z));
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t id = (1u << 4) | ((uint32_t)(64 >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    if (warp < warps) {
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        for (int c = 0; c < chains; ++c) {
            for (int i = 0; i < k; ++i) {
                const uint64_t ad = desc(a + (i & 3) * 256, 128, 1024), bd = desc(b + (i & 3) * 256, 128, 1024);
                asm volatile(
                    "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                    "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, 1;\n\t}\n" ::"r"(tm),
                    "l"(ad), "l"(bd), "r"(id));
            }
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                         smem_u32(&bar[warp])));
        asm volatile(
            "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(
                smem_u32(&bar[warp])));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp < 4) {
        const float want = 16.0f * warps * chains * k;
        for (int c = 0; c < 64; c += 8) {
            uint32_t r[8];
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                         : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            for (int e = 0; e < 8; ++e) {
                const float v = __uint_as_float(r[e]);
                if (v != want) atomicAdd(bad, 1u);
                if (blockIdx.x == 0 && warp == 0 && lane == 0 && c == 0 && e == 0) *sample = v;
            }
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tm));
}

int main() {
    unsigned *bad, hb;
    float *smp, hs;
    cudaMalloc(&bad, 4);
    cudaMalloc(&smp, 4);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int warps : {1, 2, 4, 8})
        for (int k : {1, 4, 12}) {
            unsigned tot = 0;
            for (int rep = 0; rep < 50; ++rep) {
                cudaMemset(bad, 0, 4);
                probe<<<148, 256, 64 * 1024>>>(k, 4, warps, bad, smp);
                cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost);
                tot += hb;
            }
            cudaMemcpy(&hs, smp, 4, cudaMemcpyDeviceToHost);
            printf("warps %d, 4 chains x %2d MMAs each into ONE accumulator: 50 x 148 CTAs, %u wrong elements (sample %.0f, want %.0f) %s\n",
                   warps, k, tot, hs, 16.0f * warps * 4 * k, cudaGetErrorString(cudaDeviceSynchronize()));
        }
}
