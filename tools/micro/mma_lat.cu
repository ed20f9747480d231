// Microbenchmark: latency structure of short tcgen05.mma chains (the MLP's layer phases).
// One CTA per SM, thread 0 issues.  For a chain of k MMAs (M = 128, N = 64, K = 16, SS,
// no swizzle) into one accumulator + commit, measures (clock64): the time to issue the chain
// (issue loop + commit), and the time until the commit's mbarrier completes.  Then C chains
// into C independent accumulators issued back to back before waiting on all of them: if the
// tensor pipe overlaps independent chains, C chains cost less than C x one chain.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a mma_lat.cu -o mma_lat
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
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
    return (1u << 4) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void __launch_bounds__(128, 1) lat(int k, int chains, int n, int reps, int one_commit, int acc_all, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar[8];
    __shared__ uint32_t tbase;
    for (int i = threadIdx.x; i < 64 * 1024 / 16; i += blockDim.x) reinterpret_cast<uint4 *>(smem)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
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
    if (threadIdx.x < 32) {  // warp 0 converged: uniform operands, one elected lane issues
        const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32768);
        const uint32_t id = idesc(128, n);
        unsigned long long s_issue = 0, s_done = 0;
        uint32_t par = 0;
        for (int r = 0; r < reps; ++r) {
            unsigned long long t0 = clock64();
            for (int c = 0; c < chains; ++c) {
                for (int i = 0; i < k; ++i) {
                    const int kk = i & 3;
                    const uint64_t ad = desc(a + kk * 256, 128, 1024), bd = desc(b + kk * 256, 128, 1024);
                    const uint32_t acc = (i > 0 || acc_all) ? 1u : 0u;
                    asm volatile(
                        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
                        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tm + c * 64),
                        "l"(ad), "l"(bd), "r"(id), "r"(acc));
                }
                if (!one_commit || c == chains - 1)
                    asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(
                        smem_u32(&bar[c])));
            }
            unsigned long long t1 = clock64();
            for (int c = one_commit ? chains - 1 : 0; c < chains; ++c)
                asm volatile(
                    "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(
                        smem_u32(&bar[c])), "r"(par));
            par ^= 1u;
            unsigned long long t2 = clock64();
            if (r > 0) {
                s_issue += t1 - t0;
                s_done += t2 - t0;
            }
        }
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            out[0] = s_issue / (reps - 1);
            out[1] = s_done / (reps - 1);
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

int main() {
    unsigned long long *d, h[2];
    cudaMalloc(&d, 16);
    cudaFuncSetAttribute(lat, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    for (int aa : {0, 2})
    for (int oc : {0, 1})
    for (int n : {64}) {
        for (int chains : {1, 2, 4}) {
            for (int k : {1, 2, 4, 8, 12}) {
                if (oc && chains == 1) continue;
                printf("%s%s", aa ? "alt-D   " : "zero-1st ", oc ? "one commit  " : "per-chain   ");
                lat<<<148, 128, 96 * 1024>>>(k, chains, n, 20, oc, aa, d);
                cudaError_t e = cudaDeviceSynchronize();
                cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
                printf("N=%3d chains %d x %2d MMAs: issue %6llu clk, complete %6llu clk (%6.1f clk/MMA)  %s\n", n, chains,
                       k, h[0], h[1], (double)h[1] / (chains * k), e ? cudaGetErrorString(e) : "");
            }
        }
    }
}
