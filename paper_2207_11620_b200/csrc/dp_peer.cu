// Data-parallel gradient exchange fused with the optimizer, over peer memory.
//
// The sharded optimizer of distributed.py (reduce-scatter -> Adam on this rank's 1/G slice ->
// all-gather) as ONE kernel per rank that works directly in the other ranks' memory (NVLink P2P
// mappings of their buffers, opened through CUDA IPC): rank r reads its slice of every rank's
// flat gradient, sums the G contributions in rank order, applies the reference's Adam update
// (network.py:160-183, adam_one) to its slice, writes the updated parameters into every rank's
// parameter buffer and zeroes the slice of every rank's gradient -- no NCCL launches, no staging
// copies, the exchange streamed at the rate of the update itself.  Ordering across the ranks uses
// monotonic step flags in peer memory (system-scope release / acquire):
//   ready[j] = k + 1  rank j's gradient of step k is complete (dp_signal, after its scatter)
//   done[j]  = k + 1  rank j finished writing / zeroing its slices for step k (last block of the
//                     fused kernel); a rank's step k + 1 starts (dp_wait) only once every done >= k + 1
// The step's loss is the sum of the ranks' loss sums (read in rank order by the last block), and
// the NaN limit the minimum of the ranks' NaN states (nvol.h "NaN contract"), so every rank
// records the same loss, applies the same prefix and halts together.
#include <algorithm>
#include <cstdio>
#include <utility>

#include "common.cuh"

namespace nvol {

constexpr int DP_MAXG = 8;

struct PeerSet {
    float *g[DP_MAXG];           // flat gradient of rank j (unpadded view base)
    float *p[DP_MAXG];           // flat parameters of rank j
    const double *acc[DP_MAXG];  // loss sum of rank j
    const int64_t *nan[DP_MAXG]; // NaN state of rank j
    int64_t *ready[DP_MAXG];     // step flags of rank j: [0] ready, [1] done
};

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(int64_t *p, int64_t v) {
    asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// wait until *flag >= want (system-scope acquire); a peer that never gets there (a rank that died)
// traps the kernel after kPeerTimeoutNs instead of hanging the GPU
constexpr uint64_t kPeerTimeoutNs = 60ull * 1000 * 1000 * 1000;
__device__ __forceinline__ uint64_t global_ns() {
    uint64_t t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void wait_flag(const int64_t *flag, int64_t want, unsigned sleep_ns) {
    if (ld_acquire_sys(flag) >= want) return;
    const uint64_t t0 = global_ns();
    while (ld_acquire_sys(flag) < want) {
        __nanosleep(sleep_ns);
        if (global_ns() - t0 > kPeerTimeoutNs) {
            printf("nvol dp_peer: a peer's step flag stayed below %lld for 60 s\n", (long long)want);
            __trap();
        }
    }
}

// own ready flag = step + 1, after this rank's gradient (scatter + MLP flush) is complete
__global__ void dp_signal_kernel(int64_t *flags, const int64_t *counter, const int64_t *nan_state) {
    __threadfence_system();
    st_release_sys(flags, *counter + 1);
}

// before step k: every rank's slices of step k-1 are written (done >= k); then this rank's loss
// accumulator is free again (every rank has read it)
__global__ void dp_wait_kernel(PeerSet P, int G, const int64_t *counter, double *acc_own,
                               const int64_t *nan_state) {
    if (nan_halted(nan_state)) return;
    const int64_t k = *counter;
    for (int j = 0; j < G; ++j) wait_flag(P.ready[j] + 1, k, 256);
    *acc_own = 0.0;
}

__global__ void __launch_bounds__(256) dp_fused_adam_kernel(
    PeerSet P, int G, int64_t lo, int64_t hi, float *__restrict__ m, float *__restrict__ v,
    const float *__restrict__ sched, int64_t sched_len, int64_t *__restrict__ step_counter, float b1, float omb1,
    float b2, float omb2, float eps, float l2, int64_t *__restrict__ nan_state, double *__restrict__ losses,
    int64_t t0, int64_t cap, double inv_b, uint32_t *__restrict__ ticket, int64_t *__restrict__ own_flags) {
    __shared__ int64_t s_lim;
    if (nan_halted(nan_state)) return;
    const int64_t tc = *step_counter;
    if (threadIdx.x == 0) {
        int64_t lim = kNanNone;
        for (int j = 0; j < G; ++j) {
            wait_flag(P.ready[j], tc + 1, 128);  // rank j's gradient of this step
            lim = min(lim, ld_acquire_sys(P.nan[j]));
        }
        s_lim = lim;
    }
    __syncthreads();
    const int64_t lim = s_lim;
    const int64_t t = tc >= sched_len ? sched_len - 1 : tc;
    const float lr = sched[3 * t], c1 = sched[3 * t + 1], c2 = sched[3 * t + 2];
    // one element: the ranks' contributions summed in rank order, the update written to every rank
    auto one = [&](int64_t q, float g, float &pp) -> bool {
        if (q >= lim) return false;
        if (isnan(g)) {
            // a NaN that only the sum produces (inf + -inf across ranks): every rank's limit drops,
            // so all of them halt at their next step
            for (int j = 0; j < G; ++j) atomicMin(reinterpret_cast<unsigned long long *>(const_cast<int64_t *>(P.nan[j])),
                                                  (unsigned long long)q);
            return false;
        }
        float mm = m[q], vv = v[q];
        adam_one<float>(pp, g, mm, vv, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        m[q] = mm;
        v[q] = vv;
        return true;
    };
    // 16-byte body over NVLink (the slice bounds are 128-byte aligned except the last rank's end;
    // every rank's flat buffers share their alignment), scalar tail
    const int64_t body_end = lo + ((hi - lo) & ~(int64_t)3);
    const bool vec = ((reinterpret_cast<uintptr_t>(P.g[0] + lo) | reinterpret_cast<uintptr_t>(P.p[0] + lo)) & 15) == 0;
    const int64_t vend = vec ? body_end : lo;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t q = lo + 4 * ((int64_t)blockIdx.x * blockDim.x + threadIdx.x); q < vend; q += 4 * stride) {
        float4 g4 = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
        for (int j = 0; j < G; ++j) {
            const float4 c = __ldcv(reinterpret_cast<const float4 *>(P.g[j] + q));
            g4 = make_float4(xadd(g4.x, c.x), xadd(g4.y, c.y), xadd(g4.z, c.z), xadd(g4.w, c.w));
        }
        float4 p4 = __ldcv(reinterpret_cast<const float4 *>(P.p[0] + q));  // this rank's own current value
        const bool u0 = one(q, g4.x, p4.x), u1 = one(q + 1, g4.y, p4.y), u2 = one(q + 2, g4.z, p4.z),
                   u3 = one(q + 3, g4.w, p4.w);
        if (u0 & u1 & u2 & u3) {
            for (int j = 0; j < G; ++j) __stcg(reinterpret_cast<float4 *>(P.p[j] + q), p4);
        } else {
            const float pv[4] = {p4.x, p4.y, p4.z, p4.w};
            const bool uv[4] = {u0, u1, u2, u3};
            for (int e = 0; e < 4; ++e)
                if (uv[e])
                    for (int j = 0; j < G; ++j) __stcg(P.p[j] + q + e, pv[e]);
        }
        for (int j = 0; j < G; ++j) __stcg(reinterpret_cast<float4 *>(P.g[j] + q), make_float4(0.0f, 0.0f, 0.0f, 0.0f));
    }
    for (int64_t q = vend + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < hi; q += stride) {
        float g = 0.0f;
        for (int j = 0; j < G; ++j) g = xadd(g, __ldcv(P.g[j] + q));
        float pp = __ldcv(P.p[0] + q);
        if (one(q, g, pp))
            for (int j = 0; j < G; ++j) __stcg(P.p[j] + q, pp);
        for (int j = 0; j < G; ++j) __stcg(P.g[j] + q, 0.0f);
    }
    __threadfence_system();  // every thread's peer stores, before the block's ticket / done flag
    __syncthreads();
    if (threadIdx.x == 0) {
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {  // the last block: every block's writes are out
            __threadfence_system();
            *ticket = 0u;
            double loss = 0.0;
            for (int j = 0; j < G; ++j) loss += *reinterpret_cast<const volatile double *>(P.acc[j]);
            if (lim != kNanNone) {
                nan_state[0] = lim;
                nan_state[1] = 1;  // halt (every rank sees the same limit)
                st_release_sys(own_flags + 1, tc + 1);
                return;
            }
            const int64_t kk = tc - t0;
            if (losses && kk >= 0 && kk < cap) losses[kk] = loss * inv_b;
            *step_counter = tc + 1;
            st_release_sys(own_flags + 1, tc + 1);
        }
    }
}

static int fill_peers(PeerSet &P, int G, const int64_t *g, const int64_t *p, const int64_t *acc, const int64_t *nan,
                      const int64_t *flags) {
    NVOL_REQUIRE(G >= 1 && G <= DP_MAXG, "peer exchange: 1..8 ranks");
    for (int j = 0; j < G; ++j) {
        NVOL_REQUIRE(g[j] && p[j] && acc[j] && nan[j] && flags[j], "peer exchange: null peer pointer");
        P.g[j] = reinterpret_cast<float *>(g[j]);
        P.p[j] = reinterpret_cast<float *>(p[j]);
        P.acc[j] = reinterpret_cast<const double *>(acc[j]);
        P.nan[j] = reinterpret_cast<const int64_t *>(nan[j]);
        P.ready[j] = reinterpret_cast<int64_t *>(flags[j]);
    }
    return NVOL_OK;
}

}  // namespace nvol

using namespace nvol;

extern "C" {

int nvol_dp_signal(int64_t *own_flags, const int64_t *step_counter, const int64_t *nan_state, void *stream) {
    NVOL_REQUIRE(own_flags && step_counter, "null pointer");
    dp_signal_kernel<<<1, 1, 0, as_stream(stream)>>>(own_flags, step_counter, nan_state);
    return check_launch("dp_signal");
}

int nvol_dp_wait(int32_t world, const int64_t *flags, const int64_t *step_counter, double *own_loss_acc,
                 const int64_t *nan_state, void *stream) {
    NVOL_REQUIRE(world >= 1 && world <= DP_MAXG && flags && step_counter && own_loss_acc, "bad arguments");
    PeerSet P{};
    for (int j = 0; j < world; ++j) P.ready[j] = reinterpret_cast<int64_t *>(flags[j]);
    dp_wait_kernel<<<1, 1, 0, as_stream(stream)>>>(P, world, step_counter, own_loss_acc, nan_state);
    return check_launch("dp_wait");
}

int nvol_dp_fused_adam(int32_t world, int32_t rank, const int64_t *grads, const int64_t *params, const int64_t *loss_accs,
                       const int64_t *nan_states, const int64_t *flags, int64_t lo, int64_t hi, float *m, float *v,
                       const float *sched, int64_t sched_len, int64_t *step_counter, float beta1,
                       float one_minus_beta1, float beta2, float one_minus_beta2, float eps, float l2,
                       int64_t *nan_state, double *losses, int64_t t0, int64_t cap, double inv_b, uint32_t *ticket,
                       void *stream) {
    PeerSet P{};
    int st = fill_peers(P, world, grads, params, loss_accs, nan_states, flags);
    if (st) return st;
    NVOL_REQUIRE(rank >= 0 && rank < world && lo >= 0 && hi >= lo && m && v && sched && step_counter && ticket,
                 "bad arguments");
    // rank's own parameters first: the kernel reads the current value of its slice from P.p[0]
    std::swap(P.p[0], P.p[rank]);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t n = hi - lo;
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((n / 4 + 255) / 256, (int64_t)sms * 8));
    dp_fused_adam_kernel<<<grid, 256, 0, as_stream(stream)>>>(P, world, lo, hi, m, v, sched, sched_len, step_counter,
                                                              beta1, one_minus_beta1, beta2, one_minus_beta2, eps, l2,
                                                              nan_state, losses, t0, cap, inv_b, ticket,
                                                              reinterpret_cast<int64_t *>(flags[rank]));
    return check_launch("dp_fused_adam");
}

}  // extern "C"
