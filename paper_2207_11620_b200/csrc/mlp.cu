// Generic (any width / depth / dtype) MLP forward + backward, loss and Adam.
//
// Reference: network.py:61-93 (Mlp.forward / backward, numpy sgemm),
// network.py:96-114 (loss_and_grad), network.py:160-183 (adam_step).
// These kernels back the reference-shaped API (float32 and the float64
// gradient-check builds); the training hot path uses the fused kernels in
// train_fused.cu instead.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace nvol {

// C[M,N] (=|+=) op(A)[M,K] * op(B)[K,N], optional ReLU.  64x64 tiles,
// 256 threads, 4x4 outputs per thread, k-tile 16.  gridDim.z > 1 splits K
// and accumulates with atomics (used for the dW reductions over the batch).
template <typename T, bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_kernel(int64_t M, int64_t N, int64_t K, const T *__restrict__ A,
                                                   int64_t lda, const T *__restrict__ B, int64_t ldb,
                                                   T *__restrict__ C, int64_t ldc, int accumulate, int relu,
                                                   T *__restrict__ partials) {
    // rows padded to 68 elements: 16-byte aligned vector reads of a thread's 4 consecutive m / n
    __shared__ __align__(16) T As[16][64 + 4];
    __shared__ __align__(16) T Bs[16][64 + 4];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int64_t m0 = (int64_t)blockIdx.y * 64, n0 = (int64_t)blockIdx.x * 64;
    const int64_t kchunk = (K + gridDim.z - 1) / gridDim.z;
    const int64_t kbeg = (int64_t)blockIdx.z * kchunk;
    const int64_t kend = min(K, kbeg + kchunk);
    T acc[4][4];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[a][c] = (T)0;
    for (int64_t k0 = kbeg; k0 < kend; k0 += 16) {
        for (int q = threadIdx.x; q < 16 * 64; q += 256) {
            // consecutive threads walk the operand's contiguous dimension (k for a row-major A /
            // transposed B, m / n otherwise), so every warp load is a few full sectors
            const int ka = TA ? q / 64 : q % 16, ma = TA ? q % 64 : q / 16;
            const int64_t gm = m0 + ma, gka = k0 + ka;
            T va = (T)0;
            if (gm < M && gka < kend) va = TA ? A[gka * lda + gm] : A[gm * lda + gka];
            As[ka][ma] = va;
            const int kb = TB ? q % 16 : q / 64, nb = TB ? q / 16 : q % 64;
            const int64_t gn = n0 + nb, gkb = k0 + kb;
            T vb = (T)0;
            if (gn < N && gkb < kend) vb = TB ? B[gn * ldb + gkb] : B[gkb * ldb + gn];
            Bs[kb][nb] = vb;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < 16; ++kk) {
            T a[4], b[4];
            if constexpr (sizeof(T) == 4) {
                const float4 av = *reinterpret_cast<const float4 *>(&As[kk][ty * 4]);
                const float4 bv = *reinterpret_cast<const float4 *>(&Bs[kk][tx * 4]);
                a[0] = av.x; a[1] = av.y; a[2] = av.z; a[3] = av.w;
                b[0] = bv.x; b[1] = bv.y; b[2] = bv.z; b[3] = bv.w;
            } else {
#pragma unroll
                for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
                for (int r = 0; r < 4; ++r) b[r] = Bs[kk][tx * 4 + r];
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[r][c] += a[r] * b[c];
        }
        __syncthreads();
    }
#pragma unroll
    for (int r = 0; r < 4; ++r) {
        int64_t gm = m0 + ty * 4 + r;
        if (gm >= M) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            int64_t gn = n0 + tx * 4 + c;
            if (gn >= N) continue;
            T v = acc[r][c];
            T *dst = C + gm * ldc + gn;
            if (partials) {  // ordered split-K: this K chunk's partial, summed later in z order
                partials[((int64_t)blockIdx.z * M + gm) * N + gn] = v;
            } else if (gridDim.z > 1) {
                atomicAdd(dst, v);
            } else {
                if (accumulate) v += *dst;
                if (relu) v = (v > (T)0 || v != v) ? v : (T)0;  // np.maximum(v, 0): NaN propagates
                *dst = v;
            }
        }
    }
}

// C += sum_z part[z] in a fixed order (deterministic): block (32 x 8) -- 32 consecutive outputs
// (coalesced rows of the partials) x 8 interleaved z-subsequences, folded in z-subsequence order
template <typename T>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(const T *__restrict__ part, int nz, int64_t M, int64_t N,
                                                            T *__restrict__ C, int64_t ldc) {
    __shared__ T sums[8][32];
    const int64_t i = (int64_t)blockIdx.x * 32 + threadIdx.x;
    const int64_t mn = M * N;
    T acc = (T)0;
    if (i < mn)
        for (int z = threadIdx.y; z < nz; z += 8) acc += part[(int64_t)z * mn + i];
    sums[threadIdx.y][threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.y == 0 && i < mn) {
        T t = sums[0][threadIdx.x];
#pragma unroll
        for (int y = 1; y < 8; ++y) t += sums[y][threadIdx.x];
        const int64_t r = i / N, c = i - r * N;
        C[r * ldc + c] += t;
    }
}

template <typename T, bool TA, bool TB>
static int gemm(int64_t M, int64_t N, int64_t K, const T *A, int64_t lda, const T *B, int64_t ldb, T *C,
                int64_t ldc, int accumulate, int relu, cudaStream_t s) {
    dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64), 1);
    int64_t tiles = (int64_t)grid.x * grid.y;
    if (accumulate && !relu && tiles < 296 && K > 4096) {
        // the weight-gradient reductions over the batch (M, N <= a few tiles, K = B): split K into
        // chunks of ~128 rows so the whole GPU works on them (B = 65,536: 512 CTAs), each chunk's
        // partial summed afterwards in chunk order -- one pass, no atomics, deterministic
        const int64_t split = min((int64_t)2048, max((int64_t)1, (K + 127) / 128));
        grid.z = (unsigned)split;
    }
    if (grid.z > 1) {
        // ordered split-K: partials [split][M][N], then C += sum_z in z order
        T *part = nullptr;
        if (cudaMallocAsync((void **)&part, sizeof(T) * grid.z * M * N, s) != cudaSuccess)
            return check_launch("gemm partials alloc");
        gemm_kernel<T, TA, TB><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, relu, part);
        splitk_reduce_kernel<T><<<(unsigned)((M * N + 31) / 32), dim3(32, 8), 0, s>>>(part, (int)grid.z, M, N, C, ldc);
        cudaFreeAsync(part, s);
        return check_launch("gemm (ordered split-K)");
    }
    gemm_kernel<T, TA, TB><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, accumulate, relu, (T *)nullptr);
    return check_launch("gemm");
}

template <typename T>
__global__ void relu_mask_kernel(T *__restrict__ d, const T *__restrict__ act, int64_t n) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = d[i] * (act[i] > (T)0 ? (T)1 : (T)0);
}

template <typename T>
static int mlp_forward_t(int64_t b, int nl, const int32_t *widths, const void *const *weights,
                         void *const *acts, int relu_out, cudaStream_t s) {
    for (int i = 0; i < nl; ++i) {
        int64_t win = widths[i], wout = widths[i + 1];
        bool relu = (i < nl - 1) || relu_out;
        int st = gemm<T, false, true>(b, wout, win, (const T *)acts[i], win, (const T *)weights[i], win,
                                      (T *)acts[i + 1], wout, 0, relu ? 1 : 0, s);
        if (st) return st;
    }
    return NVOL_OK;
}

template <typename T>
static int mlp_backward_t(int64_t b, int nl, const int32_t *widths, const void *const *weights,
                          const void *const *acts, const void *dl_dout, void *const *grads, void *dl_din,
                          void *s0, void *s1, int relu_out, cudaStream_t s) {
    // d = dl_dout as a (B, 1) matrix, copied so the mask can be applied in place
    T *d = (T *)s0, *dn = (T *)s1;
    if (cudaMemcpyAsync(d, dl_dout, sizeof(T) * b * widths[nl], cudaMemcpyDeviceToDevice, s) != cudaSuccess)
        return check_launch("mlp_backward copy");
    for (int i = nl - 1; i >= 0; --i) {
        int64_t win = widths[i], wout = widths[i + 1];
        if (i < nl - 1 || relu_out) {
            relu_mask_kernel<T><<<grid_for(b * wout, 256), 256, 0, s>>>(d, (const T *)acts[i + 1], b * wout);
        }
        // grads[i] += d^T @ acts[i]   (wout x win, K = B)
        int st = gemm<T, true, false>(wout, win, b, d, wout, (const T *)acts[i], win, (T *)grads[i], win, 1, 0, s);
        if (st) return st;
        // d = d @ W_i   (B x win)
        T *dst = (i == 0) ? (T *)dl_din : dn;
        st = gemm<T, false, false>(b, win, wout, d, wout, (const T *)weights[i], win, dst, win, 0, 0, s);
        if (st) return st;
        T *tmp = d;
        d = dn;
        dn = tmp;
    }
    return check_launch("mlp_backward");
}

template <typename T>
__global__ void loss_kernel(const T *__restrict__ pred, const T *__restrict__ target, int64_t b, int kind,
                            double denom, T *__restrict__ grad, double *__restrict__ loss_sum,
                            double *__restrict__ block_sums) {
    __shared__ double red[32];
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    double s = 0.0;
    if (i < b) {
        double d = __dsub_rn((double)pred[i], (double)target[i]);
        double g;
        if (kind == 0) {
            s = fabs(d);
            double sg = d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : (d == d ? 0.0 : d));  // np.sign: NaN -> NaN
            g = __ddiv_rn(sg, denom);
        } else {
            s = __dmul_rn(d, d);
            g = __ddiv_rn(__dmul_rn(2.0, d), denom);
        }
        if (grad) grad[i] = (T)g;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) {
            if (block_sums)
                block_sums[blockIdx.x] = s;  // ordered mode: summed in block order by loss_fold_kernel
            else
                atomicAdd(loss_sum, s);
        }
    }
}

__global__ void loss_fold_kernel(const double *__restrict__ block_sums, int n, double *__restrict__ loss_sum) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        double acc = 0.0;
        for (int i = 0; i < n; ++i) acc += block_sums[i];
        *loss_sum += acc;
    }
}

template <typename T>
__global__ void adam_kernel(T *__restrict__ p, T *__restrict__ g, T *__restrict__ m, T *__restrict__ v,
                            int64_t n, T lr, T b1, T omb1, T b2, T omb2, T c1, T c2, T eps, T l2) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
         j += (int64_t)gridDim.x * blockDim.x) {
        T pj = p[j], gj = g[j], mj = m[j], vj = v[j];
        adam_one<T>(pj, gj, mj, vj, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        p[j] = pj;
        g[j] = gj;
        m[j] = mj;
        v[j] = vj;
    }
}

// Flat float32 Adam for the training pipeline: float4-vectorised streaming
// over (p, g, m, v) — 32 algorithmic bytes per parameter, the dominant HBM
// term of a cfg2 step.  Scalars come from the device-side schedule so a
// captured CUDA graph replays correctly step after step.
__global__ void __launch_bounds__(256) adam_flat_kernel(
    float *__restrict__ p, float *__restrict__ g, float *__restrict__ m, float *__restrict__ v, int64_t n,
    const float *__restrict__ sched, int64_t sched_len, const int64_t *__restrict__ step_counter, float b1,
    float omb1, float b2, float omb2, float eps, float l2, uint32_t *__restrict__ nan_flag) {
    int64_t t = *step_counter;
    if (t >= sched_len) t = sched_len - 1;
    const float lr = sched[3 * t], c1 = sched[3 * t + 1], c2 = sched[3 * t + 2];
    // the flat buffers may start 4/8/12 bytes past a 16-byte boundary (nvol.h flat layout):
    // scalar head, float4 body, scalar tail
    // scalar head up to the next 128-byte boundary: each warp's float4 accesses then cover whole lines
    const int64_t head = min(n, (int64_t)(((128 - (reinterpret_cast<uintptr_t>(p) & 127)) & 127) >> 2));
    const int64_t n4 = (n - head) >> 2;
    bool bad = false;
    float4 *p4 = reinterpret_cast<float4 *>(p + head), *g4 = reinterpret_cast<float4 *>(g + head);
    float4 *m4 = reinterpret_cast<float4 *>(m + head), *v4 = reinterpret_cast<float4 *>(v + head);
    const uint64_t keep = l2_evict_last();
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += (int64_t)gridDim.x * blockDim.x) {
        float4 P = __ldcs(p4 + j);
        float4 G = ld4_hint(g4 + j, keep), M = __ldcs(m4 + j), V = __ldcs(v4 + j);
        bad |= isnan(G.x) | isnan(G.y) | isnan(G.z) | isnan(G.w);
        adam_one<float>(P.x, G.x, M.x, V.x, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        adam_one<float>(P.y, G.y, M.y, V.y, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        adam_one<float>(P.z, G.z, M.z, V.z, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        adam_one<float>(P.w, G.w, M.w, V.w, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        __stcs(p4 + j, P);
        st4_hint(g4 + j, G, keep);  // the zeroed gradient stays in L2 for the next scatter
        __stcs(m4 + j, M);
        __stcs(v4 + j, V);
    }
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < head + (n - head - 4 * n4);
         j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t q = j < head ? j : head + 4 * n4 + (j - head);  // head then tail elements
        float P = p[q], G = g[q], M = m[q], V = v[q];
        bad |= isnan(G);
        adam_one<float>(P, G, M, V, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        p[q] = P;
        g[q] = G;
        m[q] = M;
        v[q] = V;
    }
    if (nan_flag && __any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(nan_flag, 1u);
}

// Float32 Adam with host scalars (nvol_adam_step on float buffers that share
// their 16-byte alignment, e.g. the flat model buffers): adam_flat_kernel's
// float4 streaming without the device schedule table.
__global__ void __launch_bounds__(256) adam_vec_kernel(float *__restrict__ p, float *__restrict__ g,
                                                       float *__restrict__ m, float *__restrict__ v, int64_t n,
                                                       float lr, float b1, float omb1, float b2, float omb2,
                                                       float c1, float c2, float eps, float l2) {
    const int64_t head = min(n, (int64_t)(((128 - (reinterpret_cast<uintptr_t>(p) & 127)) & 127) >> 2));
    const int64_t n4 = (n - head) >> 2;
    float4 *p4 = reinterpret_cast<float4 *>(p + head), *g4 = reinterpret_cast<float4 *>(g + head);
    float4 *m4 = reinterpret_cast<float4 *>(m + head), *v4 = reinterpret_cast<float4 *>(v + head);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += stride) {
        float4 P = __ldcs(p4 + j), G = __ldcs(g4 + j), M = __ldcs(m4 + j), V = __ldcs(v4 + j);
        adam_one<float>(P.x, G.x, M.x, V.x, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        adam_one<float>(P.y, G.y, M.y, V.y, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        adam_one<float>(P.z, G.z, M.z, V.z, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        adam_one<float>(P.w, G.w, M.w, V.w, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        __stcs(p4 + j, P);
        __stcs(g4 + j, G);
        __stcs(m4 + j, M);
        __stcs(v4 + j, V);
    }
    for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < head + (n - head - 4 * n4); jj += stride) {
        const int64_t q = jj < head ? jj : head + 4 * n4 + (jj - head);  // head then tail elements
        float P = p[q], G = g[q], M = m[q], V = v[q];
        adam_one<float>(P, G, M, V, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        p[q] = P;
        g[q] = G;
        m[q] = M;
        v[q] = V;
    }
}

// Training-pipeline Adam step: adam_flat_kernel's update plus the step's bookkeeping in the last block to
// finish (ticket): losses[t - t0] = loss_sum / B, loss_sum = 0, t += 1.  Every
// block reads t before taking its ticket, so the advance cannot race a reader.
// NaN contract (common.cuh, nan_state): only q < nan_state[0] is updated (the
// parameter groups in front of the first one holding a NaN gradient,
// network.py:167-171); a NaN this kernel meets itself is left in place and
// lowers the limit.  When the limit is set the last block halts the pipeline
// instead of recording the loss / advancing t; a halted pipeline's Adam is a no-op.
__global__ void __launch_bounds__(256) adam_step_kernel(
    float *__restrict__ p, float *__restrict__ g, float *__restrict__ m, float *__restrict__ v, int64_t n,
    const float *__restrict__ sched, int64_t sched_len, int64_t *__restrict__ step_counter, float b1, float omb1,
    float b2, float omb2, float eps, float l2, int64_t *__restrict__ nan_state, double *__restrict__ loss_acc,
    double *__restrict__ losses, int64_t t0, int64_t cap, double inv_b, uint32_t *__restrict__ ticket) {
    if (nan_halted(nan_state)) return;
    const int64_t tc = *step_counter;
    const int64_t t = tc >= sched_len ? sched_len - 1 : tc;
    const float lr = sched[3 * t], c1 = sched[3 * t + 1], c2 = sched[3 * t + 2];
    const int64_t lim = nan_limit(nan_state);
    // scalar head up to the next 128-byte boundary: each warp's float4 accesses then cover whole lines
    const int64_t head = min(n, (int64_t)(((128 - (reinterpret_cast<uintptr_t>(p) & 127)) & 127) >> 2));
    const int64_t n4 = (n - head) >> 2;
    int64_t bad = kNanNone;
    float4 *p4 = reinterpret_cast<float4 *>(p + head), *g4 = reinterpret_cast<float4 *>(g + head);
    float4 *m4 = reinterpret_cast<float4 *>(m + head), *v4 = reinterpret_cast<float4 *>(v + head);
    const uint64_t keep = l2_evict_last();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // one element under the limit; a NaN gradient the detectors upstream did not see stays unapplied
    auto one = [&](float &P, float &G, float &M, float &V, int64_t q) {
        if (q >= lim) return;
        if (isnan(G)) {
            bad = min(bad, q);
            return;
        }
        adam_one<float>(P, G, M, V, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
    };
    int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; j < n4; j += stride) {
        float4 P = __ldcs(p4 + j), G = ld4_hint(g4 + j, keep), M = __ldcs(m4 + j), V = __ldcs(v4 + j);
        const int64_t q = head + 4 * j;
        if (q + 3 < lim && !(isnan(G.x) | isnan(G.y) | isnan(G.z) | isnan(G.w))) {
            adam_one<float>(P.x, G.x, M.x, V.x, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
            adam_one<float>(P.y, G.y, M.y, V.y, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
            adam_one<float>(P.z, G.z, M.z, V.z, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
            adam_one<float>(P.w, G.w, M.w, V.w, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
        } else {
            one(P.x, G.x, M.x, V.x, q);
            one(P.y, G.y, M.y, V.y, q + 1);
            one(P.z, G.z, M.z, V.z, q + 2);
            one(P.w, G.w, M.w, V.w, q + 3);
        }
        __stcs(p4 + j, P);
        st4_hint(g4 + j, G, keep);
        __stcs(m4 + j, M);
        __stcs(v4 + j, V);
    }
    for (int64_t jj = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; jj < head + (n - head - 4 * n4); jj += stride) {
        const int64_t q = jj < head ? jj : head + 4 * n4 + (jj - head);  // head then tail elements
        float P = p[q], G = g[q], M = m[q], V = v[q];
        one(P, G, M, V, q);
        p[q] = P;
        g[q] = G;
        m[q] = M;
        v[q] = V;
    }
    if (bad != kNanNone) nan_mark(nan_state, bad);
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
            __threadfence();
            *ticket = 0u;
            if (nan_limit(nan_state) != kNanNone) {
                nan_state[1] = 1;  // halt: the step is not recorded, t does not advance
                return;
            }
            const int64_t k = tc - t0;
            if (losses && k >= 0 && k < cap) losses[k] = *reinterpret_cast<volatile double *>(loss_acc) * inv_b;
            if (loss_acc) *loss_acc = 0.0;
            *step_counter = tc + 1;
        }
    }
}

// SIMT training engine's NaN detector (the tcgen05 engine detects in its MLP
// kernel): marks the start of every parameter group whose gradient holds a NaN.
struct GroupStarts {
    int64_t start[16];
    int n;
};
__global__ void nan_scan_kernel(const float *__restrict__ g, int64_t n, const GroupStarts gs,
                                int64_t *__restrict__ nan_state) {
    if (nan_halted(nan_state)) return;
    int64_t first = kNanNone;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        if (isnan(g[j])) {
            first = min(first, j);
            break;
        }
    if (first != kNanNone) {
        int64_t st = 0;
        for (int i = 0; i < gs.n; ++i)
            if (gs.start[i] <= first) st = gs.start[i];
        nan_mark(nan_state, st);
    }
}

// adam_step_kernel's update streamed by the bulk-copy (TMA) engine: each CTA walks chunks of
// AD_CH floats of the four flat arrays through an AD_ST-deep ring of shared-memory stages --
// one thread issues 4 bulk loads per chunk (p, m, v evict-first; g evict-last, it stays in L2
// for the next scatter), the CTA updates the stage in place and one thread bulk-stores it back
// (p, m, v, and g = 0).  The DMA engine keeps ~100 KB in flight per CTA without occupying
// registers, which is what the HBM-bound update needs.  Same arithmetic, same NaN contract and
// same step bookkeeping (ticket) as adam_step_kernel.
#ifndef NVOL_AD_CH
#define NVOL_AD_CH 2048
#endif
#ifndef NVOL_AD_ST
#define NVOL_AD_ST 3
#endif
constexpr int AD_CH = NVOL_AD_CH;  // floats per array per chunk (8 KB)
constexpr int AD_ST = NVOL_AD_ST;  // ring depth
constexpr int AD_THREADS = 256; // 2 float4 per thread per array per chunk

__device__ __forceinline__ void bulk_g2s_hint(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            (uint32_t)__cvta_generic_to_shared(dst)),
        "l"(src), "r"(bytes), "r"((uint32_t)__cvta_generic_to_shared(bar)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void bulk_s2g_hint(void *dst, const void *src, uint32_t bytes, uint64_t pol) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"(dst),
                 "r"((uint32_t)__cvta_generic_to_shared(src)), "r"(bytes), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__global__ void __launch_bounds__(AD_THREADS) adam_tma_kernel(
    float *__restrict__ p, float *__restrict__ g, float *__restrict__ m, float *__restrict__ v, int64_t n,
    const float *__restrict__ sched, int64_t sched_len, int64_t *__restrict__ step_counter, float b1, float omb1,
    float b2, float omb2, float eps, float l2, int64_t *__restrict__ nan_state, double *__restrict__ loss_acc,
    double *__restrict__ losses, int64_t t0, int64_t cap, double inv_b, uint32_t *__restrict__ ticket) {
    extern __shared__ __align__(128) float ring[];  // [AD_ST][4][AD_CH]: p, g, m, v
    __shared__ uint64_t full[AD_ST];
    if (nan_halted(nan_state)) return;
    const int tid = threadIdx.x;
    const int64_t tc = *step_counter;
    const int64_t t = tc >= sched_len ? sched_len - 1 : tc;
    const float lr = sched[3 * t], c1 = sched[3 * t + 1], c2 = sched[3 * t + 2];
    const int64_t lim = nan_limit(nan_state);
    const int64_t head = min(n, (int64_t)(((128 - (reinterpret_cast<uintptr_t>(p) & 127)) & 127) >> 2));
    const int64_t nbody = ((n - head) >> 2) << 2;  // float4-aligned body, whole 16-byte units
    const int64_t nch = (nbody + AD_CH - 1) / AD_CH;
    int64_t bad = kNanNone;
    auto one = [&](float &P, float &G, float &M, float &V, int64_t q) {
        if (q >= lim) return;
        if (isnan(G)) {
            bad = min(bad, q);
            return;
        }
        adam_one<float>(P, G, M, V, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
    };
    const uint64_t first = l2_evict_first(), keep = l2_evict_last();
    float *arr[4] = {p + head, g + head, m + head, v + head};
    if (tid == 0) {
        for (int s = 0; s < AD_ST; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
#if defined(NVOL_ADAM_LAYOUT_EXPT)
    // timing experiment only (tools/adam_layout.py): m / v (1) or p / m / v (2) interleaved in
    // AD_CH-float blocks, so the chunk's optimizer state is one contiguous DRAM region
    auto at = [&](int a, int64_t off) -> float * {
        const int64_t blk = off / AD_CH;
        if (NVOL_ADAM_LAYOUT_EXPT == 1 && a >= 2) return m + blk * 2 * AD_CH + (a == 3 ? AD_CH : 0);
        if (NVOL_ADAM_LAYOUT_EXPT == 2 && a != 1) return p + blk * 3 * AD_CH + (a == 0 ? 0 : (a == 2 ? AD_CH : 2 * AD_CH));
        return arr[a] + off;
    };
#else
    auto at = [&](int a, int64_t off) -> float * { return arr[a] + off; };
#endif
    auto issue = [&](int s, int64_t c) {  // thread 0: chunk c -> stage s
        const int64_t off = c * AD_CH;
        const uint32_t bytes = (uint32_t)(min((int64_t)AD_CH, nbody - off) * 4);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&full[s])),
                     "r"(4 * bytes)
                     : "memory");
        for (int a = 0; a < 4; ++a)
            bulk_g2s_hint(ring + ((int64_t)s * 4 + a) * AD_CH, at(a, off), bytes, &full[s], a == 1 ? keep : first);
    };
    int64_t c = blockIdx.x;
    if (tid == 0)
        for (int s = 0; s < AD_ST; ++s)
            if (c + (int64_t)s * gridDim.x < nch) issue(s, c + (int64_t)s * gridDim.x);
    uint32_t par = 0;
    for (int k = 0; c < nch; ++k, c += gridDim.x) {
        const int s = k % AD_ST;
        {
            const uint32_t addr = (uint32_t)__cvta_generic_to_shared(&full[s]);
            const uint32_t ph = (par >> s) & 1u;
            asm volatile(
                "{\n\t.reg .pred P1;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t@!P1 bra W_%=;\n\t}\n" ::"r"(addr),
                "r"(ph)
                : "memory");
            par ^= 1u << s;
        }
        const int64_t off = c * AD_CH;
        const int cnt = (int)min((int64_t)AD_CH, nbody - off);
        float4 *sp = reinterpret_cast<float4 *>(ring + ((int64_t)s * 4 + 0) * AD_CH);
        float4 *sg = reinterpret_cast<float4 *>(ring + ((int64_t)s * 4 + 1) * AD_CH);
        float4 *sm = reinterpret_cast<float4 *>(ring + ((int64_t)s * 4 + 2) * AD_CH);
        float4 *sv = reinterpret_cast<float4 *>(ring + ((int64_t)s * 4 + 3) * AD_CH);
        for (int j = tid; j < cnt / 4; j += AD_THREADS) {
            float4 P = sp[j], G = sg[j], M = sm[j], V = sv[j];
            const int64_t q = head + off + 4 * j;
            if (q + 3 < lim && !(isnan(G.x) | isnan(G.y) | isnan(G.z) | isnan(G.w))) {
                adam_one<float>(P.x, G.x, M.x, V.x, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
                adam_one<float>(P.y, G.y, M.y, V.y, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
                adam_one<float>(P.z, G.z, M.z, V.z, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
                adam_one<float>(P.w, G.w, M.w, V.w, lr, b1, omb1, b2, omb2, c1, c2, eps, l2);
            } else {
                one(P.x, G.x, M.x, V.x, q);
                one(P.y, G.y, M.y, V.y, q + 1);
                one(P.z, G.z, M.z, V.z, q + 2);
                one(P.w, G.w, M.w, V.w, q + 3);
            }
            sp[j] = P;
            sg[j] = G;
            sm[j] = M;
            sv[j] = V;
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> bulk stores
        __syncthreads();
        if (tid == 0) {
            const uint32_t bytes = (uint32_t)cnt * 4u;
            for (int a = 0; a < 4; ++a) bulk_s2g_hint(at(a, off), ring + ((int64_t)s * 4 + a) * AD_CH, bytes, a == 1 ? keep : first);
            bulk_commit();
            const int64_t nc = c + (int64_t)AD_ST * gridDim.x;
            if (nc < nch) {
                bulk_wait_read0();  // stage s has been read out by its stores
                issue(s, nc);
            }
        }
    }
    if (tid == 0) bulk_wait0();  // the stores are complete before the ticket publishes the step
    // scalar head / tail (block 0)
    if (blockIdx.x == 0) {
        const int64_t tail0 = head + nbody;
        for (int64_t jj = tid; jj < head + (n - tail0); jj += AD_THREADS) {
            const int64_t q = jj < head ? jj : tail0 + (jj - head);
            float P = p[q], G = g[q], M = m[q], V = v[q];
            one(P, G, M, V, q);
            p[q] = P;
            g[q] = G;
            m[q] = M;
            v[q] = V;
        }
    }
    if (bad != kNanNone) nan_mark(nan_state, bad);
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
            __threadfence();
            *ticket = 0u;
            if (nan_limit(nan_state) != kNanNone) {
                nan_state[1] = 1;  // halt: the step is not recorded, t does not advance
                return;
            }
            const int64_t kk = tc - t0;
            if (losses && kk >= 0 && kk < cap) losses[kk] = *reinterpret_cast<volatile double *>(loss_acc) * inv_b;
            if (loss_acc) *loss_acc = 0.0;
            *step_counter = tc + 1;
        }
    }
}

__global__ void step_advance_kernel(int64_t *counter) { *counter += 1; }

__global__ void loss_record_kernel(double *acc, double *losses, const int64_t *counter, int64_t t0, int64_t cap,
                                   double inv_b) {
    int64_t k = *counter - t0;
    if (k >= 0 && k < cap) losses[k] = *acc * inv_b;
    *acc = 0.0;
}

template <typename T>
__global__ void find_nan_kernel(const T *__restrict__ g, int64_t n, unsigned long long *first) {
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (int64_t)gridDim.x * blockDim.x)
        if (isnan(g[j])) atomicMin(first, (unsigned long long)j);
}

__global__ void fill_u64_kernel(unsigned long long *p, unsigned long long v) { *p = v; }
__global__ void finish_nan_kernel(unsigned long long *p) {
    if (*p == ~0ull) *reinterpret_cast<long long *>(p) = -1;
}

static unsigned stream_grid(int64_t n) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t want = (n + 255) / 256;
    int64_t cap = (int64_t)sms * 8;
    return (unsigned)max((int64_t)1, min(want, cap));
}

}  // namespace nvol

using namespace nvol;

extern "C" {

int nvol_mlp_forward(int64_t b, int32_t n_layers, const int32_t *widths, const void *const *weights,
                     void *const *acts, int32_t relu_out, int32_t dtype_bytes, void *stream) {
    NVOL_REQUIRE(n_layers >= 1 && widths && weights && acts, "bad MLP description");
    NVOL_REQUIRE(dtype_bytes == 4 || dtype_bytes == 8, "dtype must be float32 or float64");
    if (b == 0) return NVOL_OK;
    if (dtype_bytes == 4) return mlp_forward_t<float>(b, n_layers, widths, weights, acts, relu_out, as_stream(stream));
    return mlp_forward_t<double>(b, n_layers, widths, weights, acts, relu_out, as_stream(stream));
}

int nvol_mlp_backward(int64_t b, int32_t n_layers, const int32_t *widths, const void *const *weights,
                      const void *const *acts, const void *dl_dout, void *const *grads, void *dl_dinput,
                      void *scratch0, void *scratch1, int32_t relu_out, int32_t dtype_bytes, void *stream) {
    NVOL_REQUIRE(n_layers >= 1 && widths && weights && acts && grads, "bad MLP description");
    NVOL_REQUIRE(dl_dout && dl_dinput && scratch0 && scratch1, "null pointer");
    NVOL_REQUIRE(dtype_bytes == 4 || dtype_bytes == 8, "dtype must be float32 or float64");
    if (b == 0) return NVOL_OK;
    if (dtype_bytes == 4)
        return mlp_backward_t<float>(b, n_layers, widths, weights, acts, dl_dout, grads, dl_dinput, scratch0,
                                     scratch1, relu_out, as_stream(stream));
    return mlp_backward_t<double>(b, n_layers, widths, weights, acts, dl_dout, grads, dl_dinput, scratch0,
                                  scratch1, relu_out, as_stream(stream));
}

int nvol_loss_and_grad_scaled(const void *pred, const void *target, int64_t b, int64_t b_global, int32_t kind,
                              void *grad, double *loss_sum, int32_t dtype_bytes, void *stream) {
    NVOL_REQUIRE(kind == 0 || kind == 1, "loss kind must be 0 (L1) or 1 (L2)");
    NVOL_REQUIRE(b >= 1, "empty batch");
    NVOL_REQUIRE(pred && target && loss_sum, "null pointer");
    cudaStream_t s = as_stream(stream);
    const unsigned nb = grid_for(b, 256);
    double *bs = nullptr;
    if (g_deterministic && cudaMallocAsync((void **)&bs, sizeof(double) * nb, s) != cudaSuccess)
        return check_launch("loss partials alloc");
    if (dtype_bytes == 4)
        loss_kernel<float><<<nb, 256, 0, s>>>((const float *)pred, (const float *)target, b, kind, (double)b_global,
                                              (float *)grad, loss_sum, bs);
    else
        loss_kernel<double><<<nb, 256, 0, s>>>((const double *)pred, (const double *)target, b, kind,
                                               (double)b_global, (double *)grad, loss_sum, bs);
    if (bs) {
        loss_fold_kernel<<<1, 32, 0, s>>>(bs, (int)nb, loss_sum);
        cudaFreeAsync(bs, s);
    }
    return check_launch("loss_and_grad");
}

int nvol_loss_and_grad(const void *pred, const void *target, int64_t b, int32_t kind, void *grad,
                       double *loss_sum, int32_t dtype_bytes, void *stream) {
    return nvol_loss_and_grad_scaled(pred, target, b, b, kind, grad, loss_sum, dtype_bytes, stream);
}

int nvol_adam_train_step(float *p, float *g, float *m, float *v, int64_t n, const float *sched, int64_t sched_len,
                         int64_t *step_counter, float beta1, float one_minus_beta1, float beta2,
                         float one_minus_beta2, float eps, float l2, int64_t *nan_state, double *loss_acc,
                         double *losses, int64_t t0, int64_t cap, double inv_b, uint32_t *ticket, void *stream) {
    NVOL_REQUIRE(p && g && m && v && sched && step_counter && ticket && sched_len >= 1, "null pointer");
    NVOL_REQUIRE(((uintptr_t)p & 127) == ((uintptr_t)g & 127) && ((uintptr_t)p & 127) == ((uintptr_t)m & 127) &&
                     ((uintptr_t)p & 127) == ((uintptr_t)v & 127) && ((uintptr_t)p & 3) == 0,
                 "flat Adam buffers must share their alignment modulo 128 bytes");
    static int tma = -1;  // NVOL_ADAM_TMA=0: the register-streaming adam_step_kernel (A/B measurements)
    if (tma < 0) {
        const char *e = getenv("NVOL_ADAM_TMA");
        tma = (e && e[0] == '0') ? 0 : 1;
    }
    cudaStream_t s = as_stream(stream);
    if (tma) {
        const size_t smem = (size_t)AD_ST * 4 * AD_CH * 4;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(adam_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            attr = true;
        }
        int dev = 0, sms = 148, per = 1;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, adam_tma_kernel, AD_THREADS, smem);
        const int64_t nch = (n / AD_CH) + 1;
        const int64_t grid = std::max((int64_t)1, std::min((int64_t)sms * std::max(per, 1), nch));
        adam_tma_kernel<<<(unsigned)grid, AD_THREADS, smem, s>>>(p, g, m, v, n, sched, sched_len, step_counter, beta1,
                                                                 one_minus_beta1, beta2, one_minus_beta2, eps, l2,
                                                                 nan_state, loss_acc, losses, t0, cap, inv_b, ticket);
        return check_launch("adam_train_step");
    }
    adam_step_kernel<<<stream_grid((n + 3) / 4), 256, 0, s>>>(
        p, g, m, v, n, sched, sched_len, step_counter, beta1, one_minus_beta1, beta2, one_minus_beta2, eps, l2,
        nan_state, loss_acc, losses, t0, cap, inv_b, ticket);
    return check_launch("adam_train_step");
}

int nvol_nan_scan(const float *g, int64_t n, const int64_t *group_starts, int32_t n_groups, int64_t *nan_state,
                  void *stream) {
    NVOL_REQUIRE(g && group_starts && nan_state && n_groups >= 1 && n_groups <= 16, "bad arguments");
    GroupStarts gs;
    gs.n = n_groups;
    for (int i = 0; i < n_groups; ++i) gs.start[i] = group_starts[i];
    nan_scan_kernel<<<stream_grid(n), 256, 0, as_stream(stream)>>>(g, n, gs, nan_state);
    return check_launch("nan_scan");
}

int nvol_loss_record(double *acc, double *losses, const int64_t *step_counter, int64_t t0, int64_t cap,
                     double inv_b, void *stream) {
    NVOL_REQUIRE(acc && losses && step_counter && cap >= 1, "null pointer");
    loss_record_kernel<<<1, 1, 0, as_stream(stream)>>>(acc, losses, step_counter, t0, cap, inv_b);
    return check_launch("loss_record");
}

int nvol_adam_step(void *p, void *g, void *m, void *v, int64_t n, double lr, double beta1,
                   double one_minus_beta1, double beta2, double one_minus_beta2, double c1, double c2,
                   double eps, double l2, int32_t dtype_bytes, void *stream) {
    NVOL_REQUIRE(dtype_bytes == 4 || dtype_bytes == 8, "dtype must be float32 or float64");
    if (n == 0) return NVOL_OK;
    NVOL_REQUIRE(p && g && m && v, "null pointer");
    cudaStream_t s = as_stream(stream);
    const uintptr_t al = (uintptr_t)p & 15;
    if (dtype_bytes == 4 && n >= 1024 && al == ((uintptr_t)g & 15) && al == ((uintptr_t)m & 15) &&
        al == ((uintptr_t)v & 15) && (al & 3) == 0)
        adam_vec_kernel<<<stream_grid((n + 3) / 4), 256, 0, s>>>((float *)p, (float *)g, (float *)m, (float *)v, n,
                                                                  (float)lr, (float)beta1, (float)one_minus_beta1,
                                                                  (float)beta2, (float)one_minus_beta2, (float)c1,
                                                                  (float)c2, (float)eps, (float)l2);
    else if (dtype_bytes == 4)
        adam_kernel<float><<<stream_grid(n), 256, 0, s>>>((float *)p, (float *)g, (float *)m, (float *)v, n,
                                                          (float)lr, (float)beta1, (float)one_minus_beta1,
                                                          (float)beta2, (float)one_minus_beta2, (float)c1,
                                                          (float)c2, (float)eps, (float)l2);
    else
        adam_kernel<double><<<stream_grid(n), 256, 0, s>>>((double *)p, (double *)g, (double *)m, (double *)v, n,
                                                           lr, beta1, one_minus_beta1, beta2, one_minus_beta2,
                                                           c1, c2, eps, l2);
    return check_launch("adam_step");
}

int nvol_adam_flat_dev(float *p, float *g, float *m, float *v, int64_t n, const float *sched, int64_t sched_len,
                       int64_t *step_counter, float beta1, float one_minus_beta1, float beta2,
                       float one_minus_beta2, float eps, float l2, uint32_t *nan_flag, void *stream) {
    NVOL_REQUIRE(p && g && m && v && sched && step_counter && sched_len >= 1, "null pointer");
    NVOL_REQUIRE(((uintptr_t)p & 127) == ((uintptr_t)g & 127) && ((uintptr_t)p & 127) == ((uintptr_t)m & 127) &&
                     ((uintptr_t)p & 127) == ((uintptr_t)v & 127) && ((uintptr_t)p & 3) == 0,
                 "flat Adam buffers must share their alignment modulo 128 bytes");
    cudaStream_t s = as_stream(stream);
    adam_flat_kernel<<<stream_grid((n + 3) / 4), 256, 0, s>>>(p, g, m, v, n, sched, sched_len, step_counter, beta1,
                                                              one_minus_beta1, beta2, one_minus_beta2, eps, l2,
                                                              nan_flag);
    step_advance_kernel<<<1, 1, 0, s>>>(step_counter);
    return check_launch("adam_flat");
}

int nvol_find_nan(const void *g, int64_t n, int64_t *first, int32_t dtype_bytes, void *stream) {
    NVOL_REQUIRE(first, "null pointer");
    cudaStream_t s = as_stream(stream);
    unsigned long long *f = reinterpret_cast<unsigned long long *>(first);
    fill_u64_kernel<<<1, 1, 0, s>>>(f, ~0ull);
    if (n > 0) {
        if (dtype_bytes == 4)
            find_nan_kernel<float><<<stream_grid(n), 256, 0, s>>>((const float *)g, n, f);
        else
            find_nan_kernel<double><<<stream_grid(n), 256, 0, s>>>((const double *)g, n, f);
    }
    finish_nan_kernel<<<1, 1, 0, s>>>(f);
    return check_launch("find_nan");
}

}  // extern "C"
