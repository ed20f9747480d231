// Exact per-sample field evaluation building blocks shared by the fused
// evaluator / decode (field.cu) and the in-shader ray marcher (render.cu).
// Reference: _kernels.py:95-151 (_mlp_row, _field_one): float32, dot
// products folded in k order without FMA contraction (bit-identical).
#pragma once
#include "common.cuh"

namespace nvol {

struct MlpShape {
    int32_t n_layers;
    int32_t widths[12];
    int32_t relu_out;
};

constexpr int FE_THREADS = 128;

// Encode one sample into feat[k * FE_THREADS] (column of this thread).
__device__ __forceinline__ void encode_exact(float x, float y, float z, const float *__restrict__ params,
                                             const GridTables &tab, float *feat) {
    const int m = tab.n_levels, n = tab.n_feat;
    for (int l = 0; l < m; ++l) {
        const int32_t res = tab.res[l];
        Cell<float> c = cell_of<float>(x, y, z, res);
        float acc[8];
#pragma unroll
        for (int f = 0; f < 8; ++f) acc[f] = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int64_t slot = vertex_slot(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), res,
                                       tab.entries[l], tab.dense[l] != 0);
            float w = corner_weight<float>(c, k);
            // w == 0 adds +-0 to a sum that starts at +0: skipping the gather is
            // bit-exact for finite tables (voxel-centre decodes: every level finer
            // than the output grid has fx = fy = fz = 0, i.e. one live corner)
            if (w == 0.0f) continue;
            const float *p = params + tab.offset[l] + slot * n;
            for (int f = 0; f < n; ++f) acc[f] = xadd(acc[f], xmul(w, __ldg(p + f)));
        }
        for (int f = 0; f < n; ++f) feat[(l * n + f) * FE_THREADS] = acc[f];
    }
}

// Hidden width NN known at compile time: activations live in registers.
template <int NN>
__device__ __forceinline__ float mlp_exact_reg(const float *feat, int nin, const float *__restrict__ wt,
                                               const MlpShape &sh) {
    float h[NN];
    // layer 0: nin -> NN, wt holds W0^T (nin x NN)
    {
        float acc[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) acc[j] = 0.0f;
        for (int k = 0; k < nin; ++k) {
            float hk = feat[k * FE_THREADS];
            const float4 *wr = reinterpret_cast<const float4 *>(wt + k * NN);
#pragma unroll
            for (int j4 = 0; j4 < NN / 4; ++j4) {
                float4 w = wr[j4];
                acc[4 * j4 + 0] = xadd(acc[4 * j4 + 0], xmul(w.x, hk));
                acc[4 * j4 + 1] = xadd(acc[4 * j4 + 1], xmul(w.y, hk));
                acc[4 * j4 + 2] = xadd(acc[4 * j4 + 2], xmul(w.z, hk));
                acc[4 * j4 + 3] = xadd(acc[4 * j4 + 3], xmul(w.w, hk));
            }
        }
        const bool relu = sh.n_layers > 1 || sh.relu_out;
#pragma unroll
        for (int j = 0; j < NN; ++j) h[j] = relu ? fmaxf(acc[j], 0.0f) : acc[j];
        wt += nin * NN;
    }
    const int nl = sh.n_layers;
    for (int li = 1; li < nl - 1; ++li) {
        float acc[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) acc[j] = 0.0f;
#pragma unroll
        for (int k = 0; k < NN; ++k) {
            const float4 *wr = reinterpret_cast<const float4 *>(wt + k * NN);
#pragma unroll
            for (int j4 = 0; j4 < NN / 4; ++j4) {
                float4 w = wr[j4];
                acc[4 * j4 + 0] = xadd(acc[4 * j4 + 0], xmul(w.x, h[k]));
                acc[4 * j4 + 1] = xadd(acc[4 * j4 + 1], xmul(w.y, h[k]));
                acc[4 * j4 + 2] = xadd(acc[4 * j4 + 2], xmul(w.z, h[k]));
                acc[4 * j4 + 3] = xadd(acc[4 * j4 + 3], xmul(w.w, h[k]));
            }
        }
#pragma unroll
        for (int j = 0; j < NN; ++j) h[j] = fmaxf(acc[j], 0.0f);
        wt += NN * NN;
    }
    if (nl == 1) return h[0];
    // output layer NN -> 1
    float o = 0.0f;
#pragma unroll
    for (int k = 0; k < NN; ++k) o = xadd(o, xmul(wt[k], h[k]));
    return sh.relu_out ? fmaxf(o, 0.0f) : o;
}

// Uniform hidden width NN: the activations of each thread live in its own
// shared-memory column (h[k] at col[k * FE_THREADS]) and the k-major weights are
// read as broadcast float4s (through L1 from global memory, GLOBAL_W, or from
// shared memory), one per 4 outputs, so the k loop stays
// rolled: a fully unrolled 64 x 64 layer is ~150 KB of SASS and the warps
// starved on instruction fetch.  The column must hold max(nin, NN) rows.  Same folds in the same order (acc[j] over k,
// xmul then xadd) as mlp_exact_reg: bit-identical.
template <int NN, bool GLOBAL_W>
__device__ __forceinline__ float mlp_exact_col(float *col, int nin, const float *__restrict__ wt, const MlpShape &sh) {
    auto ldw4 = [](const float4 *a) { return GLOBAL_W ? __ldg(a) : *a; };
    auto ldw = [](const float *a) { return GLOBAL_W ? __ldg(a) : *a; };
    const int nl = sh.n_layers;
    for (int li = 0; li < nl - 1; ++li) {
        const int win = li == 0 ? nin : NN;
        float acc[NN];
#pragma unroll
        for (int j = 0; j < NN; ++j) acc[j] = 0.0f;
#pragma unroll 2
        for (int k = 0; k < win; ++k) {
            const float hk = col[k * FE_THREADS];
            const float4 *wr = reinterpret_cast<const float4 *>(wt + k * NN);
#pragma unroll
            for (int j4 = 0; j4 < NN / 4; ++j4) {
                const float4 w = ldw4(wr + j4);
                acc[4 * j4 + 0] = xadd(acc[4 * j4 + 0], xmul(w.x, hk));
                acc[4 * j4 + 1] = xadd(acc[4 * j4 + 1], xmul(w.y, hk));
                acc[4 * j4 + 2] = xadd(acc[4 * j4 + 2], xmul(w.z, hk));
                acc[4 * j4 + 3] = xadd(acc[4 * j4 + 3], xmul(w.w, hk));
            }
        }
        // every hidden layer is followed by ReLU (the output layer is separate below)
#pragma unroll
        for (int j = 0; j < NN; ++j) col[j * FE_THREADS] = fmaxf(acc[j], 0.0f);
        wt += win * NN;
    }
    // output layer NN -> 1, one serial fold
    float o = 0.0f;
    for (int k = 0; k < NN; ++k) o = xadd(o, xmul(ldw(wt + k), col[k * FE_THREADS]));
    return sh.relu_out ? fmaxf(o, 0.0f) : o;
}

// Generic widths: activations ping-pong through this thread's smem columns.
__device__ __forceinline__ float mlp_exact_smem(float *h0, float *h1, const float *__restrict__ wt, const MlpShape &sh) {
    float *cur = h0, *nxt = h1;
    for (int li = 0; li < sh.n_layers; ++li) {
        int win = sh.widths[li], wout = sh.widths[li + 1];
        bool relu = li < sh.n_layers - 1 || sh.relu_out;
        for (int j = 0; j < wout; ++j) {
            float acc = 0.0f;
            for (int k = 0; k < win; ++k) acc = xadd(acc, xmul(wt[k * wout + j], cur[k * FE_THREADS]));
            nxt[j * FE_THREADS] = relu ? fmaxf(acc, 0.0f) : acc;
        }
        wt += win * wout;
        float *t = cur;
        cur = nxt;
        nxt = t;
    }
    return cur[0];
}

// Stage the MLP weights transposed (k-major) into shared memory; returns the
// number of floats written (rounded up to a multiple of 4).
__device__ __forceinline__ int stage_weights_t(const float *__restrict__ weights, const MlpShape &sh, float *wt) {
    int off = 0;
    for (int li = 0; li < sh.n_layers; ++li) {
        int win = sh.widths[li], wout = sh.widths[li + 1];
        for (int q = threadIdx.x; q < win * wout; q += blockDim.x) {
            int j = q / win, k = q % win;
            wt[off + k * wout + j] = weights[off + q];
        }
        off += win * wout;
    }
    return (off + 3) & ~3;
}

}  // namespace nvol
