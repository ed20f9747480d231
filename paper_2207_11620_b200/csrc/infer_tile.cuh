// One 128-sample tile of tcgen05 field inference (encode + MLP forward), shared by
// infer_tc_kernel (decode, batched Phi: infer_tc.cu) and the in-shader tcgen05 ray marcher
// (rm_tc_kernel: render.cu).  Every value-producing operation is an explicit round-to-nearest
// intrinsic (no contraction decisions left to the compiler), so the two translation units --
// compiled with different -fmad settings -- produce bit-identical field values.
//
// Reference: _kernels.py:31-79 (encode), network.py:43-62 (forward); the split-fp16
// forward and the activation scaling are described in tc.cuh.
#pragma once
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace nvol {

constexpr int IT_THREADS = 256;
constexpr int IT_TILE = 128;
constexpr int IT_LB = 4;  // levels whose corner gathers are in flight together

struct InferShape {
    int m, n, nin, ninp, nn, nh, relu_out;
    uint32_t o_w[8], o_wout, o_wlo[8], o_x, o_xlo, o_h, o_hlo, o_part, smem_bytes, t_alloc;
};

static inline int build_infer_shape(InferShape &s, int m, int n, int nn, int nh, int relu_out) {
    s.m = m;
    s.n = n;
    s.nin = m * n;
    s.ninp = (s.nin + 15) & ~15;
    s.nn = nn;
    s.nh = nh;
    s.relu_out = relu_out;
    if (nh < 1 || nh > 8 || !(nn == 16 || nn == 32 || nn == 64 || nn == 128) || s.ninp > 128) return 0;
    uint32_t off = 0;
    auto take = [&](uint32_t bytes) {
        uint32_t r = off;
        off += (bytes + 127) & ~127u;
        return r;
    };
    // [0, o_x): the packed weight image; each layer's lo tile directly follows its hi
    // tile, so [W_hi; W_lo] is one N = 2*nn B operand (hi*W_hi and hi*W_lo in one MMA)
    for (int i = 0; i < nh; ++i) {
        s.o_w[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
        s.o_wlo[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
    }
    s.o_wout = take(4u * nn);
    s.o_x = take(2u * IT_TILE * s.ninp);
    s.o_xlo = take(2u * IT_TILE * s.ninp);
    // one activation buffer (+ lo): a layer's epilogue overwrites the operand
    // its own MMA already consumed
    s.o_h = take(2u * IT_TILE * nn);
    s.o_hlo = take(2u * IT_TILE * nn);
    s.o_part = take(4u * IT_TILE);
    s.smem_bytes = off;
    s.t_alloc = 2 * nn < 32 ? 32 : 2 * nn;
    return s.smem_bytes <= 112 * 1024;
}

__device__ __forceinline__ void st_f16x16(uint8_t *tile, int row, int c, int w, const float *v) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const float *a = v + q * 8;
        uint4 pk = make_uint4(tc::pack_half2(a[0], a[1]), tc::pack_half2(a[2], a[3]), tc::pack_half2(a[4], a[5]),
                              tc::pack_half2(a[6], a[7]));
        *reinterpret_cast<uint4 *>(tile + tc::tile_off(row, c + q * 8, w)) = pk;
    }
}

__device__ __forceinline__ uint32_t slot32i(uint32_t vx, uint32_t vy, uint32_t vz, uint32_t r1, uint32_t mask,
                                            bool dense) {
    if (dense) return (vz * r1 + vy) * r1 + vx;
    return (vx ^ (vy * 2654435761u) ^ (vz * 805459861u)) & mask;
}


// Prologue of a persistent inference CTA (all IT_THREADS threads): the packed weight image into
// shared memory, zeroed feature tiles (the padding columns stay 0), TMEM, the MMA mbarrier.
__device__ __forceinline__ void infer_prologue(uint8_t *smem, const InferShape &sh, const uint8_t *__restrict__ wimg,
                                               uint64_t *mbar, uint32_t *tmem_base_sh) {
    const int tid = threadIdx.x, warp = tid >> 5;
    const uint4 *src = reinterpret_cast<const uint4 *>(wimg);
    uint4 *dst = reinterpret_cast<uint4 *>(smem);
    for (int q = tid; q < (int)(sh.o_x / 16); q += IT_THREADS) dst[q] = __ldg(src + q);
    for (int q = tid; q < 2 * IT_TILE * sh.ninp / 8; q += IT_THREADS)   // hi + lo feature tiles
        reinterpret_cast<uint4 *>(smem + sh.o_x)[q] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tc::tmem_alloc(tmem_base_sh, sh.t_alloc);
    if (tid == 0) {
        tc::mbar_init(mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
}

__device__ __forceinline__ void infer_teardown(uint32_t tmem, const InferShape &sh) {
    tc::fence_before();
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) tc::tmem_dealloc(tmem, sh.t_alloc);
}

// One tile (all IT_THREADS threads): thread (s = tid % 128, h = tid / 128) encodes half of sample
// s's levels at (x, y, z) (bit-exact fp32, zero-weight corners skipped), the MLP runs on the tensor
// cores, and the returned value -- Phi(x, y, z) with the output activation, before any decode
// scaling -- is meaningful in the h == 0 threads (valid samples).
// PAIR: fetch x-adjacent corner pairs with one 16-byte load where the slots allow (arbitrary
// sample positions: render / field evaluation).  Voxel-centre decodes skip most corners by zero
// weight instead, where the pair logic only costs issue slots.
template <int NF, bool PAIR>
__device__ __forceinline__ float infer_tile(uint8_t *smem, const InferShape &sh, const GridTables &tab,
                                            const float *__restrict__ params, float x, float y, float z, bool valid,
                                            uint32_t tmem, uint64_t *mbar, uint32_t &phase) {
    const int tid = threadIdx.x, s = tid & (IT_TILE - 1), h = tid >> 7, warp = tid >> 5;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int NN = sh.nn, NINP = sh.ninp, NH = sh.nh, M = sh.m;
    const uint32_t tlo = tmem + NN;
    const float *s_wout = reinterpret_cast<const float *>(smem + sh.o_wout);
    float *s_part = reinterpret_cast<float *>(smem + sh.o_part);
    const uint32_t idesc = tc::make_idesc(128, NN, 0, 0), idesc2 = tc::make_idesc(128, 2 * NN, 0, 0);
    const int mh = (M + 1) / 2, l_lo = h * mh, l_hi = min(M, (h + 1) * mh);
    const int c0 = NN >= 32 ? h * (NN >> 1) : 0, nc = NN >= 32 ? (NN >> 1) : (h == 0 ? NN : 0);
    uint8_t *sx = smem + sh.o_x, *sxl = smem + sh.o_xlo;
    // levels in batches of IT_LB: every corner load of the batch is issued
    // before any is consumed (IT_LB x 8 gathers in flight per thread)
    for (int lb = l_lo; lb < l_hi; lb += IT_LB) {
        float vals[IT_LB][8][NF];
        float fxs[IT_LB], fys[IT_LB], fzs[IT_LB];
#pragma unroll
        for (int u = 0; u < IT_LB; ++u) {
            const int l = min(lb + u, l_hi - 1);  // a past-the-end slot recomputes the last level (discarded)
            {
                const int32_t res = tab.res[l];
                const uint32_t r1 = (uint32_t)res + 1, mask = (uint32_t)(tab.entries[l] - 1);
                const bool dense = tab.dense[l] != 0;
                const float *tb = params + tab.offset[l];
                const Cell<float> c = cell_of<float>(x, y, z, res);
                fxs[u] = c.fx;
                fys[u] = c.fy;
                fzs[u] = c.fz;
                const uint32_t cx = (uint32_t)c.cx, cy = (uint32_t)c.cy, cz = (uint32_t)c.cz;
                // corners whose weight is exactly 0 contribute w*v = +-0 to a
                // sum that starts at +0, i.e. nothing: their gathers are skipped
                // (bit-exact for finite tables).  Voxel-centre decodes hit this
                // on every level finer than the output grid (fx = fy = fz = 0).
                const bool zx = c.fx == 0.0f, zy = c.fy == 0.0f, zz = c.fz == 0.0f;
                if constexpr (NF == 2 && PAIR) {
                    // x-adjacent corners (k, k+1) whose slots are an aligned pair {lo, lo+1}
                    // (dense levels, and hashed levels at even x: the hash differs in bit 0)
                    // share one 16-byte load; the pair is aligned iff address(entry 0) / 8 + lo is even
                    const uint32_t par = (uint32_t)((reinterpret_cast<uintptr_t>(tb) >> 3) & 1u);
#pragma unroll
                    for (int k = 0; k < 8; k += 2) {
                        const bool s0 = ((k & 2) && zy) || ((k & 4) && zz), s1 = s0 || zx;
                        const uint32_t sa = slot32i(cx, cy + ((k >> 1) & 1), cz + ((k >> 2) & 1), r1, mask, dense);
                        const uint32_t sb =
                            slot32i(cx + 1, cy + ((k >> 1) & 1), cz + ((k >> 2) & 1), r1, mask, dense);
                        const uint32_t lo = min(sa, sb);
                        // branch-free (predicated loads): every gather of the level batch stays in flight
                        const bool pair = !s1 && max(sa, sb) == lo + 1 && ((lo + par) & 1u) == 0u;
                        const float2 z2 = make_float2(0.0f, 0.0f);
                        const float4 q = pair ? __ldg(reinterpret_cast<const float4 *>(tb + 2 * (size_t)lo))
                                              : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                        const float2 a2 = (!pair && !s0) ? __ldg(reinterpret_cast<const float2 *>(tb) + sa) : z2;
                        const float2 b2 = (!pair && !s1) ? __ldg(reinterpret_cast<const float2 *>(tb) + sb) : z2;
                        const bool a_first = sa == lo;
                        const float2 qa = a_first ? make_float2(q.x, q.y) : make_float2(q.z, q.w);
                        const float2 qb = a_first ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
                        const float2 va = pair ? qa : a2, vb = pair ? qb : b2;
                        vals[u][k][0] = va.x;
                        vals[u][k][1] = va.y;
                        vals[u][k + 1][0] = vb.x;
                        vals[u][k + 1][1] = vb.y;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        const bool skip = ((k & 1) && zx) || ((k & 2) && zy) || ((k & 4) && zz);
                        const uint32_t sl =
                            slot32i(cx + (k & 1), cy + ((k >> 1) & 1), cz + ((k >> 2) & 1), r1, mask, dense);
                        if constexpr (NF == 2) {
                            const float2 v = skip ? make_float2(0.0f, 0.0f)
                                                  : __ldg(reinterpret_cast<const float2 *>(tb) + sl);
                            vals[u][k][0] = v.x;
                            vals[u][k][1] = v.y;
                        } else {
#pragma unroll
                            for (int f = 0; f < NF; ++f)
                                vals[u][k][f] = skip ? 0.0f : __ldg(tb + (size_t)sl * NF + f);
                        }
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < IT_LB; ++u) {
            const int l = lb + u;
            if (l < l_hi) {
                float acc[NF];
#pragma unroll
                for (int f = 0; f < NF; ++f) acc[f] = 0.0f;
                // corner weights in the reference order w = (wx * wy) * wz (_kernels.py:59-61)
                const float ox = xsub(1.0f, fxs[u]), oy = xsub(1.0f, fys[u]), oz = xsub(1.0f, fzs[u]);
                const float wxy[4] = {xmul(ox, oy), xmul(fxs[u], oy), xmul(ox, fys[u]), xmul(fxs[u], fys[u])};
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float w = xmul(wxy[k & 3], (k & 4) ? fzs[u] : oz);
#pragma unroll
                    for (int f = 0; f < NF; ++f) acc[f] = xadd(acc[f], xmul(w, vals[u][k][f]));
                }
#pragma unroll
                for (int f = 0; f < NF; ++f) {
                    __half hi, lw;
                    tc::split_f16(valid ? acc[f] * tc::kActScale : 0.0f, hi, lw);
                    const uint32_t o = tc::tile_off(s, l * NF + f, NINP);
                    *reinterpret_cast<__half *>(sx + o) = hi;
                    *reinterpret_cast<__half *>(sxl + o) = lw;
                }
            }
        }
    }
    tc::fence_proxy_async();
    __syncthreads();
    float outp = 0.0f;
    for (int li = 0; li < NH; ++li) {
        const int win = li == 0 ? NINP : NN;
        if (tid == 0) {
            tc::fence_after();
            const uint32_t ah = tc::smem_u32(smem + (li == 0 ? sh.o_x : sh.o_h));
            const uint32_t al = tc::smem_u32(smem + (li == 0 ? sh.o_xlo : sh.o_hlo));
            const uint32_t bh = tc::smem_u32(smem + sh.o_w[li]);  // [W_hi; W_lo] rows 0..2NN-1
            const uint32_t sbo = (win / 8) * 128;
            for (int k = 0; k < win / 16; ++k) {
                const uint64_t adh = tc::make_desc(ah + k * 256, 128, sbo), adl = tc::make_desc(al + k * 256, 128, sbo);
                const uint64_t bdh = tc::make_desc(bh + k * 256, 128, sbo);
                // [hi*W_hi | hi*W_lo] -> [tmem | tlo] in one N = 2*NN MMA, then lo*W_hi -> tlo
                tc::mma_f16(tmem, adh, bdh, idesc2, k > 0);
                tc::mma_f16(tlo, adl, bdh, idesc, 1);
            }
            tc::mma_commit(mbar);
        }
        tc::mbar_wait_sleep(mbar, phase);
        phase ^= 1;
        tc::fence_after();
        uint8_t *dst = smem + sh.o_h, *dstl = smem + sh.o_hlo;
        for (int c = c0; c < c0 + nc; c += 16) {   // values carry kActScale (see tc.cuh)
            float v[16], vl[16];
            tc::tmem_ld16(tmem + lane_base + c, v);
            tc::tmem_ld16(tlo + lane_base + c, vl);
            tc::tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = fmaxf(__fmaf_rn(vl[e], 1.0f / tc::kLoScale, v[e]), 0.0f);
            if (li < NH - 1) {
#pragma unroll
                for (int e = 0; e < 16; ++e) vl[e] = __fmul_rn(__fsub_rn(v[e], __half2float(__float2half_rn(v[e]))), tc::kLoScale);
                st_f16x16(dst, s, c, NN, v);
                st_f16x16(dstl, s, c, NN, vl);
            } else {
#pragma unroll
                for (int e = 0; e < 16; ++e) outp = __fmaf_rn(s_wout[c + e], v[e], outp);
            }
        }
        tc::fence_before();
        tc::fence_proxy_async();
        __syncthreads();
    }
    if (h == 1) s_part[s] = outp;
    __syncthreads();
    float o = 0.0f;
    if (h == 0) {
        o = __fmul_rn(__fadd_rn(outp, s_part[s]), 1.0f / tc::kActScale);
        if (sh.relu_out) o = fmaxf(o, 0.0f);
    }
    __syncthreads();  // s_part and the tiles are reused by the next tile
    return o;
}

}  // namespace nvol
