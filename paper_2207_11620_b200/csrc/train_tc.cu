// Training step forward/backward on the tensor cores (sm_100a), as three
// specialised kernels that each run at their own bound:
//
//  1. encode_tiles_kernel — hash-grid gather (_kernels.py:31-79), one thread
//     per (sample, level), full occupancy: L2-latency/throughput bound.  The
//     fp32 features (bit-exact) are rounded to fp16 and written straight
//     into the UMMA core-matrix tile layout of tc.cuh (4 MB at cfg2, stays
//     in L2).
//  2. mlp_tc_kernel — one persistent CTA per SM walks 128-sample tiles:
//     forward (network.py:61-74) as one tcgen05.mma chain per layer
//     (M=128 samples, fp16 operands, fp32 accumulator in TMEM) with a
//     ReLU/fp16 epilogue back into smem; output layer and L1/L2 gradient on
//     CUDA cores (network.py:96-114); backward (network.py:76-93): per layer
//     dW_j += delta^T H_j (accumulated in TMEM across all tiles of the CTA)
//     and dX = delta W_j masked by the stored activations.  dL/dfeat leaves
//     as fp32; dW leaves once per CTA as fp32 partials.
//  3. scatter_kernel — encoder backward (_kernels.py:82-92): corners
//     recomputed from the coordinates; the small dense coarse levels
//     (contended by every sample) accumulate in shared memory and leave as
//     per-CTA partials, the fine levels scatter with float2 REDs.
// Partials are summed in fixed CTA order (deterministic MLP and coarse-level
// gradients).
//
// Accuracy contract (north star): fp16 operands / fp32 accumulation, MLP
// outputs and gradients within 1e-2 relative of the fp32 reference.
#include <cuda_fp16.h>

#include "common.cuh"
#include "tc.cuh"

namespace nvol {

constexpr int TC_THREADS = 256;
constexpr int TILE = 128;
constexpr int MAX_NH = 8;
constexpr int SC_THREADS = 1024;
constexpr uint32_t COARSE_BYTES = 48 * 1024;

struct TcShape {
    int m, n, nin, ninp, nn, nh;
    int relu_out, loss_kind;
    uint32_t o_w[MAX_NH], o_wout, o_wlo[MAX_NH], o_x, o_xlo, o_h[MAX_NH + 1], o_hlo[2], o_d[2], o_dout, o_misc,
        smem_bytes;
    uint32_t t_f, t_flo, t_g, t_dw[MAX_NH], t_dwout, t_alloc;
    int64_t w_floats;
};

static int build_shape(TcShape &s, int m, int n, int nn, int nh, int relu_out, int loss_kind) {
    s.m = m;
    s.n = n;
    s.nin = m * n;
    s.ninp = (s.nin + 15) & ~15;
    s.nn = nn;
    s.nh = nh;
    s.relu_out = relu_out;
    s.loss_kind = loss_kind;
    if (nh < 1 || nh > MAX_NH) return 0;
    if (!(nn == 16 || nn == 32 || nn == 64 || nn == 128)) return 0;
    if (s.ninp > 128) return 0;
    uint32_t off = 0;
    auto take = [&](uint32_t bytes) {
        uint32_t r = off;
        off += (bytes + 127) & ~127u;
        return r;
    };
    for (int i = 0; i < nh; ++i) s.o_w[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
    s.o_wout = take(4u * nn);
    for (int i = 0; i < nh; ++i) s.o_wlo[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
    s.o_x = take(2u * TILE * s.ninp);      // [o_x, o_x + 2 tiles): hi then lo feature tile
    s.o_xlo = take(2u * TILE * s.ninp);
    s.o_h[0] = s.o_x;
    for (int i = 1; i <= nh; ++i) s.o_h[i] = take(2u * TILE * nn);
    s.o_hlo[0] = take(2u * TILE * nn);
    s.o_hlo[1] = take(2u * TILE * nn);
    s.o_d[0] = take(2u * TILE * nn);
    s.o_d[1] = take(2u * TILE * nn);
    s.o_dout = take(2048 + 256);
    s.o_misc = take(4u * TILE * 4 + 64);
    take(4096);  // slack: padded-M operand rows read past the last tile (values unused)
    s.smem_bytes = off;
    uint32_t col = 0;
    s.t_f = col;
    col += nn;
    s.t_flo = col;  // forward lo-product accumulator (split-fp16 forward, see tc.cuh)
    col += nn;
    s.t_g = col;
    col += (uint32_t)max(s.ninp, nn);
    for (int i = 0; i < nh; ++i) {
        s.t_dw[i] = col;
        col += (i == 0) ? s.ninp : nn;
    }
    s.t_dwout = col;
    col += nn;
    if (col > 512) return 0;
    uint32_t a = 32;
    while (a < col) a <<= 1;
    s.t_alloc = a;
    s.w_floats = (int64_t)nn * s.nin + (int64_t)(nh - 1) * nn * nn + nn;
    return s.smem_bytes <= 227 * 1024;
}

// Hash-grid levels fit 32-bit slot arithmetic (entries <= 2^24 for hashed
// levels, dense levels hold <= T entries).
__device__ __forceinline__ uint32_t slot32(uint32_t vx, uint32_t vy, uint32_t vz, uint32_t r1, uint32_t mask,
                                           bool dense) {
    if (dense) return (vz * r1 + vy) * r1 + vx;
    return (vx ^ (vy * 2654435761u) ^ (vz * 805459861u)) & mask;
}

struct Cell32 {
    uint32_t cx, cy, cz;
    float fx, fy, fz;
};

__device__ __forceinline__ Cell32 cell32(float x, float y, float z, int32_t res) {
    Cell<float> c = cell_of<float>(x, y, z, res);
    return Cell32{(uint32_t)c.cx, (uint32_t)c.cy, (uint32_t)c.cz, c.fx, c.fy, c.fz};
}

__device__ __forceinline__ float cw32(const Cell32 &c, int k) {
    float w = (k & 1) ? c.fx : xsub(1.0f, c.fx);
    w = xmul(w, (k & 2) ? c.fy : xsub(1.0f, c.fy));
    return xmul(w, (k & 4) ? c.fz : xsub(1.0f, c.fz));
}

// ============================================================================ 1. encode
template <int NF>
__global__ void __launch_bounds__(256) encode_tiles_kernel(const float *__restrict__ coords, int64_t b,
                                                           const float *__restrict__ params, const GridTables tab,
                                                           int ninp, uint8_t *__restrict__ xtiles) {
    const int m = tab.n_levels;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b * m) return;
    // level-major: a warp covers 32 consecutive samples of one level (uniform
    // level constants, coalesced coordinates, L1 reuse on coarse levels)
    const int l = (int)(t / b);
    const int64_t i = t - (int64_t)l * b;
    const int32_t res = tab.res[l];
    const uint32_t r1 = (uint32_t)res + 1, mask = (uint32_t)(tab.entries[l] - 1);
    const bool dense = tab.dense[l] != 0;
    const float *tb = params + tab.offset[l];
    Cell32 c = cell32(__ldg(coords + 3 * i), __ldg(coords + 3 * i + 1), __ldg(coords + 3 * i + 2), res);
    float acc[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) acc[f] = 0.0f;
    uint32_t sl[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) sl[k] = slot32(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), r1, mask, dense);
    if constexpr (NF == 2) {
        // x-adjacent corners (k, k+1) whose slots differ only in bit 0 share
        // one aligned 16-byte entry pair: fetch it with a single float4 load
        // (a pair {e, e+1} is 16-byte aligned iff the level offset + 2e is a
        // multiple of 4 floats; odd-sized dense levels shift later offsets)
        float2 v[8];
        const uint32_t par = (uint32_t)(tab.offset[l] >> 1) & 1u;
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const uint32_t lo = min(sl[k], sl[k + 1]);
            if (max(sl[k], sl[k + 1]) == lo + 1 && ((lo + par) & 1u) == 0u) {
                const float4 q = __ldg(reinterpret_cast<const float4 *>(tb + 2 * (size_t)lo));
                const bool lo_first = sl[k] == lo;
                v[k] = lo_first ? make_float2(q.x, q.y) : make_float2(q.z, q.w);
                v[k + 1] = lo_first ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
            } else {
                v[k] = __ldg(reinterpret_cast<const float2 *>(tb) + sl[k]);
                v[k + 1] = __ldg(reinterpret_cast<const float2 *>(tb) + sl[k + 1]);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float w = cw32(c, k);
            acc[0] = xadd(acc[0], xmul(w, v[k].x));
            acc[1] = xadd(acc[1], xmul(w, v[k].y));
        }
    } else {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            float w = cw32(c, k);
#pragma unroll
            for (int f = 0; f < NF; ++f) acc[f] = xadd(acc[f], xmul(w, __ldg(tb + (size_t)sl[k] * NF + f)));
        }
    }
    const int64_t tile = i >> 7;
    const int s = (int)(i & 127);
    // per tile: fp16 hi tile followed by the fp16 lo tile (split-fp16 forward)
    uint8_t *base = xtiles + tile * (int64_t)(2 * TILE * ninp * 2);
    uint8_t *base_lo = base + TILE * ninp * 2;
    __half hv[NF], lv[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) tc::split_f16(acc[f] * tc::kActScale, hv[f], lv[f]);
#pragma unroll
    for (int f = 0; f < NF; f += 2) {
        if constexpr (NF == 1) {
            *reinterpret_cast<__half *>(base + tc::tile_off(s, l, ninp)) = hv[0];
            *reinterpret_cast<__half *>(base_lo + tc::tile_off(s, l, ninp)) = lv[0];
        } else {
            const uint32_t o = tc::tile_off(s, l * NF + f, ninp);
            *reinterpret_cast<__half2 *>(base + o) = __halves2half2(hv[f], hv[f + 1]);
            *reinterpret_cast<__half2 *>(base_lo + o) = __halves2half2(lv[f], lv[f + 1]);
        }
    }
    if (l == m - 1) {
        for (int cidx = m * NF; cidx < ninp; ++cidx) {
            *reinterpret_cast<__half *>(base + tc::tile_off(s, cidx, ninp)) = __float2half_rn(0.0f);
            *reinterpret_cast<__half *>(base_lo + tc::tile_off(s, cidx, ninp)) = __float2half_rn(0.0f);
        }
    }
}

// ============================================================================ 2. MLP
__device__ __forceinline__ void half_cols(int w, int h, int &c0, int &nc) {
    if (w >= 32) {
        c0 = h * (w >> 1);
        nc = w >> 1;
    } else {
        c0 = 0;
        nc = h == 0 ? w : 0;
    }
}

__device__ __forceinline__ void store_row_f16(uint8_t *tile, int row, int c, int w, const float *v16, bool relu) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        float a[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = relu ? fmaxf(v16[q * 8 + e], 0.0f) : v16[q * 8 + e];
        uint4 pk = make_uint4(tc::pack_half2(a[0], a[1]), tc::pack_half2(a[2], a[3]), tc::pack_half2(a[4], a[5]),
                              tc::pack_half2(a[6], a[7]));
        *reinterpret_cast<uint4 *>(tile + tc::tile_off(row, c + q * 8, w)) = pk;
    }
}

__device__ __forceinline__ void load_row_f16(const uint8_t *tile, int row, int c, int w, float *v16) {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        uint4 pk = *reinterpret_cast<const uint4 *>(tile + tc::tile_off(row, c + q * 8, w));
        const __half2 *h2 = reinterpret_cast<const __half2 *>(&pk);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            float2 f = __half22float2(h2[e]);
            v16[q * 8 + 2 * e] = f.x;
            v16[q * 8 + 2 * e + 1] = f.y;
        }
    }
}

// fp32 weights (flat buffer) -> the shared-memory image the MLP kernels copy
// verbatim: W_0..W_{nh-1} as fp16 core-matrix tiles at o_w[i] (input columns
// padded to ninp with zeros) and the fp32 output row at o_wout.
struct MlpImage {
    uint32_t o_w[MAX_NH], o_wout, o_wlo[MAX_NH];
    int with_lo;
};

__global__ void pack_mlp_image_kernel(const float *__restrict__ wflat, int nin, int ninp, int nn, int nh,
                                      const MlpImage img, uint8_t *__restrict__ out) {
    const int stride = gridDim.x * blockDim.x;
    const int t0 = blockIdx.x * blockDim.x + threadIdx.x;
    const float *src = wflat;
    for (int i = 0; i < nh; ++i) {
        const int win = i == 0 ? nin : nn, wp = i == 0 ? ninp : nn;
        for (int q = t0; q < nn * wp; q += stride) {
            int o = q / wp, j = q % wp;
            const uint32_t off = tc::tile_off(o, j, wp);
            __half hi, lo;
            tc::split_f16(j < win ? src[o * win + j] : 0.0f, hi, lo);
            *reinterpret_cast<__half *>(out + img.o_w[i] + off) = hi;
            if (img.with_lo) *reinterpret_cast<__half *>(out + img.o_wlo[i] + off) = lo;
        }
        src += (int64_t)nn * win;
    }
    for (int q = t0; q < nn; q += stride) reinterpret_cast<float *>(out + img.o_wout)[q] = src[q];
}

// o_wlo == nullptr: hi tiles only (the inference kernels' image)
int pack_mlp_image(const float *wflat, int nin, int ninp, int nn, int nh, const uint32_t *o_w, uint32_t o_wout,
                   uint8_t *image, cudaStream_t s, const uint32_t *o_wlo) {
    MlpImage img;
    for (int i = 0; i < nh; ++i) {
        img.o_w[i] = o_w[i];
        img.o_wlo[i] = o_wlo ? o_wlo[i] : 0;
    }
    img.o_wout = o_wout;
    img.with_lo = o_wlo != nullptr;
    pack_mlp_image_kernel<<<64, 256, 0, s>>>(wflat, nin, ninp, nn, nh, img, image);
    return check_launch("pack_mlp_image");
}

__global__ void __launch_bounds__(TC_THREADS, 1) mlp_tc_kernel(
    const uint8_t *__restrict__ xtiles, const float *__restrict__ targets, int64_t b, double inv_bglobal, float dscale,
    const TcShape sh, const uint8_t *__restrict__ wimg, double *__restrict__ loss_sum, float *__restrict__ dfeat,
    int64_t stride, float *__restrict__ partials) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x;
    const int s = tid & (TILE - 1);
    const int h = tid >> 7;
    const int warp = tid >> 5;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int NN = sh.nn, NINP = sh.ninp, NH = sh.nh, NIN = sh.nin;
    {
        // fp16 weight tiles + fp32 output row, pre-packed once per step (independent 16-byte loads)
        const uint4 *src = reinterpret_cast<const uint4 *>(wimg);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int q = tid; q < (int)(sh.o_x / 16); q += TC_THREADS) dst[q] = __ldg(src + q);
        for (int q = tid; q < (2048 + 256) / 16; q += TC_THREADS)
            reinterpret_cast<uint4 *>(smem + sh.o_dout)[q] = make_uint4(0, 0, 0, 0);
    }
    if (warp == 0) tc::tmem_alloc(&tmem_base_sh, sh.t_alloc);
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::fence_mbar_init();
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base_sh;
    uint32_t phase = 0;
    float *s_part = reinterpret_cast<float *>(smem + sh.o_misc);
    float *s_delta = s_part + TILE;
    const float *s_wout = reinterpret_cast<const float *>(smem + sh.o_wout);
    const uint32_t idesc_fwd = tc::make_idesc(128, NN, 0, 0);
    const int64_t ntiles = (b + TILE - 1) / TILE;
    const int tile_u4 = TILE * NINP * 2 / 16;
    bool first_tile = true;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row = tile * TILE + s;
        const bool valid = row < b;
        const float tgt = valid ? targets[row] : 0.0f;
        // ---- X tile: global (L2) -> smem; rows past the batch are zeroed
        {
            // hi tile then lo tile (contiguous both in global and in smem: o_xlo = o_x + tile bytes)
            const uint4 *src = reinterpret_cast<const uint4 *>(xtiles + tile * (int64_t)(2 * TILE * NINP * 2));
            uint4 *dst = reinterpret_cast<uint4 *>(smem + sh.o_x);
            const int64_t nvalid = b - tile * TILE;
            for (int q = tid; q < 2 * tile_u4; q += TC_THREADS) {
                // core-matrix row (q % tile_u4)*16 bytes -> sample row ((..)/(NINP/8))*8 + (q%8)
                const int qq = q % tile_u4;
                int cm = qq >> 3, r = ((cm / (NINP / 8)) << 3) + (qq & 7);
                dst[q] = r < nvalid ? src[q] : make_uint4(0, 0, 0, 0);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();

        // ---- forward
        float outp = 0.0f;
        for (int i = 0; i < NH; ++i) {
            const int win = (i == 0) ? NINP : NN;
            if (tid == 0) {
                // split-fp16 forward: hi*hi -> t_f; lo*hi + hi*lo -> t_flo (x kLoScale)
                tc::fence_after();
                const uint32_t ah = tc::smem_u32(smem + sh.o_h[i]);
                const uint32_t al = tc::smem_u32(smem + (i == 0 ? sh.o_xlo : sh.o_hlo[(i - 1) & 1]));
                const uint32_t bh = tc::smem_u32(smem + sh.o_w[i]);
                const uint32_t bl = tc::smem_u32(smem + sh.o_wlo[i]);
                const uint32_t sbo = (win / 8) * 128;
                for (int k = 0; k < win / 16; ++k) {
                    const uint64_t adh = tc::make_desc(ah + k * 256, 128, sbo), adl = tc::make_desc(al + k * 256, 128, sbo);
                    const uint64_t bdh = tc::make_desc(bh + k * 256, 128, sbo), bdl = tc::make_desc(bl + k * 256, 128, sbo);
                    tc::mma_f16(tmem + sh.t_f, adh, bdh, idesc_fwd, k > 0);
                    tc::mma_f16(tmem + sh.t_flo, adl, bdh, idesc_fwd, k > 0);
                    tc::mma_f16(tmem + sh.t_flo, adh, bdl, idesc_fwd, 1);
                }
                tc::mma_commit(&mbar);
            }
            tc::mbar_wait(&mbar, phase);
            phase ^= 1;
            tc::fence_after();
            int c0, nc;
            half_cols(NN, h, c0, nc);
            uint8_t *dst = smem + sh.o_h[i + 1];
            uint8_t *dst_lo = smem + sh.o_hlo[i & 1];
            // accumulator = kActScale * pre-activation: ReLU commutes with the
            // positive scale, so the stored activations stay scaled too
            for (int c = c0; c < c0 + nc; c += 16) {
                float v[16], vl[16];
                tc::tmem_ld16(tmem + lane_base + sh.t_f + c, v);
                tc::tmem_ld16(tmem + lane_base + sh.t_flo + c, vl);
                tc::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] = fmaxf(v[e] + vl[e] * (1.0f / tc::kLoScale), 0.0f);
                store_row_f16(dst, s, c, NN, v, false);
                if (i < NH - 1) {
                    // lo part of the activation for the next layer's split product
#pragma unroll
                    for (int e = 0; e < 16; ++e) vl[e] = (v[e] - __half2float(__float2half_rn(v[e]))) * tc::kLoScale;
                    store_row_f16(dst_lo, s, c, NN, vl, false);
                }
                if (i == NH - 1) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) outp += s_wout[c + e] * fmaxf(v[e], 0.0f);
                }
            }
            tc::fence_before();
            tc::fence_proxy_async();
            __syncthreads();
        }
        // ---- output layer + loss gradient
        if (h == 1) s_part[s] = outp;
        __syncthreads();
        if (h == 0) {
            float o = (outp + s_part[s]) * (1.0f / tc::kActScale);
            float pred = sh.relu_out ? fmaxf(o, 0.0f) : o;
            double d = (double)pred - (double)tgt;
            double g, sl;
            if (sh.loss_kind == 0) {
                sl = fabs(d);
                g = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : 0.0)) * inv_bglobal;
            } else {
                sl = d * d;
                g = 2.0 * d * inv_bglobal;
            }
            float gf = (float)g;
            if (sh.relu_out && !(pred > 0.0f)) gf = 0.0f;
            if (!valid) {
                gf = 0.0f;
                sl = 0.0;
            }
            s_delta[s] = gf;
            *reinterpret_cast<__half *>(smem + sh.o_dout + (s >> 3) * 128 + (s & 7) * 16) = __float2half_rn(gf * dscale);
            for (int o2 = 16; o2 > 0; o2 >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o2);
            if ((tid & 31) == 0) atomicAdd(loss_sum, sl);
        }
        __syncthreads();
        {
            int c0, nc;
            half_cols(NN, h, c0, nc);
            const float g = s_delta[s] * dscale;
            const uint8_t *hn = smem + sh.o_h[NH];
            uint8_t *dd = smem + sh.o_d[0];
            for (int c = c0; c < c0 + nc; c += 16) {
                float hv[16], dv[16];
                load_row_f16(hn, s, c, NN, hv);
#pragma unroll
                for (int e = 0; e < 16; ++e) dv[e] = hv[e] > 0.0f ? g * s_wout[c + e] : 0.0f;
                store_row_f16(dd, s, c, NN, dv, false);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();

        // ---- backward
        int cur = 0;
        for (int j = NH - 1; j >= 0; --j) {
            const int win = (j == 0) ? NINP : NN;
            if (tid == 0) {
                tc::fence_after();
                const uint32_t dA = tc::smem_u32(smem + sh.o_d[cur]);
                if (j == NH - 1) {
                    const uint32_t a0 = tc::smem_u32(smem + sh.o_dout);
                    const uint32_t b0 = tc::smem_u32(smem + sh.o_h[NH]);
                    const uint32_t id = tc::make_idesc(128, NN, 1, 1);
                    for (int k = 0; k < TILE / 16; ++k) {
                        uint64_t ad = tc::make_desc(a0 + k * 256, 128, 16);
                        uint64_t bd = tc::make_desc(b0 + k * 2 * (NN / 8) * 128, (NN / 8) * 128, 128);
                        tc::mma_f16(tmem + sh.t_dwout, ad, bd, id, (first_tile && k == 0) ? 0 : 1);
                    }
                }
                {
                    const uint32_t b0 = tc::smem_u32(smem + sh.o_h[j]);
                    const uint32_t id = tc::make_idesc(128, win, 1, 1);
                    for (int k = 0; k < TILE / 16; ++k) {
                        uint64_t ad = tc::make_desc(dA + k * 2 * (NN / 8) * 128, (NN / 8) * 128, 128);
                        uint64_t bd = tc::make_desc(b0 + k * 2 * (win / 8) * 128, (win / 8) * 128, 128);
                        tc::mma_f16(tmem + sh.t_dw[j], ad, bd, id, (first_tile && k == 0) ? 0 : 1);
                    }
                }
                {
                    const uint32_t b0 = tc::smem_u32(smem + sh.o_w[j]);
                    const uint32_t id = tc::make_idesc(128, win, 0, 1);
                    for (int k = 0; k < NN / 16; ++k) {
                        uint64_t ad = tc::make_desc(dA + k * 256, 128, (NN / 8) * 128);
                        uint64_t bd = tc::make_desc(b0 + k * 2 * (win / 8) * 128, (win / 8) * 128, 128);
                        tc::mma_f16(tmem + sh.t_g, ad, bd, id, k > 0);
                    }
                }
                tc::mma_commit(&mbar);
            }
            tc::mbar_wait(&mbar, phase);
            phase ^= 1;
            tc::fence_after();
            int c0, nc;
            half_cols(win, h, c0, nc);
            if (j > 0) {
                const uint8_t *hj = smem + sh.o_h[j];
                uint8_t *dn = smem + sh.o_d[cur ^ 1];
                for (int c = c0; c < c0 + nc; c += 16) {
                    float v[16], hv[16];
                    tc::tmem_ld16(tmem + lane_base + sh.t_g + c, v);
                    tc::tmem_wait_ld();
                    load_row_f16(hj, s, c, NN, hv);
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = hv[e] > 0.0f ? v[e] : 0.0f;
                    store_row_f16(dn, s, c, NN, v, false);
                }
            } else {
                for (int c = c0; c < c0 + nc; c += 16) {
                    float v[16];
                    tc::tmem_ld16(tmem + lane_base + sh.t_g + c, v);
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] *= 1.0f / dscale;
                    if (valid) {
                        // feature-major dL/dfeat [NIN][B]: a warp stores 32 consecutive rows per column
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (c + e < NIN) dfeat[(int64_t)(c + e) * stride + row] = v[e];
                    }
                }
            }
            tc::fence_before();
            tc::fence_proxy_async();
            __syncthreads();
            cur ^= 1;
        }
        first_tile = false;
    }

    // ---- flush dW partials (fp32) once per CTA
    float *dst = partials + (int64_t)blockIdx.x * sh.w_floats;
    if (!first_tile) {
        const int o = (warp & 3) * 32 + (tid & 31);
        int64_t base = 0;
        for (int j = 0; j <= NH; ++j) {
            const int win = (j == 0) ? NIN : NN;
            const int wacc = (j == 0) ? NINP : NN;
            const int rows = (j == NH) ? 1 : NN;
            const uint32_t tcol = (j == NH) ? sh.t_dwout : sh.t_dw[j];
            const float unscale = 1.0f / (dscale * tc::kActScale);  // dW = (dscale*delta)^T (kActScale*H)
            int c0, nc;
            half_cols(wacc, h, c0, nc);
            for (int c = c0; c < c0 + nc; c += 16) {
                float v[16];
                tc::tmem_ld16(tmem + lane_base + tcol + c, v);
                tc::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) v[e] *= unscale;
                if (o < rows) {
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (c + e < win) dst[base + (int64_t)o * win + c + e] = v[e];
                }
            }
            base += (int64_t)rows * win;
        }
    } else {
        for (int64_t q = tid; q < sh.w_floats; q += TC_THREADS) dst[q] = 0.0f;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, sh.t_alloc);
}

// ============================================================================ 3. scatter
template <int NF>
__global__ void __launch_bounds__(SC_THREADS, 1) scatter_kernel(const float *__restrict__ coords,
                                                                const float *__restrict__ dfeat, int64_t b,
                                                                int64_t stride,
                                                                const GridTables tab, int n_coarse, int coarse_floats,
                                                                float *__restrict__ grads,
                                                                float *__restrict__ partials) {
    extern __shared__ float acc_s[];
    for (int q = threadIdx.x; q < coarse_floats; q += SC_THREADS) acc_s[q] = 0.0f;
    __syncthreads();
    const int m = tab.n_levels, nin = m * NF;
    const int64_t items = b * m;
    for (int64_t t = (int64_t)blockIdx.x * SC_THREADS + threadIdx.x; t < items; t += (int64_t)gridDim.x * SC_THREADS) {
        const int l = (int)(t / b);          // level-major, as the encode kernel
        const int64_t i = t - (int64_t)l * b;
        const int32_t res = tab.res[l];
        const uint32_t r1 = (uint32_t)res + 1, mask = (uint32_t)(tab.entries[l] - 1);
        const bool dense = tab.dense[l] != 0;
        Cell32 c = cell32(__ldg(coords + 3 * i), __ldg(coords + 3 * i + 1), __ldg(coords + 3 * i + 2), res);
        float d[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) d[f] = __ldg(dfeat + (int64_t)(l * NF + f) * stride + i);
        const bool coarse = l < n_coarse;
        float *gl = coarse ? acc_s + tab.offset[l] : grads + tab.offset[l];
        if constexpr (NF == 2) {
            const uint32_t par = (uint32_t)(tab.offset[l] >> 1) & 1u;
            if (!coarse) {
                // fine levels: x-adjacent corner pairs in one aligned 16-byte
                // entry pair go out as a single float4 RED
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    const uint32_t yo = (k >> 1) & 1, zo = (k >> 2) & 1;
                    uint32_t s0 = slot32(c.cx, c.cy + yo, c.cz + zo, r1, mask, dense);
                    uint32_t s1 = slot32(c.cx + 1, c.cy + yo, c.cz + zo, r1, mask, dense);
                    float w0 = cw32(c, k), w1 = cw32(c, k + 1);
                    const uint32_t lo = min(s0, s1);
                    if (max(s0, s1) == lo + 1 && ((lo + par) & 1u) == 0u) {   // adjacent and 16-byte aligned
                        float4 q = s0 == lo ? make_float4(w0 * d[0], w0 * d[1], w1 * d[0], w1 * d[1])
                                            : make_float4(w1 * d[0], w1 * d[1], w0 * d[0], w0 * d[1]);
                        atomicAdd(reinterpret_cast<float4 *>(gl + 2 * (size_t)lo), q);
                    } else {
                        atomicAdd(reinterpret_cast<float2 *>(gl) + s0, make_float2(w0 * d[0], w0 * d[1]));
                        atomicAdd(reinterpret_cast<float2 *>(gl) + s1, make_float2(w1 * d[0], w1 * d[1]));
                    }
                }
                continue;
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            uint32_t slot = slot32(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), r1, mask, dense);
            float w = cw32(c, k);
            float *g = gl + (size_t)slot * NF;
            if (coarse) {
#pragma unroll
                for (int f = 0; f < NF; ++f) atomicAdd(g + f, w * d[f]);
            } else if constexpr (NF == 2) {
                atomicAdd(reinterpret_cast<float2 *>(g), make_float2(w * d[0], w * d[1]));
            } else if constexpr (NF == 4 || NF == 8) {
#pragma unroll
                for (int q = 0; q < NF / 4; ++q)
                    atomicAdd(reinterpret_cast<float4 *>(g) + q,
                              make_float4(w * d[4 * q], w * d[4 * q + 1], w * d[4 * q + 2], w * d[4 * q + 3]));
            } else {
                atomicAdd(g, w * d[0]);
            }
        }
    }
    __syncthreads();
    float *dst = partials + (int64_t)blockIdx.x * coarse_floats;
    for (int q = threadIdx.x; q < coarse_floats; q += SC_THREADS) dst[q] = acc_s[q];
}

// g[i] += sum_c partials[c][i] in fixed c order.  Block = 32 outputs x 8
// CTA groups; the 8 group sums combine in fixed order through shared memory.
__global__ void __launch_bounds__(256) reduce_partials_kernel(const float *__restrict__ partials, int nparts,
                                                              int64_t n, float *__restrict__ g) {
    __shared__ float red[8][33];
    const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
    const int64_t i = (int64_t)blockIdx.x * 32 + lane;
    float acc = 0.0f;
    if (i < n)
        for (int c = grp; c < nparts; c += 8) acc += partials[(int64_t)c * n + i];
    red[grp][lane] = acc;
    __syncthreads();
    if (grp == 0 && i < n) {
        float s = 0.0f;
#pragma unroll
        for (int q = 0; q < 8; ++q) s += red[q][lane];
        g[i] += s;
    }
}

// ============================================================================ host side
// The batch is processed in `nchunks` row chunks on three streams so the
// L2-bound encode / scatter kernels of one chunk overlap the tensor-core
// MLP kernel of another (encode(c+1) || mlp(c) || scatter(c-1)); all of it
// is ordinary stream fork/join, so it captures into the step's CUDA graph.
constexpr int MAX_CHUNKS = 4;

struct TcPlan {
    TcShape sh;
    int grid_mlp, grid_sc, n_coarse, coarse_floats, nchunks;
    int64_t ntiles, chunk_tiles, off_x, off_dfeat, off_wpart, off_cpart, off_img, total;
};

static int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

static int make_plan(TcPlan &p, int64_t b, const GridTables &tab, int nn, int nh, int relu_out, int loss_kind) {
    if (!build_shape(p.sh, tab.n_levels, tab.n_feat, nn, nh, relu_out, loss_kind)) return 0;
    for (int l = 0; l < tab.n_levels; ++l)
        if (tab.entries[l] >= (1ll << 31)) return 0;
    const int sms = num_sms();
    p.ntiles = (b + TILE - 1) / TILE;
    // chunks of >= ~1.5 MLP tiles per SM: 2 chunks at B = 65,536
    p.nchunks = (int)(p.ntiles / (sms + sms / 2));
    p.nchunks = p.nchunks < 1 ? 1 : (p.nchunks > MAX_CHUNKS ? MAX_CHUNKS : p.nchunks);
    p.chunk_tiles = (p.ntiles + p.nchunks - 1) / p.nchunks;
    p.nchunks = (int)((p.ntiles + p.chunk_tiles - 1) / p.chunk_tiles);  // every chunk non-empty
    p.grid_mlp = (int)(p.chunk_tiles < sms ? p.chunk_tiles : sms);
    p.grid_sc = sms;
    p.n_coarse = 0;
    p.coarse_floats = 0;
    for (int l = 0; l < tab.n_levels; ++l) {
        int64_t end = tab.offset[l] + tab.entries[l] * tab.n_feat;
        if (!tab.dense[l] || end * 4 > (int64_t)COARSE_BYTES) break;
        p.n_coarse = l + 1;
        p.coarse_floats = (int)end;
    }
    auto al = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
    p.off_x = 0;
    p.off_dfeat = al(p.ntiles * TILE * p.sh.ninp * 4);  // hi + lo fp16 tiles
    p.off_wpart = p.off_dfeat + al(b * p.sh.nin * 4);
    p.off_cpart = p.off_wpart + al((int64_t)MAX_CHUNKS * p.grid_mlp * p.sh.w_floats * 4);
    p.off_img = p.off_cpart + al((int64_t)MAX_CHUNKS * p.grid_sc * p.coarse_floats * 4);
    p.total = p.off_img + al(p.sh.o_x) + 256;
    return 1;
}

int64_t train_tc_workspace(int64_t b, int m, int n, int nn, int nh) {
    // upper bound over level tables: the coarse prefix is capped by COARSE_BYTES
    TcPlan p;
    if (!build_shape(p.sh, m, n, nn, nh, 1, 0)) return 0;
    const int sms = num_sms();
    int64_t ntiles = (b + TILE - 1) / TILE;
    int grid_mlp = (int)(ntiles < sms ? ntiles : sms);
    auto al = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
    return al(ntiles * TILE * p.sh.ninp * 4) + al(b * p.sh.nin * 4) +
           al((int64_t)MAX_CHUNKS * grid_mlp * p.sh.w_floats * 4) +
           al((int64_t)MAX_CHUNKS * sms * (COARSE_BYTES / 4) * 4) + al(p.sh.o_x) + 256;
}

static cudaEvent_t g_stage_events[8];
static int g_stage_events_n = 0;

struct SideStreams {
    cudaStream_t enc = nullptr, sc = nullptr;
    cudaEvent_t fork, join_enc, join_sc, enc_done[MAX_CHUNKS], mlp_done[MAX_CHUNKS];
};

static SideStreams &side_streams() {
    static SideStreams ss;
    if (ss.enc == nullptr) {
        cudaStreamCreateWithFlags(&ss.enc, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&ss.sc, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss.join_enc, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss.join_sc, cudaEventDisableTiming);
        for (int c = 0; c < MAX_CHUNKS; ++c) {
            cudaEventCreateWithFlags(&ss.enc_done[c], cudaEventDisableTiming);
            cudaEventCreateWithFlags(&ss.mlp_done[c], cudaEventDisableTiming);
        }
    }
    return ss;
}

int train_tc_launch(const float *coords, const float *targets, int64_t b, int64_t b_global, const float *params,
                    float *grads, const GridTables &tab, int nn, int nh, int relu_out, int loss_kind,
                    double *loss_sum, void *workspace, int64_t ws_bytes, cudaStream_t s) {
    TcPlan p;
    if (!make_plan(p, b, tab, nn, nh, relu_out, loss_kind)) {
        set_error("MLP / grid shape not supported by the tcgen05 path");
        return NVOL_EINVAL;
    }
    NVOL_REQUIRE(ws_bytes >= p.total, "workspace too small for the tcgen05 pipeline");
    uint8_t *ws = reinterpret_cast<uint8_t *>(workspace);
    uint8_t *xt = ws + p.off_x;
    float *dfeat = reinterpret_cast<float *>(ws + p.off_dfeat);
    float *wpart = reinterpret_cast<float *>(ws + p.off_wpart);
    float *cpart = reinterpret_cast<float *>(ws + p.off_cpart);
    uint8_t *wimg = ws + p.off_img;
    int64_t enc = 0;
    for (int l = 0; l < tab.n_levels; ++l) enc = max(enc, tab.offset[l] + tab.entries[l] * tab.n_feat);
    const int64_t woff = (enc + 3) & ~(int64_t)3;
    int st = pack_mlp_image(params + woff, p.sh.nin, p.sh.ninp, nn, nh, p.sh.o_w, p.sh.o_wout, wimg, s, p.sh.o_wlo);
    if (st) return st;
    cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p.sh.smem_bytes);
    const size_t csm = (size_t)p.coarse_floats * 4;
    switch (tab.n_feat) {
        case 1: cudaFuncSetAttribute(scatter_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm); break;
        case 2: cudaFuncSetAttribute(scatter_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm); break;
        case 4: cudaFuncSetAttribute(scatter_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm); break;
        default: cudaFuncSetAttribute(scatter_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm); break;
    }
    const float dscale = exp2f(rintf(log2f((float)b_global)));  // ~B: L1 deltas become +-1 in fp16
    // profiling: one chunk, events at the stage boundaries on the caller's stream
    cudaEvent_t *pev = g_stage_events;
    const bool prof = g_stage_events_n >= 4;
    const int nc = prof ? 1 : p.nchunks;
    if (prof) cudaEventRecord(pev[0], s);
    SideStreams &ss = side_streams();
    cudaStream_t se = nc > 1 ? ss.enc : s, sc = nc > 1 ? ss.sc : s;
    if (nc > 1) {
        cudaEventRecord(ss.fork, s);
        cudaStreamWaitEvent(ss.enc, ss.fork, 0);
        cudaStreamWaitEvent(ss.sc, ss.fork, 0);
    }
    const int64_t tile_bytes = 2 * TILE * p.sh.ninp * 2;
    for (int c = 0; c < nc; ++c) {
        const int64_t t0 = c * p.chunk_tiles;
        const int64_t r0 = t0 * TILE;
        if (r0 >= b) break;
        const int64_t nb = (r0 + p.chunk_tiles * TILE < b ? p.chunk_tiles * TILE : b - r0);
        const unsigned egrid = grid_for(nb * tab.n_levels, 256);
        uint8_t *xtc = xt + t0 * tile_bytes;
        const float *cc = coords + 3 * r0;
        switch (tab.n_feat) {
            case 1: encode_tiles_kernel<1><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc); break;
            case 2: encode_tiles_kernel<2><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc); break;
            case 4: encode_tiles_kernel<4><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc); break;
            default: encode_tiles_kernel<8><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc); break;
        }
        st = check_launch("encode_tiles_kernel");
        if (st) return st;
        if (nc > 1) {
            cudaEventRecord(ss.enc_done[c], se);
            cudaStreamWaitEvent(s, ss.enc_done[c], 0);
        }
        if (prof) cudaEventRecord(pev[1], s);
        const int64_t ct = (nb + TILE - 1) / TILE;
        const int gm = (int)(ct < p.grid_mlp ? ct : p.grid_mlp);
        float *wp = wpart + (int64_t)c * p.grid_mlp * p.sh.w_floats;
        mlp_tc_kernel<<<gm, TC_THREADS, p.sh.smem_bytes, s>>>(xtc, targets + r0, nb, 1.0 / (double)b_global, dscale,
                                                              p.sh, wimg, loss_sum, dfeat + r0, b, wp);
        st = check_launch("mlp_tc_kernel");
        if (st) return st;
        if (gm < p.grid_mlp)  // unused partial slots of a short chunk must sum to zero
            cudaMemsetAsync(wp + (int64_t)gm * p.sh.w_floats, 0, (size_t)(p.grid_mlp - gm) * p.sh.w_floats * 4, s);
        if (nc > 1) {
            cudaEventRecord(ss.mlp_done[c], s);
            cudaStreamWaitEvent(sc, ss.mlp_done[c], 0);
        }
        if (prof) cudaEventRecord(pev[2], s);
        float *cp = cpart + (int64_t)c * p.grid_sc * p.coarse_floats;
        switch (tab.n_feat) {
#define LAUNCH_SC(NFV)                                                                                             \
    case NFV:                                                                                                      \
        scatter_kernel<NFV><<<p.grid_sc, SC_THREADS, csm, sc>>>(cc, dfeat + r0, nb, b, tab, p.n_coarse,            \
                                                                p.coarse_floats, grads, cp);                       \
        break;
            LAUNCH_SC(1)
            LAUNCH_SC(2)
            LAUNCH_SC(4)
            LAUNCH_SC(8)
#undef LAUNCH_SC
        }
        st = check_launch("scatter_kernel");
        if (st) return st;
        if (prof) cudaEventRecord(pev[3], s);
    }
    if (nc > 1) {
        cudaEventRecord(ss.join_enc, ss.enc);
        cudaEventRecord(ss.join_sc, ss.sc);
        cudaStreamWaitEvent(s, ss.join_enc, 0);
        cudaStreamWaitEvent(s, ss.join_sc, 0);
    }
    reduce_partials_kernel<<<grid_for(p.sh.w_floats, 32), 256, 0, s>>>(wpart, nc * p.grid_mlp, p.sh.w_floats,
                                                                       grads + woff);
    if (p.coarse_floats > 0)
        reduce_partials_kernel<<<grid_for(p.coarse_floats, 32), 256, 0, s>>>(cpart, nc * p.grid_sc, p.coarse_floats,
                                                                             grads);
    return check_launch("reduce_partials");
}

}  // namespace nvol

// Profiling hook: with >= 4 events set, nvol_train_fwd_bwd (mode 1) runs as a
// single chunk on the caller's stream and records events[0..3] before encode,
// after encode, after pack+MLP and after scatter.  n = 0 disables.
extern "C" int nvol_set_stage_events(void *const *events, int32_t n) {
    n = n > 8 ? 8 : (n < 0 ? 0 : n);
    for (int i = 0; i < n; ++i) nvol::g_stage_events[i] = reinterpret_cast<cudaEvent_t>(events[i]);
    nvol::g_stage_events_n = n;
    return NVOL_OK;
}

extern "C" int nvol_has_tcgen05(int device) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    return major == 10 && minor == 0;
}
