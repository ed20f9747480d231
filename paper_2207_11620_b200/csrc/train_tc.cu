// Fused tcgen05 training tile pipeline (sm_100a).
//
// One persistent CTA per SM walks 128-sample tiles of the batch.  Per tile:
//   encode (hash-grid gather, _kernels.py:31-79)  -> fp16 feature tile in smem
//   forward MLP (network.py:61-74): per layer one tcgen05.mma chain (M=128
//     samples, N = width, K = 16 per instruction, fp16 operands, fp32
//     accumulator in TMEM) + a ReLU/fp16 epilogue back into smem
//   output layer + L1/L2 loss gradient on CUDA cores (network.py:96-114)
//   backward (network.py:76-93): per layer dW_j += delta^T H_j (M=128 padded
//     rows, K = 128 samples, accumulated in TMEM across all tiles of the CTA)
//     and dX = delta W_j, masked by the stored activations
//   encoder scatter of dL/dfeat (_kernels.py:82-92) with float2 atomics.
// Weight gradients leave TMEM once per CTA as fp32 partials; a second kernel
// sums them in fixed CTA order (deterministic MLP gradients).
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

struct TcShape {
    int m, n, nin, ninp, nn, nh;
    int relu_out, loss_kind;
    // smem byte offsets
    uint32_t o_w[MAX_NH], o_wout, o_x, o_h[MAX_NH + 1], o_d[2], o_dout, o_dx, o_misc, smem_bytes;
    // TMEM columns
    uint32_t t_f, t_g, t_dw[MAX_NH], t_dwout, t_alloc;
    int64_t w_floats;  // MLP weights in the flat buffer
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
    s.o_x = take(2u * TILE * s.ninp);
    s.o_h[0] = s.o_x;
    for (int i = 1; i <= nh; ++i) s.o_h[i] = take(2u * TILE * nn);
    s.o_d[0] = take(2u * TILE * nn);
    s.o_d[1] = take(2u * TILE * nn);
    s.o_dout = take(2048 + 256);
    s.o_dx = take(4u * TILE * s.ninp);
    s.o_misc = take(4u * TILE * 3 + 4u * TILE * 3 + 64);
    take(4096);  // slack: padded-M operand rows read past the last tile (values unused)
    s.smem_bytes = off;
    uint32_t col = 0;
    s.t_f = col;
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

// Columns [c0, c0+nc) of a width-W accumulator handled by thread half h.
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
    // 16 consecutive columns c..c+15 of `row` (two 16-byte core-matrix rows)
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        uint4 pk;
        float a[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) a[e] = relu ? fmaxf(v16[q * 8 + e], 0.0f) : v16[q * 8 + e];
        pk.x = tc::pack_half2(a[0], a[1]);
        pk.y = tc::pack_half2(a[2], a[3]);
        pk.z = tc::pack_half2(a[4], a[5]);
        pk.w = tc::pack_half2(a[6], a[7]);
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

template <int NF>
__global__ void __launch_bounds__(TC_THREADS, 1) train_tc_kernel(
    const float *__restrict__ coords, const float *__restrict__ targets, int64_t b, double inv_bglobal,
    const float *__restrict__ params, float *__restrict__ grads, const GridTables tab, const TcShape sh,
    const float *__restrict__ wflat, double *__restrict__ loss_sum, float *__restrict__ partials) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    const int tid = threadIdx.x;
    const int s = tid & (TILE - 1);     // sample row == TMEM lane
    const int h = tid >> 7;             // thread half
    const int warp = tid >> 5;
    const uint32_t lane_base = (uint32_t)((warp & 3) * 32) << 16;
    const int NN = sh.nn, NINP = sh.ninp, NH = sh.nh, M = sh.m;

    // ---------------------------------------------------------------- setup
    // weights -> fp16 tiles (padded input columns are zero)
    {
        const float *src = wflat;
        for (int i = 0; i < NH; ++i) {
            int win = (i == 0) ? sh.nin : NN, wp = (i == 0) ? NINP : NN;
            uint8_t *dst = smem + sh.o_w[i];
            for (int q = tid; q < NN * wp; q += TC_THREADS) {
                int o = q / wp, j = q % wp;
                float v = j < win ? src[o * win + j] : 0.0f;
                *reinterpret_cast<__half *>(dst + tc::tile_off(o, j, wp)) = __float2half_rn(v);
            }
            src += (int64_t)NN * win;
        }
        float *wout = reinterpret_cast<float *>(smem + sh.o_wout);
        for (int q = tid; q < NN; q += TC_THREADS) wout[q] = src[q];
        // zero the whole feature tile once (padding columns stay zero)
        for (int q = tid; q < TILE * NINP / 8; q += TC_THREADS)
            reinterpret_cast<uint4 *>(smem + sh.o_x)[q] = make_uint4(0, 0, 0, 0);
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

    float *s_coords = reinterpret_cast<float *>(smem + sh.o_misc);
    float *s_part = s_coords + TILE * 3;
    float *s_delta = s_part + TILE;
    float *s_dx = reinterpret_cast<float *>(smem + sh.o_dx);
    const float *s_wout = reinterpret_cast<const float *>(smem + sh.o_wout);

    const uint32_t idesc_fwd = tc::make_idesc(128, NN, 0, 0);
    const int mh = (M + 1) / 2;  // levels per thread half
    const int l_lo = h * mh, l_hi = min(M, (h + 1) * mh);
    const int64_t ntiles = (b + TILE - 1) / TILE;
    bool first_tile = true;

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t row = tile * TILE + s;
        const bool valid = row < b;
        float x = 0.f, y = 0.f, z = 0.f, tgt = 0.f;
        if (valid) {
            x = coords[3 * row];
            y = coords[3 * row + 1];
            z = coords[3 * row + 2];
            tgt = targets[row];
        }
        // ------------------------------------------------------------ encode (bit-exact fp32, stored fp16)
        {
            uint8_t *sx = smem + sh.o_x;
            for (int l = l_lo; l < l_hi; ++l) {
                const int32_t res = tab.res[l];
                Cell<float> c = cell_of<float>(x, y, z, res);
                float acc[NF];
#pragma unroll
                for (int f = 0; f < NF; ++f) acc[f] = 0.0f;
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    int64_t slot = vertex_slot(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), res,
                                               tab.entries[l], tab.dense[l] != 0);
                    float w = corner_weight<float>(c, k);
                    const float *p = params + tab.offset[l] + slot * NF;
                    if constexpr (NF == 2) {
                        float2 v = __ldg(reinterpret_cast<const float2 *>(p));
                        acc[0] = xadd(acc[0], xmul(w, v.x));
                        acc[1] = xadd(acc[1], xmul(w, v.y));
                    } else {
#pragma unroll
                        for (int f = 0; f < NF; ++f) acc[f] = xadd(acc[f], xmul(w, __ldg(p + f)));
                    }
                }
#pragma unroll
                for (int f = 0; f < NF; ++f)
                    *reinterpret_cast<__half *>(sx + tc::tile_off(s, l * NF + f, NINP)) =
                        __float2half_rn(valid ? acc[f] : 0.0f);
            }
        }
        tc::fence_proxy_async();
        __syncthreads();

        // ------------------------------------------------------------ forward
        float outp = 0.0f;
        for (int i = 0; i < NH; ++i) {
            const int win = (i == 0) ? NINP : NN;
            if (tid == 0) {
                tc::fence_after();
                uint32_t a0 = tc::smem_u32(smem + sh.o_h[i]);
                uint32_t b0 = tc::smem_u32(smem + sh.o_w[i]);
                for (int k = 0; k < win / 16; ++k) {
                    uint64_t ad = tc::make_desc(a0 + k * 256, 128, (win / 8) * 128);
                    uint64_t bd = tc::make_desc(b0 + k * 256, 128, (win / 8) * 128);
                    tc::mma_f16(tmem + sh.t_f, ad, bd, idesc_fwd, k > 0);
                }
                tc::mma_commit(&mbar);
            }
            tc::mbar_wait(&mbar, phase);
            phase ^= 1;
            tc::fence_after();
            int c0, nc;
            half_cols(NN, h, c0, nc);
            uint8_t *dst = smem + sh.o_h[i + 1];
            for (int c = c0; c < c0 + nc; c += 16) {
                float v[16];
                tc::tmem_ld16(tmem + lane_base + sh.t_f + c, v);
                tc::tmem_wait_ld();
                store_row_f16(dst, s, c, NN, v, true);
                if (i == NH - 1) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) outp += s_wout[c + e] * fmaxf(v[e], 0.0f);
                }
            }
            tc::fence_before();
            tc::fence_proxy_async();
            __syncthreads();
        }
        // ------------------------------------------------------------ output layer + loss
        if (h == 1) s_part[s] = outp;
        __syncthreads();
        if (h == 0) {
            float o = outp + s_part[s];
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
            // delta_out as the MN-major A operand of dW_out: element (m=0, k=s)
            *reinterpret_cast<__half *>(smem + sh.o_dout + (s >> 3) * 128 + (s & 7) * 16) = __float2half_rn(gf);
            for (int o2 = 16; o2 > 0; o2 >>= 1) sl += __shfl_xor_sync(0xffffffffu, sl, o2);
            if ((tid & 31) == 0) atomicAdd(loss_sum, sl);
        }
        __syncthreads();
        // delta_NH = g * w_out * 1[h_NH > 0]
        {
            int c0, nc;
            half_cols(NN, h, c0, nc);
            const float g = s_delta[s];
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

        // ------------------------------------------------------------ backward
        int cur = 0;
        for (int j = NH - 1; j >= 0; --j) {
            const int win = (j == 0) ? NINP : NN;
            if (tid == 0) {
                tc::fence_after();
                const uint32_t dA = tc::smem_u32(smem + sh.o_d[cur]);
                if (j == NH - 1) {
                    // dW_out += delta_out^T H_NH  (row 0 of an M=128 accumulator)
                    const uint32_t a0 = tc::smem_u32(smem + sh.o_dout);
                    const uint32_t b0 = tc::smem_u32(smem + sh.o_h[NH]);
                    const uint32_t id = tc::make_idesc(128, NN, 1, 1);
                    for (int k = 0; k < TILE / 16; ++k) {
                        uint64_t ad = tc::make_desc(a0 + k * 256, 128, 16);
                        uint64_t bd = tc::make_desc(b0 + k * 2 * (NN / 8) * 128, (NN / 8) * 128, 128);
                        tc::mma_f16(tmem + sh.t_dwout, ad, bd, id, (first_tile && k == 0) ? 0 : 1);
                    }
                }
                // dW_j += delta^T H_j   (A: delta MN-major, B: H_j MN-major)
                {
                    const uint32_t b0 = tc::smem_u32(smem + sh.o_h[j]);
                    const uint32_t id = tc::make_idesc(128, win, 1, 1);
                    for (int k = 0; k < TILE / 16; ++k) {
                        uint64_t ad = tc::make_desc(dA + k * 2 * (NN / 8) * 128, (NN / 8) * 128, 128);
                        uint64_t bd = tc::make_desc(b0 + k * 2 * (win / 8) * 128, (win / 8) * 128, 128);
                        tc::mma_f16(tmem + sh.t_dw[j], ad, bd, id, (first_tile && k == 0) ? 0 : 1);
                    }
                }
                // dX = delta W_j   (A: delta K-major, B: W_j MN-major)
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
                    for (int e = 0; e < 16; ++e) s_dx[s * NINP + c + e] = v[e];
                }
            }
            tc::fence_before();
            tc::fence_proxy_async();
            __syncthreads();
            cur ^= 1;
        }
        // ------------------------------------------------------------ encoder scatter
        if (valid) {
            for (int l = l_lo; l < l_hi; ++l) {
                const int32_t res = tab.res[l];
                Cell<float> c = cell_of<float>(x, y, z, res);
                float dv[NF];
#pragma unroll
                for (int f = 0; f < NF; ++f) dv[f] = s_dx[s * NINP + l * NF + f];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    int64_t slot = vertex_slot(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), res,
                                               tab.entries[l], tab.dense[l] != 0);
                    float w = corner_weight<float>(c, k);
                    float *g = grads + tab.offset[l] + slot * NF;
                    if constexpr (NF == 2) {
                        atomicAdd(reinterpret_cast<float2 *>(g), make_float2(w * dv[0], w * dv[1]));
                    } else if constexpr (NF == 4 || NF == 8) {
#pragma unroll
                        for (int q = 0; q < NF / 4; ++q)
                            atomicAdd(reinterpret_cast<float4 *>(g) + q,
                                      make_float4(w * dv[4 * q], w * dv[4 * q + 1], w * dv[4 * q + 2], w * dv[4 * q + 3]));
                    } else {
                        atomicAdd(g, w * dv[0]);
                    }
                }
            }
        }
        first_tile = false;
    }

    // ---------------------------------------------------------------- flush dW partials
    if (!first_tile) {
        float *dst = partials + (int64_t)blockIdx.x * sh.w_floats;
        const int o = (warp & 3) * 32 + (tid & 31);  // accumulator row == output neuron
        int64_t base = 0;
        for (int j = 0; j <= NH; ++j) {
            const int win = (j == 0) ? sh.nin : NN;     // unpadded columns
            const int wacc = (j == 0) ? NINP : NN;
            const int rows = (j == NH) ? 1 : NN;
            const uint32_t tcol = (j == NH) ? sh.t_dwout : sh.t_dw[j];
            int c0, nc;
            half_cols(wacc, h, c0, nc);
            for (int c = c0; c < c0 + nc; c += 16) {
                float v[16];
                tc::tmem_ld16(tmem + lane_base + tcol + c, v);
                tc::tmem_wait_ld();
                if (o < rows) {
#pragma unroll
                    for (int e = 0; e < 16; ++e)
                        if (c + e < win) dst[base + (int64_t)o * win + c + e] = v[e];
                }
            }
            base += (int64_t)rows * win;
        }
    } else {
        float *dst = partials + (int64_t)blockIdx.x * sh.w_floats;
        for (int64_t q = tid; q < sh.w_floats; q += TC_THREADS) dst[q] = 0.0f;
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, sh.t_alloc);
}

// grads_w[i] += sum over CTAs (fixed order) of partials[c][i]
__global__ void reduce_partials_kernel(const float *__restrict__ partials, int nparts, int64_t n,
                                       float *__restrict__ gw) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float acc = 0.0f;
    for (int c = 0; c < nparts; ++c) acc += partials[(int64_t)c * n + i];
    gw[i] += acc;
}

static int g_sms = 0;

int64_t train_tc_workspace(int64_t b, int m, int n, int nn, int nh) {
    TcShape sh;
    if (!build_shape(sh, m, n, nn, nh, 1, 0)) return 0;
    if (g_sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return (int64_t)g_sms * sh.w_floats * 4 + 256;
}

int train_tc_launch(const float *coords, const float *targets, int64_t b, int64_t b_global, const float *params,
                    float *grads, const GridTables &tab, int nn, int nh, int relu_out, int loss_kind,
                    double *loss_sum, void *workspace, int64_t ws_bytes, cudaStream_t s) {
    TcShape sh;
    if (!build_shape(sh, tab.n_levels, tab.n_feat, nn, nh, relu_out, loss_kind)) {
        set_error("MLP shape not supported by the tcgen05 path");
        return NVOL_EINVAL;
    }
    int64_t enc = 0;
    for (int l = 0; l < tab.n_levels; ++l) enc = max(enc, tab.offset[l] + tab.entries[l] * tab.n_feat);
    int64_t woff = (enc + 3) & ~(int64_t)3;
    int64_t ntiles = (b + TILE - 1) / TILE;
    int64_t sms = g_sms > 0 ? g_sms : 148;
    int grid = (int)(ntiles < sms ? ntiles : sms);
    float *partials = reinterpret_cast<float *>(workspace);
    NVOL_REQUIRE(ws_bytes >= (int64_t)grid * sh.w_floats * 4, "workspace too small for tcgen05 partials");
    const double inv_bg = 1.0 / (double)b_global;
    switch (tab.n_feat) {
#define LAUNCH_TC(NFV)                                                                                        \
    case NFV:                                                                                                 \
        cudaFuncSetAttribute(train_tc_kernel<NFV>, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem_bytes); \
        train_tc_kernel<NFV><<<grid, TC_THREADS, sh.smem_bytes, s>>>(coords, targets, b, inv_bg, params, grads, tab, \
                                                                    sh, params + woff, loss_sum, partials);    \
        break;
        LAUNCH_TC(1)
        LAUNCH_TC(2)
        LAUNCH_TC(4)
        LAUNCH_TC(8)
#undef LAUNCH_TC
    }
    int st = check_launch("train_tc_kernel");
    if (st) return st;
    reduce_partials_kernel<<<grid_for(sh.w_floats, 256), 256, 0, s>>>(partials, grid, sh.w_floats, grads + woff);
    return check_launch("reduce_partials");
}

int nvol_decode_tc(const float *, const GridTables &, const float *, const int32_t *, int32_t, int32_t, int64_t,
                   int64_t, int64_t, int64_t, int64_t, double, double, float *, cudaStream_t) {
    set_error("tcgen05 decode path not built");
    return NVOL_EINVAL;
}

}  // namespace nvol

extern "C" int nvol_has_tcgen05(int device) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    return major == 10 && minor == 0;
}
