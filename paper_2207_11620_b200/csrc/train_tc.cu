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
//     as fp32; dW leaves TMEM once per CTA as fp32 vector REDs.
//  3. scatter_kernel — encoder backward (_kernels.py:82-92): corners
//     recomputed from the coordinates; the small dense coarse levels
//     (contended by every sample) accumulate in shared memory and leave as
//     one float4 RED per entry quad per CTA, the fine levels scatter with
//     float2/float4 REDs.  (Float atomics make the fast path's gradient sums
//     order-dependent; encoding.set_deterministic selects the sort-based
//     bit-exact scatter of the API path.)
//
// Accuracy contract (north star): fp16 operands / fp32 accumulation, MLP
// outputs and gradients within 1e-2 relative of the fp32 reference.
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "tc.cuh"

namespace nvol {

constexpr int TILE = 128;
constexpr int MAX_NH = 8;
// MLP kernel: two 128-sample tiles in flight per CTA ("slots"), each with 8
// epilogue warps (2 per TMEM lane quarter, one column half each), plus one
// MMA-issuer warp that round-robins the slots' layer phases.
constexpr int PP_EPI_WARPS = 16;
constexpr int PP_THREADS = (PP_EPI_WARPS + 1) * 32;
#ifndef NVOL_SC_THREADS
#define NVOL_SC_THREADS 1024
#endif
constexpr int SC_THREADS = NVOL_SC_THREADS;
constexpr int SC_LG = 4;  // levels per scatter item
constexpr uint32_t COARSE_BYTES = 48 * 1024;

struct TcShape {
    int m, n, nin, ninp, nn, nh, wbuf;
    int relu_out, loss_kind;
    // weights: fp16 hi / lo core-matrix tiles + fp32 output row
    uint32_t o_w[MAX_NH], o_wout, o_wlo[MAX_NH];
    // per slot t: o_d[t] (X hi during the forward, then the fp16 delta tile),
    // o_hlo[t] (X lo, then activation lo parts, h_NH, then the X hi reload),
    // o_h[t][i] (hidden activations h_1..h_{nh-1}, fp16 hi)
    uint32_t o_d[2], o_hlo[2], o_h[2][MAX_NH], o_dout[2], o_part, smem_bytes, xhalf;
    // TMEM: per slot [forward acc | forward lo acc] (backward dX aliases the
    // first), then the dW_0..dW_{nh-1} accumulators shared by both slots
    uint32_t t_acc[2], t_dw[MAX_NH], t_dwout, t_alloc;
    int64_t w_floats;
};

static int build_shape(TcShape &s, int m, int n, int nn, int nh, int relu_out, int loss_kind) {
    s.m = m;
    s.n = n;
    s.nin = m * n;
    s.ninp = (s.nin + 15) & ~15;
    s.nn = nn;
    s.nh = nh;
    s.wbuf = max(nn, s.ninp);
    s.relu_out = relu_out;
    s.loss_kind = loss_kind;
    if (nh < 1 || nh > MAX_NH) return 0;
    if (!(nn == 16 || nn == 32 || nn == 64)) return 0;
    if (s.ninp > 2 * nn || s.ninp > 128) return 0;
    uint32_t off = 0;
    auto take = [&](uint32_t bytes) {
        uint32_t r = off;
        off += (bytes + 127) & ~127u;
        return r;
    };
    // each layer's lo tile directly follows its hi tile: [W_hi; W_lo] is one N = 2*nn
    // B operand (the forward's hi*W_hi and hi*W_lo products in one MMA)
    for (int i = 0; i < nh; ++i) {
        s.o_w[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
        s.o_wlo[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
    }
    s.o_wout = take(4u * nn);
    for (int t = 0; t < 2; ++t) {
        s.o_d[t] = take(2u * TILE * s.wbuf);
        s.o_hlo[t] = take(2u * TILE * s.wbuf);
        s.o_h[t][0] = 0;
        for (int i = 1; i < nh; ++i) s.o_h[t][i] = take(2u * TILE * nn);
    }
    // per slot: the output-layer delta as an N = 8 K-major B operand (column 0 = delta_out)
    s.o_dout[0] = take(2u * 8 * TILE);
    s.o_dout[1] = take(2u * 8 * TILE);
    s.o_part = take(4u * 2 * 2 * TILE);
    // no slack needed: the M = 128 MN-major A operands (delta^T for dW, h_NH^T for dW_out) read up to
    // ~2 KB past an nn-wide tile (rows >= nn, values unused), which lands in the next slot buffer
    s.smem_bytes = off;
    s.xhalf = 2u * TILE * s.ninp;
    uint32_t col = 0;
    s.t_acc[0] = col;
    col += 2 * nn;
    s.t_acc[1] = col;
    col += 2 * nn;
    for (int i = 0; i < nh; ++i) {
        s.t_dw[i] = col;
        col += (i == 0) ? s.ninp : nn;
    }
    s.t_dwout = col;  // dW_out^T = h_NH^T delta_out: lanes = hidden units, column 0
    col += 8;
    if (col > 512) return 0;
    uint32_t a = 32;
    while (a < col) a <<= 1;
    s.t_alloc = a;
    s.w_floats = (int64_t)nn * s.nin + (int64_t)(nh - 1) * nn * nn + nn;
    // the prologue stages the fp32 weights over the slot buffers
    if ((int64_t)s.o_part - (int64_t)s.o_d[0] < s.w_floats * 4) return 0;
    return s.smem_bytes <= 227 * 1024 - 1024;
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
// Table reads: the standalone kernel may use the read-only path; the fused
// Adam + encode kernel reads parameters other CTAs of the same launch just
// wrote, so it loads through L2 (ld.global.cg, coherent).
template <bool COHERENT, typename V>
__device__ __forceinline__ V tab_ld(const V *p) {
    if constexpr (COHERENT)
        return __ldcg(p);
    else
        return __ldg(p);
}

// hashed-level gathers do not allocate in L1 (no reuse there), which keeps L1 for the dense
// coarse levels every warp of a level shares (measured 29.5 -> 28.8 us per encode)
__device__ __forceinline__ float4 ld_na4(const float4 *p) {
    float4 v;
    asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ float2 ld_na2(const float2 *p) {
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0,%1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
}

// One (sample i, level l) item of the encoder forward (_kernels.py:31-79), bit-exact
// fp32, split into fp16 hi + lo and stored straight into the UMMA tile layout.
template <int NF, bool COHERENT>
__device__ __forceinline__ void encode_item(const float *__restrict__ coords, const float *__restrict__ params,
                                            const GridTables &tab, int ninp, uint8_t *__restrict__ xtiles, int l,
                                            int64_t i, float lo_scale, float *__restrict__ dbg_feat = nullptr) {
    const int m = tab.n_levels;
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
        // x-adjacent corners (k, k+1) whose slots differ only in bit 0 share one
        // aligned 16-byte entry pair: fetch it with a single float4 load; the pair
        // {lo, lo+1} is 16-byte aligned iff (address of entry 0) / 8 + lo is even
        float2 v[8];
        const uint32_t par = (uint32_t)((reinterpret_cast<uintptr_t>(tb) >> 3) & 1u);
#pragma unroll
        for (int k = 0; k < 8; k += 2) {
            const uint32_t lo = min(sl[k], sl[k + 1]);
            if (max(sl[k], sl[k + 1]) == lo + 1 && ((lo + par) & 1u) == 0u) {
                const float4 q = (!COHERENT && !dense) ? ld_na4(reinterpret_cast<const float4 *>(tb + 2 * (size_t)lo))
                                                       : tab_ld<COHERENT>(reinterpret_cast<const float4 *>(tb + 2 * (size_t)lo));
                const bool lo_first = sl[k] == lo;
                v[k] = lo_first ? make_float2(q.x, q.y) : make_float2(q.z, q.w);
                v[k + 1] = lo_first ? make_float2(q.z, q.w) : make_float2(q.x, q.y);
            } else {
                if (!COHERENT && !dense) {
                    v[k] = ld_na2(reinterpret_cast<const float2 *>(tb) + sl[k]);
                    v[k + 1] = ld_na2(reinterpret_cast<const float2 *>(tb) + sl[k + 1]);
                } else {
                    v[k] = tab_ld<COHERENT>(reinterpret_cast<const float2 *>(tb) + sl[k]);
                    v[k + 1] = tab_ld<COHERENT>(reinterpret_cast<const float2 *>(tb) + sl[k + 1]);
                }
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
            for (int f = 0; f < NF; ++f) acc[f] = xadd(acc[f], xmul(w, tab_ld<COHERENT>(tb + (size_t)sl[k] * NF + f)));
        }
    }
    if (dbg_feat) {  // parity hook (nvol_train_tc_debug): the fp32 features, sample-major [b][m*NF]
#pragma unroll
        for (int f = 0; f < NF; ++f) dbg_feat[i * (m * NF) + l * NF + f] = acc[f];
    }
    const int64_t tile = i >> 7;
    const int s = (int)(i & 127);
    // per tile: fp16 hi tile followed by the fp16 lo tile (split-fp16 forward)
    uint8_t *base = xtiles + tile * (int64_t)(2 * TILE * ninp * 2);
    uint8_t *base_lo = base + TILE * ninp * 2;
    __half hv[NF], lv[NF];
#pragma unroll
    for (int f = 0; f < NF; ++f) {  // lo_scale: kLoScale (mlp_tc_kernel) or 1 (mlp_tc4_kernel, folded lo products)
        const float a = acc[f] * tc::kActScale;
        hv[f] = __float2half_rn(a);
        lv[f] = __float2half_rn((a - __half2float(hv[f])) * lo_scale);
    }
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

template <int NF>
__global__ void __launch_bounds__(256) encode_tiles_kernel(const float *__restrict__ coords, int64_t b,
                                                           const float *__restrict__ params, const GridTables tab,
                                                           int ninp, uint8_t *__restrict__ xtiles,
                                                           float lo_scale, float *__restrict__ dbg_feat,
                                                           const int64_t *__restrict__ nan_state) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b * tab.n_levels || nan_halted(nan_state)) return;
    // level-major: a warp covers 32 consecutive samples of one level (uniform
    // level constants, coalesced coordinates, L1 reuse on coarse levels)
    const int l = (int)(t / b);
    encode_item<NF, false>(coords, params, tab, ninp, xtiles, l, t - (int64_t)l * b, lo_scale, dbg_feat);
}

// ---------------------------------------------------------------------------- Adam(k) + encode(k+1)
// The step tail fused with the next step's encoder forward.  Adam streams the
// flat buffers in table order (network.py:160-183); the encoder forward of the
// NEXT batch (_kernels.py:31-79, sampled ahead on the side stream) of level l
// only needs level l's updated table, so it can run as soon as the Adam sweep
// has passed that level instead of after a kernel boundary.  CTAs take a role
// in arrival order: the first n_adam to start sweep the flat buffers in
// grid-stride chunks (chunk c after chunk c - n_adam, so the sweep advances
// through the levels in order) and count finished chunks per level; the rest
// run the encoder items level-major, each waiting (acquire) until its level's
// chunk count is complete.  Arrival-order roles make the wait deadlock-free:
// every chunk an encoder CTA waits on belongs to a CTA that is already running
// and never waits.  The last CTA out records the loss, advances the step
// counter and re-arms the work words.
struct AdamArgs {
    float *p, *g, *m, *v;
    int64_t n;
    const float *sched;
    int64_t sched_len;
    int64_t *counter;
    float b1, omb1, b2, omb2, eps, l2;
    int64_t *nan_state;
    double *loss_acc, *losses;
    int64_t t0, cap;
    double inv_b;
};

// CTA = 4 Adam warps + 12 encoder warps (warp-specialised, 3 CTAs per SM).
// Adam warps dequeue warp chunks (32 lanes x 8 float4 of each of p, g, m, v)
// from an atomic counter, so the sweep runs in table order; each lane streams
// its float4s through a 3-deep cp.async ring in shared memory (the in-flight
// bytes live in shared memory, not registers, so 4 warps per CTA keep enough
// DRAM traffic in flight) and publishes each finished chunk with a fence and
// one add per level the chunk overlaps.  Encoder warps take (level, 32
// samples) items level-major and poll (acquire) their level's chunk count
// before gathering.  Dynamic dequeue keeps this deadlock-free whatever the
// residency: every chunk is claimed by a running Adam warp, which never waits.
constexpr int AE_ADAM_WARPS = 4, AE_ENC_WARPS = 12;
constexpr int AE_THREADS = 32 * (AE_ADAM_WARPS + AE_ENC_WARPS);
#ifndef NVOL_AE_CHUNK_U
#define NVOL_AE_CHUNK_U 32
#endif
constexpr int AE_CHUNK_U = NVOL_AE_CHUNK_U;       // float4 per lane per chunk
constexpr int AE_WARP_F4 = 32 * AE_CHUNK_U;       // 4,096 floats per array per chunk
constexpr int AE_D = 3;                           // cp.async ring depth

// Per-level range of warp chunks covering the level's table (host-computed).
struct LevelChunks {
    int32_t lo[NVOL_MAX_LEVELS], hi[NVOL_MAX_LEVELS];
};

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
                 "l"(gmem)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// one parameter under the NaN contract (common.cuh): only q < lim, a NaN gradient stays unapplied
__device__ __forceinline__ void adam_lim(const AdamArgs &a, float &P, float &G, float &M, float &V, int64_t q,
                                         int64_t lim, float lr, float c1, float c2, int64_t &bad) {
    if (q >= lim) return;
    if (isnan(G)) {
        bad = min(bad, q);
        return;
    }
    adam_one<float>(P, G, M, V, lr, a.b1, a.omb1, a.b2, a.omb2, c1, c2, a.eps, a.l2);
}

__device__ __forceinline__ void adam_scalar(const AdamArgs &a, int64_t q, float lr, float c1, float c2, int64_t lim,
                                            int64_t &bad) {
    float P = a.p[q], G = a.g[q], M = a.m[q], V = a.v[q];
    adam_lim(a, P, G, M, V, q, lim, lr, c1, c2, bad);
    a.p[q] = P;
    a.g[q] = G;
    a.m[q] = M;
    a.v[q] = V;
}

// work words: [0] chunk queue, [1] exit ticket, [2 + l] finished warp chunks of level l
template <int NF>
__global__ void __launch_bounds__(AE_THREADS, 3) adam_encode_kernel(AdamArgs a, int64_t head, int64_t n4,
                                                                    int64_t nch, const LevelChunks lc,
                                                                    const float *__restrict__ coords, int64_t b,
                                                                    const GridTables tab, int ninp,
                                                                    uint8_t *__restrict__ xtiles,
                                                                    uint32_t *__restrict__ work, float lo_scale) {
    __shared__ float4 ring[AE_D][4][AE_ADAM_WARPS * 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (nan_halted(a.nan_state)) return;
    const int64_t tc = *a.counter;
    const int64_t lim = nan_limit(a.nan_state);
    const int m = tab.n_levels;
    if (warp < AE_ADAM_WARPS) {
        const int64_t t = tc >= a.sched_len ? a.sched_len - 1 : tc;
        const float lr = a.sched[3 * t], c1 = a.sched[3 * t + 1], c2 = a.sched[3 * t + 2];
        float4 *p4 = reinterpret_cast<float4 *>(a.p + head), *g4 = reinterpret_cast<float4 *>(a.g + head);
        float4 *m4 = reinterpret_cast<float4 *>(a.m + head), *v4 = reinterpret_cast<float4 *>(a.v + head);
        const uint64_t keep = l2_evict_last();
        const int64_t ntail = a.n - head - 4 * n4;
        int64_t bad = kNanNone;
        auto dequeue = [&]() -> int64_t {
            uint32_t c = 0;
            if (lane == 0) c = atomicAdd(work, 1u);
            return (int64_t)__shfl_sync(0xffffffffu, c, 0);
        };
        // prefetch cursor (pc, pu) runs AE_D slots ahead of the compute cursor (cc, cu)
        int64_t cc = dequeue(), pc = cc, nxt = -1;
        int pu = 0, cu = 0;
        auto issue = [&](int slot) {
            if (pc < nch) {
                const int64_t j = pc * AE_WARP_F4 + pu * 32 + lane;
                if (j < n4) {
                    cp_async16(&ring[slot][0][tid], p4 + j);
                    cp_async16(&ring[slot][1][tid], g4 + j);
                    cp_async16(&ring[slot][2][tid], m4 + j);
                    cp_async16(&ring[slot][3][tid], v4 + j);
                }
                if (++pu == AE_CHUNK_U) {
                    pu = 0;
                    pc = nxt = dequeue();
                }
            }
            cp_async_commit();
        };
#pragma unroll
        for (int d = 0; d < AE_D; ++d) issue(d);
        int slot = 0;
        while (cc < nch) {
            cp_async_wait<AE_D - 1>();
            const int64_t j = cc * AE_WARP_F4 + cu * 32 + lane;
            if (j < n4) {
                float4 P = ring[slot][0][tid], G = ring[slot][1][tid], M = ring[slot][2][tid], V = ring[slot][3][tid];
                const int64_t q = head + 4 * j;
                if (q + 3 < lim && !(isnan(G.x) | isnan(G.y) | isnan(G.z) | isnan(G.w))) {
                    adam_one<float>(P.x, G.x, M.x, V.x, lr, a.b1, a.omb1, a.b2, a.omb2, c1, c2, a.eps, a.l2);
                    adam_one<float>(P.y, G.y, M.y, V.y, lr, a.b1, a.omb1, a.b2, a.omb2, c1, c2, a.eps, a.l2);
                    adam_one<float>(P.z, G.z, M.z, V.z, lr, a.b1, a.omb1, a.b2, a.omb2, c1, c2, a.eps, a.l2);
                    adam_one<float>(P.w, G.w, M.w, V.w, lr, a.b1, a.omb1, a.b2, a.omb2, c1, c2, a.eps, a.l2);
                } else {
                    adam_lim(a, P.x, G.x, M.x, V.x, q, lim, lr, c1, c2, bad);
                    adam_lim(a, P.y, G.y, M.y, V.y, q + 1, lim, lr, c1, c2, bad);
                    adam_lim(a, P.z, G.z, M.z, V.z, q + 2, lim, lr, c1, c2, bad);
                    adam_lim(a, P.w, G.w, M.w, V.w, q + 3, lim, lr, c1, c2, bad);
                }
                p4[j] = P;                    // default policy: the encoder warps gather it next
                st4_hint(g4 + j, G, keep);    // the zeroed gradient stays in L2 for the next scatter
                __stcs(m4 + j, M);
                __stcs(v4 + j, V);
            }
            issue(slot);  // this lane's slot is consumed: refill it AE_D slots ahead
            slot = slot + 1 == AE_D ? 0 : slot + 1;
            if (++cu == AE_CHUNK_U) {
                // chunk done: scalar head (chunk 0) / tail (last chunk), then publish
                if (cc == 0 && lane < head) adam_scalar(a, lane, lr, c1, c2, lim, bad);
                if (cc == nch - 1 && lane < ntail) adam_scalar(a, head + 4 * n4 + lane, lr, c1, c2, lim, bad);
                __threadfence();
                __syncwarp();
                if (lane < m && lc.lo[lane] <= cc && cc <= lc.hi[lane]) atomicAdd(work + 2 + lane, 1u);
                cu = 0;
                cc = nxt;
            }
        }
        cp_async_wait<0>();
        if (bad != kNanNone) nan_mark(a.nan_state, bad);
    } else {
        const int64_t nblk = (b + 31) >> 5;
        const int64_t n_enc = (int64_t)gridDim.x * AE_ENC_WARPS;
        int ready = -1;
        for (int64_t it = (int64_t)blockIdx.x * AE_ENC_WARPS + (warp - AE_ADAM_WARPS); it < nblk * m; it += n_enc) {
            const int l = (int)(it / nblk);
            const int64_t i = (it - (int64_t)l * nblk) * 32 + lane;
            if (l > ready) {
                // lane 0 polls (acquire) with backoff; __syncwarp orders the lanes' gathers after it
                if (lane == 0) {
                    const uint32_t need = (uint32_t)(lc.hi[l] - lc.lo[l] + 1);
                    uint32_t ns = 256;
                    for (;;) {
                        uint32_t got;
                        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(got) : "l"(work + 2 + l) : "memory");
                        if (got >= need) break;
                        __nanosleep(ns);
                        ns = ns < 2048 ? 2 * ns : ns;
                    }
                }
                __syncwarp();
                ready = l;
            }
            if (i < b) encode_item<NF, true>(coords, a.p, tab, ninp, xtiles, l, i, lo_scale);
        }
    }
    // exit ticket: the last CTA records the loss, advances the counter, re-arms the work words
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        if (atomicAdd(work + 1, 1u) == gridDim.x - 1) {
            __threadfence();
            if (nan_limit(a.nan_state) != kNanNone) {
                a.nan_state[1] = 1;  // halt (NaN contract): no loss record, t does not advance
            } else {
                const int64_t k = tc - a.t0;
                if (a.losses && k >= 0 && k < a.cap)
                    a.losses[k] = *reinterpret_cast<volatile double *>(a.loss_acc) * a.inv_b;
                if (a.loss_acc) *a.loss_acc = 0.0;
                *a.counter = tc + 1;
            }
            for (int l = 0; l < m; ++l) work[2 + l] = 0u;
            work[0] = 0u;
            work[1] = 0u;
        }
    }
}

// ============================================================================ 2. MLP
// Columns [c0, c0 + nc) of a w-wide accumulator handled by column group h of
// ng (16-column TMEM loads; groups past the width get nc = 0).
__device__ __forceinline__ void group_cols(int w, int h, int ng, int &c0, int &nc) {
    const int chunks = w >> 4, per = (chunks + ng - 1) / ng;
    const int k0 = h * per, k1 = min(chunks, k0 + per);
    c0 = k0 * 16;
    nc = k1 > k0 ? (k1 - k0) * 16 : 0;
}

// ReLU with numpy's NaN semantics (np.maximum(x, 0) propagates NaN; fmaxf would swallow it),
// so a NaN parameter reaches the gradients as in the reference and trips the NaN contract
__device__ __forceinline__ float relu_nan(float x) { return (x > 0.0f || x != x) ? x : 0.0f; }

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc::smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void named_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
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

#ifdef NVOL_TIMELINE
__device__ unsigned long long g_tl[4096];
__device__ __forceinline__ unsigned long long gtime() {
    unsigned long long t;
#ifdef NVOL_TIMELINE_CLOCK  // SM cycle counter (cheaper to read; stamps of CTA 0 share one SM)
    asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));
#else
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
#endif
    return t;
}
#define TL(slot, val)                                              \
    do {                                                           \
        if (blockIdx.x == 0) g_tl[(slot) & 4095] = (val);          \
    } while (0)
#else
#define TL(slot, val) \
    do {              \
    } while (0)
#endif

// Forward (network.py:61-74), L1/L2 loss gradient (network.py:96-114) and
// backward (network.py:76-93) of 128-sample tiles, two tiles in flight per
// CTA so one slot's epilogue overlaps the other slot's tensor-core phase.
__global__ void __launch_bounds__(PP_THREADS, 1) mlp_tc_kernel(
    const uint8_t *__restrict__ xtiles, const float *__restrict__ targets, int64_t b, double inv_bglobal, float dscale,
    const TcShape sh, const float *__restrict__ wflat, double *__restrict__ loss_sum, float *__restrict__ dfeat,
    int64_t stride, float *__restrict__ dw_grads, float *__restrict__ dbg_pred, int64_t *__restrict__ nan_state,
    int64_t woff) {
    if (nan_halted(nan_state)) return;  // NaN contract: a halted pipeline does no more work
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar_x[2], bar_xr[2], bar_acc[2], bar_op[2], bar_w, bar_dwo;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double s_loss[PP_EPI_WARPS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NN = sh.nn, NINP = sh.ninp, NH = sh.nh, NIN = sh.nin;
    const int64_t ntiles = (b + TILE - 1) / TILE;
    const int64_t xtile_bytes = 2 * (int64_t)sh.xhalf;
    int64_t nan_at = kNanNone;  // NaN contract: start of the first parameter group this thread saw a NaN gradient in

    // ---- prologue: fp32 weights staged by one bulk copy, packed to fp16 hi/lo tiles
    float *stage = reinterpret_cast<float *>(smem + sh.o_d[0]);
    if (tid == 0) {
        for (int t = 0; t < 2; ++t) {
            tc::mbar_init(&bar_x[t], 1);
            tc::mbar_init(&bar_xr[t], 1);
            tc::mbar_init(&bar_acc[t], 1);
            tc::mbar_init(&bar_op[t], 8);  // one arrive per epilogue warp of the slot
        }
        tc::mbar_init(&bar_w, 1);
        tc::mbar_init(&bar_dwo, 1);
        tc::fence_mbar_init();
        const uint32_t wbytes = (uint32_t)sh.w_floats * 4u;  // multiple of 16 (nn in {16, 32, 64})
        tc::mbar_arrive_expect_tx(&bar_w, wbytes);
        tc::bulk_g2s(stage, wflat, wbytes, &bar_w);
    }
    __syncthreads();
    tc::mbar_wait(&bar_w, 0);
    {
        // one 16-byte core-matrix row (8 consecutive inputs of one output) per item
        const float *src = stage;
        for (int i = 0; i < NH; ++i) {
            const int win = i == 0 ? NIN : NN, wp = i == 0 ? NINP : NN, g8 = wp >> 3;
            for (int q = tid; q < NN * g8; q += PP_THREADS) {
                const int o = q / g8, j0 = (q - o * g8) * 8;
                float v[8];
#pragma unroll
                for (int e = 0; e < 8; ++e) v[e] = (j0 + e < win) ? src[o * win + j0 + e] : 0.0f;
                uint32_t hw[4], lw[4];
#pragma unroll
                for (int e = 0; e < 8; e += 2) {
                    __half h0, l0, h1, l1;
                    tc::split_f16(v[e], h0, l0);
                    tc::split_f16(v[e + 1], h1, l1);
                    __half2 hh2 = __halves2half2(h0, h1), ll2 = __halves2half2(l0, l1);
                    hw[e / 2] = *reinterpret_cast<uint32_t *>(&hh2);
                    lw[e / 2] = *reinterpret_cast<uint32_t *>(&ll2);
                }
                const uint32_t off = tc::tile_off(o, j0, wp);
                *reinterpret_cast<uint4 *>(smem + sh.o_w[i] + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
                *reinterpret_cast<uint4 *>(smem + sh.o_wlo[i] + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
            }
            src += NN * win;
        }
        for (int q = tid; q < NN; q += PP_THREADS) reinterpret_cast<float *>(smem + sh.o_wout)[q] = src[q];
    }
    for (int q = tid; q < 2 * 8 * TILE * 2 / 16; q += PP_THREADS)  // both dout tiles (contiguous)
        reinterpret_cast<uint4 *>(smem + sh.o_dout[0])[q] = make_uint4(0, 0, 0, 0);
    if (warp == 0) tc::tmem_alloc(&tmem_base_sh, sh.t_alloc);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base_sh;
    auto load_x = [&](int t, int64_t tile) {  // X hi -> o_d[t], X lo -> o_hlo[t]
        const uint8_t *src = xtiles + tile * xtile_bytes;
        tc::mbar_arrive_expect_tx(&bar_x[t], 2 * sh.xhalf);
        tc::bulk_g2s(smem + sh.o_d[t], src, sh.xhalf, &bar_x[t]);
        tc::bulk_g2s(smem + sh.o_hlo[t], src + sh.xhalf, sh.xhalf, &bar_x[t]);
    };
    if (tid == 0) {
        for (int t = 0; t < 2; ++t)
            if ((int64_t)blockIdx.x + t * (int64_t)gridDim.x < ntiles) load_x(t, blockIdx.x + t * (int64_t)gridDim.x);
    }
    const int nph = 2 * NH;

    if (warp == PP_EPI_WARPS) {
        // ================================================================ MMA issuer
        if (lane == 0) {
            uint32_t par_x = 0, par_xr = 0, par_op = 0, dw_started = 0, started = 0, par_dwo = 0;
            int64_t kt0 = 0, kt1 = 1;
            int ph0 = 0, ph1 = 0;
            const uint32_t idesc_fwd = tc::make_idesc(128, NN, 0, 0), idesc_fwd2 = tc::make_idesc(128, 2 * NN, 0, 0);
#ifdef NVOL_TIMELINE
            int mma_n = 0;
            TL(4000, gtime());
#endif
            for (;;) {
                bool any = false;
                for (int t = 0; t < 2; ++t) {
                    const int64_t kt = t ? kt1 : kt0;
                    const int ph = t ? ph1 : ph0;
                    if ((int64_t)blockIdx.x + kt * (int64_t)gridDim.x >= ntiles) continue;
                    any = true;
                    if ((started >> t) & 1u) {  // previous phase's epilogue released its operands / TMEM
                        tc::mbar_wait(&bar_op[t], (par_op >> t) & 1u);
                        par_op ^= 1u << t;
                    }
                    started |= 1u << t;
                    if (ph == 0) {
                        tc::mbar_wait(&bar_x[t], (par_x >> t) & 1u);
                        par_x ^= 1u << t;
                    }
                    if (ph == nph - 1 && NH > 1) {  // dW_0 reads the reloaded X hi tile
                        tc::mbar_wait(&bar_xr[t], (par_xr >> t) & 1u);
                        par_xr ^= 1u << t;
                    }
                    tc::fence_after();
#ifdef NVOL_TIMELINE
                    TL(2 * mma_n, gtime());
#endif
                    const uint32_t acc = tmem + sh.t_acc[t];
                    const uint32_t dbuf = tc::smem_u32(smem + sh.o_d[t]), lbuf = tc::smem_u32(smem + sh.o_hlo[t]);
                    if (ph < NH) {
                        // forward layer i, split fp16: hi*hi -> acc; lo*hi + hi*lo -> acc + NN (x kLoScale)
                        const int i = ph;
                        const int win = (i == 0) ? NINP : NN;
                        const uint32_t sbo = (win / 8) * 128;
                        const uint32_t ah = (i == 0) ? dbuf : tc::smem_u32(smem + sh.o_h[t][i]);
                        const uint64_t adh = tc::make_desc(ah, 128, sbo), adl = tc::make_desc(lbuf, 128, sbo);
                        const uint64_t bdh = tc::make_desc(tc::smem_u32(smem + sh.o_w[i]), 128, sbo);
                        for (int k = 0; k < win / 16; ++k) {
                            const uint64_t dk = (uint64_t)(k * 16);  // +256 bytes per K step
                            // [hi*W_hi | hi*W_lo] -> [acc | acc + NN] in one N = 2*NN MMA (B = [W_hi; W_lo]),
                            // then lo*W_hi -> acc + NN
                            tc::mma_f16(acc, adh + dk, bdh + dk, idesc_fwd2, k > 0);
                            tc::mma_f16(acc + NN, adl + dk, bdh + dk, idesc_fwd, 1);
                        }
                    } else {
                        // backward layer j: dW_j += delta^T H_j (both slots accumulate), dX = delta W_j
                        const int j = nph - 1 - ph;
                        const int win = (j == 0) ? NINP : NN;
                        const uint32_t hb = (j == 0) ? lbuf : tc::smem_u32(smem + sh.o_h[t][j]);
                        if (j == NH - 1) {
                            // dW_out^T [hidden x 8] += h_NH^T (lbuf, MN-major A) x delta_out (K-major B, N = 8)
                            const uint32_t id = tc::make_idesc(128, 8, 1, 0);
                            const uint64_t ad = tc::make_desc(lbuf, (NN / 8) * 128, 128);
                            const uint64_t bd = tc::make_desc(tc::smem_u32(smem + sh.o_dout[t]), 128, 2048);
                            const uint32_t first = ((dw_started >> 31) & 1u) ? 1u : 0u;
                            for (int k = 0; k < TILE / 16; ++k)
                                tc::mma_f16(tmem + sh.t_dwout, ad + (uint64_t)(k * 2 * (NN / 8) * 8),
                                            bd + (uint64_t)(k * 16), id, (first || k > 0) ? 1 : 0);
                            dw_started |= 1u << 31;
                            if (NH == 1) {
                                // one hidden layer: dW_out (reads h_1 in lbuf) and dW_0 (reads the X hi
                                // reload into lbuf) share this phase, so the reload happens here, after
                                // the dW_out MMAs completed, instead of in the epilogue
                                tc::mma_commit(&bar_dwo);
                                tc::mbar_wait(&bar_dwo, par_dwo);
                                par_dwo ^= 1u;
                                tc::mbar_arrive_expect_tx(&bar_xr[t], sh.xhalf);
                                tc::bulk_g2s(smem + sh.o_hlo[t], xtiles + ((int64_t)blockIdx.x + kt * (int64_t)gridDim.x) * xtile_bytes,
                                             sh.xhalf, &bar_xr[t]);
                                tc::mbar_wait(&bar_xr[t], (par_xr >> t) & 1u);
                                par_xr ^= 1u << t;
                                tc::fence_after();
                            }
                        }
                        {
                            const uint32_t id = tc::make_idesc(128, win, 1, 1);
                            const uint64_t ad = tc::make_desc(dbuf, (NN / 8) * 128, 128);
                            const uint64_t bd = tc::make_desc(hb, (win / 8) * 128, 128);
                            const uint32_t first = ((dw_started >> j) & 1u) ? 1u : 0u;
                            for (int k = 0; k < TILE / 16; ++k)
                                tc::mma_f16(tmem + sh.t_dw[j], ad + (uint64_t)(k * 2 * (NN / 8) * 8),
                                            bd + (uint64_t)(k * 2 * (win / 8) * 8), id, (first || k > 0) ? 1 : 0);
                            dw_started |= 1u << j;
                        }
                        {
                            const uint32_t id = tc::make_idesc(128, win, 0, 1);
                            const uint64_t ad = tc::make_desc(dbuf, 128, (NN / 8) * 128);
                            const uint64_t bd = tc::make_desc(tc::smem_u32(smem + sh.o_w[j]), (win / 8) * 128, 128);
                            for (int k = 0; k < NN / 16; ++k)
                                tc::mma_f16(acc, ad + (uint64_t)(k * 16), bd + (uint64_t)(k * 2 * (win / 8) * 8), id,
                                            k > 0);
                        }
                    }
                    tc::mma_commit(&bar_acc[t]);
#ifdef NVOL_TIMELINE
                    TL(2 * mma_n + 1, ((unsigned long long)t << 60) | ((unsigned long long)ph << 52) | (gtime() & ((1ull << 52) - 1)));
                    ++mma_n;
#endif
                    int nph_next = ph + 1;
                    int64_t nkt = kt;
                    if (nph_next == nph) {
                        nph_next = 0;
                        nkt += 2;
                    }
                    if (t) {
                        ph1 = nph_next;
                        kt1 = nkt;
                    } else {
                        ph0 = nph_next;
                        kt0 = nkt;
                    }
                }
                if (!any) break;
            }
        }
        __syncwarp();
    } else {
        // ================================================================ epilogue slot t
        const int t = warp >> 3, hh = (warp >> 2) & 1, q = warp & 3;
        const int s = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const uint32_t tacc = tmem + lane_base + sh.t_acc[t];
        uint8_t *dbuf = smem + sh.o_d[t];
        uint8_t *lbuf = smem + sh.o_hlo[t];
        float *s_part = reinterpret_cast<float *>(smem + sh.o_part) + t * 2 * TILE;
        const float *s_wout = reinterpret_cast<const float *>(smem + sh.o_wout);
        uint32_t par_acc = 0;
        double lsum = 0.0;  // this row's loss terms over the slot's tiles (column half 0 only)
        int cn0, cnn;
        group_cols(NN, hh, 2, cn0, cnn);  // this thread's hidden columns [cn0, cn0 + cnn), cnn <= 32
#ifdef NVOL_TIMELINE
        int epi_n = 0;
#endif
        auto release = [&]() {            // smem operands written / TMEM reads done -> MMA warp
#ifdef NVOL_TIMELINE
            if ((warp & 7) == 0 && lane == 0) TL(1024 + t * 1024 + 2 * epi_n + 1, gtime());
            if (t == 0 && lane == 0 && epi_n < 12) TL(3100 + epi_n * 8 + (warp & 7), gtime());
#endif
            tc::fence_before();
            tc::fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&bar_op[t]);
        };
        for (int64_t kt = t;; kt += 2) {
            const int64_t tile = (int64_t)blockIdx.x + kt * (int64_t)gridDim.x;
            if (tile >= ntiles) break;
            const int64_t row = tile * TILE + s;
            const bool valid = row < b;
            const float tgt = valid ? __ldg(targets + row) : 0.0f;
            // ---- forward epilogues: accumulator = kActScale * pre-activation
            float outp = 0.0f;
            for (int i = 0; i < NH; ++i) {
                tc::mbar_wait_sleep(&bar_acc[t], par_acc);
                par_acc ^= 1u;
                tc::fence_after();
#ifdef NVOL_TIMELINE
                ++epi_n;
                if ((warp & 7) == 0 && lane == 0) TL(1024 + t * 1024 + 2 * epi_n, gtime());
#endif
                const bool last = i == NH - 1;
                uint8_t *dst = last ? lbuf : smem + sh.o_h[t][i + 1];
                // chunk 0's hi + lo and chunk 1's hi in flight together; chunk 1's lo
                // is fetched while chunk 0 is processed
                float v0[16], vl[16], v1[16];
                const bool two = cnn > 16;
                tc::tmem_ld16(tacc + cn0, v0);
                tc::tmem_ld16(tacc + NN + cn0, vl);
                if (two) tc::tmem_ld16(tacc + cn0 + 16, v1);
                tc::tmem_wait_ld();
                auto chunk = [&](float(&v)[16], int c) {
#pragma unroll
                    for (int e = 0; e < 16; ++e) v[e] = relu_nan(v[e] + vl[e] * (1.0f / tc::kLoScale));
                    store_row_f16(dst, s, c, NN, v, false);
                    if (!last) {
#pragma unroll
                        for (int e = 0; e < 16; ++e) vl[e] = (v[e] - __half2float(__float2half_rn(v[e]))) * tc::kLoScale;
                        store_row_f16(lbuf, s, c, NN, vl, false);
                    } else {
#pragma unroll
                        for (int e = 0; e < 16; ++e) outp += s_wout[c + e] * v[e];
                    }
                };
                if (cnn > 0) chunk(v0, cn0);
                if (two) {
                    tc::tmem_ld16(tacc + NN + cn0 + 16, vl);
                    tc::tmem_wait_ld();
                    chunk(v1, cn0 + 16);
                }
                if (!last) release();
            }
            // ---- output layer + loss gradient (both column halves of a row see the same sum)
            s_part[hh * TILE + s] = outp;
            named_sync(1 + t, 256);
            const float o = (s_part[s] + s_part[TILE + s]) * (1.0f / tc::kActScale);
            const float pred = sh.relu_out ? relu_nan(o) : o;
            if (dbg_pred && valid && hh == 0) dbg_pred[row] = pred;  // parity hook (nvol_train_tc_debug)
            const double d = (double)pred - (double)tgt;
            double g, sl;
            if (sh.loss_kind == 0) {
                sl = fabs(d);
                g = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : (d == d ? 0.0 : d))) * inv_bglobal;  // np.sign(NaN) = NaN
            } else {
                sl = d * d;
                g = 2.0 * d * inv_bglobal;
            }
            float gf = (float)g;
            if (sh.relu_out && !(pred > 0.0f)) gf *= 0.0f;  // d * (act > 0): a NaN d stays NaN (numpy)
            if (!valid) {
                gf = 0.0f;
                sl = 0.0;
            }
            lsum += sl;
            // ---- delta_out for the dW_out MMA (fp16, x dscale) and delta_NH = mask(h_NH) * g * w_out
            {
                const float gd = gf * dscale;
                if (hh == 0)
                    *reinterpret_cast<__half *>(smem + sh.o_dout[t] + tc::tile_off(0, s, TILE)) = __float2half_rn(gd);
#pragma unroll
                for (int ch = 0; ch < 2; ++ch) {
                    const int c = cn0 + ch * 16;
                    if (ch * 16 < cnn) {
                        float hv[16], dv[16];
                        load_row_f16(lbuf, s, c, NN, hv);
#pragma unroll
                        for (int e = 0; e < 16; ++e) dv[e] = hv[e] > 0.0f ? gd * s_wout[c + e] : gd * s_wout[c + e] * 0.0f;
                        store_row_f16(dbuf, s, c, NN, dv, false);
                    }
                }
            }
            release();
            // ---- backward epilogues
            for (int j = NH - 1; j >= 0; --j) {
                tc::mbar_wait_sleep(&bar_acc[t], par_acc);
                par_acc ^= 1u;
                tc::fence_after();
#ifdef NVOL_TIMELINE
                ++epi_n;
                if ((warp & 7) == 0 && lane == 0) TL(1024 + t * 1024 + 2 * epi_n, gtime());
#endif
                if (j == NH - 1 && NH > 1 && hh == 0 && q == 0 && lane == 0) {
                    // the dW_out / dW_{NH-1} MMAs that read lbuf (h_NH) are done: reload X hi for dW_0
                    tc::mbar_arrive_expect_tx(&bar_xr[t], sh.xhalf);
                    tc::bulk_g2s(lbuf, xtiles + tile * xtile_bytes, sh.xhalf, &bar_xr[t]);
                }
                if (j > 0) {
                    const uint8_t *hj = smem + sh.o_h[t][j];
                    float v[2][16];
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch)
                        if (ch * 16 < cnn) tc::tmem_ld16(tacc + cn0 + ch * 16, v[ch]);
#pragma unroll
                    for (int ch = 0; ch < 2; ++ch) {
                        if (ch * 16 >= cnn) continue;
                        const int c = cn0 + ch * 16;
                        float hv[16];
                        load_row_f16(hj, s, c, NN, hv);
                        if (ch == 0) tc::tmem_wait_ld();
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[ch][e] = hv[e] > 0.0f ? v[ch][e] : v[ch][e] * 0.0f;
                        store_row_f16(dbuf, s, c, NN, v[ch], false);
                    }
                } else {
                    // the slot's smem buffers are free once dW_0 / dX_0 completed: next X tile
                    if (hh == 0 && q == 0 && lane == 0 && tile + 2 * (int64_t)gridDim.x < ntiles)
                        load_x(t, tile + 2 * (int64_t)gridDim.x);
                    int c0, nc;
                    group_cols(NINP, hh, 2, c0, nc);
                    for (int c = c0; c < c0 + nc; c += 16) {
                        float v[16];
                        tc::tmem_ld16(tacc + c, v);
                        tc::tmem_wait_ld();
                        if (valid) {
                            // feature-major dL/dfeat [NIN][B]: a warp stores 32 consecutive rows per column
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                if (c + e < NIN) {
                                    const float dv = v[e] * (1.0f / dscale);
                                    if (isnan(dv)) nan_at = 0;  // the encoder group (group 0) gets a NaN gradient
                                    dfeat[(int64_t)(c + e) * stride + row] = dv;
                                }
                        }
                    }
                }
                release();
            }
        }
        // ---- the loss: warp-reduce, one double atomic per CTA after the barrier
        for (int o2 = 16; o2 > 0; o2 >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o2);
        if (lane == 0) s_loss[warp] = hh == 0 ? lsum : 0.0;
    }
    __syncthreads();
    if (tid == PP_THREADS - 32) {
        double l = 0.0;
        for (int w = 0; w < PP_EPI_WARPS; ++w) l += s_loss[w];
        atomicAdd(loss_sum, l);
    }
    // ---- flush dW_0..dW_{nh-1} (fp32) once per CTA: vector REDs straight into the gradient
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp < PP_EPI_WARPS) {
        const int q = warp & 3, grp = warp >> 2;
        const int o = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const float unscale = 1.0f / (dscale * tc::kActScale);  // dW = (dscale*delta)^T (kActScale*H)
        int64_t base = 0;
        for (int j = 0; j < NH; ++j) {
            const int win = (j == 0) ? NIN : NN;
            const int wacc = (j == 0) ? NINP : NN;
            int c0, nc;
            group_cols(wacc, grp, 4, c0, nc);
            if (q * 32 < NN) {  // warp-uniform: lanes of quarters past nn hold no dW rows
                for (int c = c0; c < c0 + nc; c += 16) {
                    float v[16];
                    tc::tmem_ld16(tmem + lane_base + sh.t_dw[j] + c, v);
                    tc::tmem_wait_ld();
                    if (o < NN) {
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (c + e < win && isnan(v[e])) nan_at = min(nan_at, woff + base);  // W_j's group
                        float *g = dw_grads + base + (int64_t)o * win + c;
                        if (c + 16 <= win && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
#pragma unroll
                            for (int e = 0; e < 16; e += 4)
                                atomicAdd(reinterpret_cast<float4 *>(g + e),
                                          make_float4(v[e] * unscale, v[e + 1] * unscale, v[e + 2] * unscale,
                                                      v[e + 3] * unscale));
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                if (c + e < win) atomicAdd(g + e, v[e] * unscale);
                        }
                    }
                }
            }
            base += (int64_t)NN * win;
        }
        if (grp == 0 && q * 32 < NN) {  // dW_out^T: lane o = hidden unit, column 0
            float v[16];
            tc::tmem_ld16(tmem + lane_base + sh.t_dwout, v);  // columns 0..15 (8 allocated + neighbours; only 0 used)
            tc::tmem_wait_ld();
            if (o < NN) {
                if (isnan(v[0])) nan_at = min(nan_at, woff + base);
                atomicAdd(dw_grads + base + o, v[0] * unscale);
            }
        }
    }
    if (nan_at != kNanNone) nan_mark(nan_state, nan_at);
    tc::fence_before();
    __syncthreads();
#ifdef NVOL_TIMELINE
    if (tid == 0) TL(4001, gtime());
#endif
    if (warp == 0) tc::tmem_dealloc(tmem, sh.t_alloc);
}

// ============================================================================ 2b. MLP, four slots
// mlp_tc4_kernel: the same forward / loss / backward as mlp_tc_kernel, with up to
// FOUR 128-sample tiles in flight per SM, so the ~3.5 tiles an SM gets at B = 65,536
// all run concurrently (one dependent 2*NH-phase chain per SM instead of two).
// What makes the room: (1) the split-fp16 forward folds its hi*hi, lo*hi and hi*lo
// products into ONE accumulator (lo parts stored unscaled; fp16 subnormals are
// exact tensor-core inputs), so a slot needs nn TMEM columns instead of 2*nn;
// (2) a slot owns just two operand buffers P and Q (32 KB at nn = 64) that the
// epilogue overwrites in place: forward P/Q = activation hi/lo, backward P = delta
// and Q = the activation h_j the dW_j MMA needs, streamed back by a bulk copy from a
// global scratch the forward epilogue wrote it to (L2-resident, 48 KB per tile);
// (3) ReLU masks live in registers (bits), and dW_out = sum g*h_NH is reduced on
// CUDA cores (warp transpose-reduce + shared atomics).  Two MMA warps each serve
// half of the slots in round-robin order, blocking on each slot's barriers
// (Tc4Shape::rr; NVOL_MMA_RR=0: poll all slots and serve whichever is ready).
constexpr int M4_SLOTS = 4;
constexpr int M4_MMA_WARPS = 2;  // up to this many MMA issuers (launch: NVOL_MMA_WARPS, default 2); warp m
                                  // serves the slots t with t % (issuers) == m
constexpr int M4_WARPS = 4 * M4_SLOTS + M4_MMA_WARPS;  // 4 epilogue warps per slot (one per TMEM lane quarter) + MMA
constexpr int M4_THREADS = M4_WARPS * 32;

struct Tc4Shape {
    int nin, ninp, nn, nh, accw, slots, relu_out, loss_kind;
    int split;  // 1: split-fp16 forward (hi*W_hi + lo*W_hi + hi*W_lo); 0: plain fp16 forward (hi*W_hi)
    int rr;     // 1: the MMA warp serves the slots in round-robin order, blocking on each (no polling)
    uint32_t o_w[MAX_NH], o_wl[MAX_NH], o_wout, o_dwout, o_p[M4_SLOTS], o_q[M4_SLOTS], smem_bytes, half_bytes;
    uint32_t xhalf, t_acc[M4_SLOTS], t_dw[MAX_NH], t_alloc;
    uint32_t img_bytes;              // the packed weight image [0, img_bytes) of shared memory (pack_w4)
    int64_t w_floats, h_tile_bytes;  // per tile, per stored activation h_1..h_{nh-1} in the scratch
};

static bool mlp_split_enabled() {
    static int on = -1;  // NVOL_MLP_SPLIT=0: plain fp16 training forward (A/B measurements)
    if (on < 0) {
        const char *e = getenv("NVOL_MLP_SPLIT");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

static int build_shape4(Tc4Shape &s, int m, int n, int nn, int nh, int relu_out, int loss_kind) {
    s.nin = m * n;
    s.ninp = (s.nin + 15) & ~15;
    s.nn = nn;
    s.nh = nh;
    s.relu_out = relu_out;
    s.loss_kind = loss_kind;
    s.split = mlp_split_enabled() ? 1 : 0;
    {
        static int rr = -1;  // NVOL_MMA_RR=0: the polling MMA issuer (A/B measurements)
        if (rr < 0) {
            const char *e = getenv("NVOL_MMA_RR");
            rr = (e && e[0] == '0') ? 0 : 1;
        }
        s.rr = rr;
    }
    if (nh < 1 || nh > MAX_NH || !(nn == 16 || nn == 32 || nn == 64)) return 0;
    if (s.ninp > 2 * nn || s.ninp > 128) return 0;
    s.accw = max(nn, s.ninp);
    s.xhalf = 2u * TILE * s.ninp;
    s.half_bytes = 2u * TILE * s.accw;
    s.h_tile_bytes = 2ll * TILE * nn;
    s.w_floats = (int64_t)nn * s.nin + (int64_t)(nh - 1) * nn * nn + nn;
    const int dwcols = s.ninp + (nh - 1) * nn;
    for (int slots = M4_SLOTS; slots >= 3; --slots) {
        if (slots * s.accw + dwcols > 512) continue;
        uint32_t off = 0;
        auto take = [&](uint32_t bytes) {
            uint32_t r = off;
            off += (bytes + 127) & ~127u;
            return r;
        };
        for (int i = 0; i < nh; ++i) {
            s.o_w[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
            s.o_wl[i] = take(2u * nn * (i == 0 ? s.ninp : nn));
        }
        s.o_wout = take(4u * nn);
        s.img_bytes = off;
        s.o_dwout = take(4u * nn * 4 * M4_SLOTS);  // dW_out partials, one row per epilogue warp
        off = (off + 1023) & ~1023u;
        for (int t = 0; t < slots; ++t) {
            s.o_p[t] = take(s.half_bytes);
            s.o_q[t] = take(s.half_bytes);
        }
        // the M = 128 MN-major delta^T operand of the dW MMAs reads up to ~2 KB past an
        // nn-wide tile (rows >= nn, unused): slack after the last buffer; the prologue
        // stages the fp32 weights over the slot buffers
        const uint32_t slot_area = off - s.o_p[0];
        off += 4096;
        if ((int64_t)slot_area < s.w_floats * 4) continue;
        if (off > 227u * 1024u - 1024u) continue;
        s.slots = slots;
        s.smem_bytes = off;
        uint32_t col = 0;
        for (int t = 0; t < slots; ++t) {
            s.t_acc[t] = col;
            col += s.accw;
        }
        for (int i = 0; i < nh; ++i) {
            s.t_dw[i] = col;
            col += (i == 0) ? s.ninp : nn;
        }
        uint32_t a = 32;
        while (a < col) a <<= 1;
        s.t_alloc = a;
        return 1;
    }
    return 0;
}

__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile(
        "{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(p));
    return p != 0;
}

__device__ __forceinline__ bool mbar_test(uint64_t *bar, uint32_t phase) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(tc::smem_u32(bar)), "r"(phase)
        : "memory");
    return ok != 0;
}

// the generic-proxy stores of the activation scratch become visible to the bulk copies that read them
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// dead step scratch (activation scratch, X tiles, dL/dfeat): drop the 128-byte L2 line without a
// DRAM write-back once its last reader is done (the next step rewrites it before reading)
__device__ __forceinline__ void discard_l2(const void *p) {
    asm volatile("discard.global.L2 [%0], 128;" ::"l"(p) : "memory");
}

__device__ __forceinline__ void st_global_v4(void *p, uint4 v) {
    asm volatile("st.global.v4.b32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
}

// 16 consecutive fp32 -> fp16 hi (+ unscaled fp16 lo) in the core-matrix layout at (row, c)
__device__ __forceinline__ void split_row16(const float *v, uint4 &h0, uint4 &h1, uint4 &l0, uint4 &l1) {
    uint32_t hw[8], lw[8];
#pragma unroll
    for (int e = 0; e < 16; e += 2) {
        const __half a = __float2half_rn(v[e]), b = __float2half_rn(v[e + 1]);
        const __half la = __float2half_rn(v[e] - __half2float(a)), lb = __float2half_rn(v[e + 1] - __half2float(b));
        __half2 hh = __halves2half2(a, b), ll = __halves2half2(la, lb);
        hw[e / 2] = *reinterpret_cast<uint32_t *>(&hh);
        lw[e / 2] = *reinterpret_cast<uint32_t *>(&ll);
    }
    h0 = make_uint4(hw[0], hw[1], hw[2], hw[3]);
    h1 = make_uint4(hw[4], hw[5], hw[6], hw[7]);
    l0 = make_uint4(lw[0], lw[1], lw[2], lw[3]);
    l1 = make_uint4(lw[4], lw[5], lw[6], lw[7]);
}

// The MLP weights as mlp_tc4_kernel's shared-memory image [0, img_bytes): per layer the fp16 hi
// tile then the unscaled fp16 lo tile (core-matrix layout, input columns padded to ninp), then
// the fp32 output row.  Built once per step by the first blocks of the encoder kernel (or
// pack_w4_kernel), so the MLP kernel's prologue is one bulk copy.
__device__ __forceinline__ void pack_w4(const float *__restrict__ w, int nin, int ninp, int nn, int nh,
                                        uint8_t *__restrict__ img, int64_t t0, int64_t nthreads) {
    const uint32_t w1 = 4u * nn * ninp, wst = 4u * nn * nn;
    const float *src = w;
    for (int i = 0; i < nh; ++i) {
        const int win = i == 0 ? nin : nn, wp = i == 0 ? ninp : nn, g8 = wp >> 3;
        const uint32_t ow = i == 0 ? 0u : w1 + (uint32_t)(i - 1) * wst;
        const uint32_t owl = ow + (i == 0 ? 2u * nn * ninp : 2u * nn * nn);
        for (int64_t q = t0; q < (int64_t)nn * g8; q += nthreads) {
            const int o = (int)(q / g8), j0 = (int)(q - (int64_t)o * g8) * 8;
            uint32_t hw[4], lw[4];
#pragma unroll
            for (int e = 0; e < 8; e += 2) {
                const float a = (j0 + e < win) ? src[o * win + j0 + e] : 0.0f;
                const float b = (j0 + e + 1 < win) ? src[o * win + j0 + e + 1] : 0.0f;
                const __half ha = __float2half_rn(a), hb = __float2half_rn(b);
                const __half la = __float2half_rn(a - __half2float(ha)), lb = __float2half_rn(b - __half2float(hb));
                __half2 hh = __halves2half2(ha, hb), ll = __halves2half2(la, lb);
                hw[e / 2] = *reinterpret_cast<uint32_t *>(&hh);
                lw[e / 2] = *reinterpret_cast<uint32_t *>(&ll);
            }
            const uint32_t off = tc::tile_off(o, j0, wp);
            *reinterpret_cast<uint4 *>(img + ow + off) = make_uint4(hw[0], hw[1], hw[2], hw[3]);
            *reinterpret_cast<uint4 *>(img + owl + off) = make_uint4(lw[0], lw[1], lw[2], lw[3]);
        }
        src += (int64_t)nn * win;
    }
    const uint32_t owout = w1 + (uint32_t)(nh - 1) * wst;
    for (int64_t q = t0; q < nn; q += nthreads) reinterpret_cast<float *>(img + owout)[q] = src[q];
}

constexpr int PACK_BLOCKS = 8;

__global__ void __launch_bounds__(256) pack_w4_kernel(const float *__restrict__ w, int nin, int ninp, int nn, int nh,
                                                      uint8_t *__restrict__ img) {
    pack_w4(w, nin, ninp, nn, nh, img, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
}

__global__ void __launch_bounds__(M4_THREADS, 1) mlp_tc4_kernel(
    const uint8_t *__restrict__ xtiles, const float *__restrict__ targets, int64_t b, double inv_bglobal, float dscale,
    const Tc4Shape sh, const float *__restrict__ wflat, double *__restrict__ loss_sum, float *__restrict__ dfeat,
    int64_t stride, float *__restrict__ dw_grads, uint8_t *__restrict__ hscratch, float *__restrict__ dbg_pred,
    int64_t *__restrict__ nan_state, int64_t woff, const uint8_t *__restrict__ wimg, float *__restrict__ dw_part) {
    if (nan_halted(nan_state)) return;  // NaN contract: a halted pipeline does no more work
#ifdef NVOL_TIMELINE
    if (threadIdx.x == 0) TL(4002, gtime());
#endif
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar_x[M4_SLOTS], bar_h[M4_SLOTS], bar_acc[M4_SLOTS], bar_op[M4_SLOTS], bar_w;
    __shared__ uint32_t tmem_base_sh;
    __shared__ double s_loss[4 * M4_SLOTS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int NN = sh.nn, NINP = sh.ninp, NH = sh.nh, NIN = sh.nin, S = sh.slots;
    const int64_t ntiles = (b + TILE - 1) / TILE;
    const int64_t xtile_bytes = 2 * (int64_t)sh.xhalf;
    const int64_t hs_tile = (int64_t)(NH - 1) * sh.h_tile_bytes;
    int64_t nan_at = kNanNone;
    auto tile_of = [&](int t, int64_t k) -> int64_t { return (int64_t)blockIdx.x + ((int64_t)t + (int64_t)S * k) * gridDim.x; };

    auto load_x = [&](int t, int64_t tile) {  // X hi -> P[t], X lo -> Q[t] (split forward only)
        const uint8_t *src = xtiles + tile * xtile_bytes;
        tc::mbar_arrive_expect_tx(&bar_x[t], (sh.split ? 2 : 1) * sh.xhalf);
        tc::bulk_g2s(smem + sh.o_p[t], src, sh.xhalf, &bar_x[t]);
        if (sh.split) tc::bulk_g2s(smem + sh.o_q[t], src + sh.xhalf, sh.xhalf, &bar_x[t]);
    };
    // ---- prologue: the packed weight image (pack_w4) by one bulk copy
    if (tid == 0) {
        for (int t = 0; t < M4_SLOTS; ++t) {
            tc::mbar_init(&bar_x[t], 1);
            tc::mbar_init(&bar_h[t], 1);
            tc::mbar_init(&bar_acc[t], 1);
            tc::mbar_init(&bar_op[t], 4);  // one arrive per epilogue warp of the slot
        }
        tc::mbar_init(&bar_w, 1);
        tc::fence_mbar_init();
        tc::mbar_arrive_expect_tx(&bar_w, sh.img_bytes);
        tc::bulk_g2s(smem, wimg, sh.img_bytes, &bar_w);
        // the slots' first X tiles right behind it (the slot buffers lie past the image): their
        // latency overlaps the TMEM allocation and the dW zeroing below
        for (int t = 0; t < S; ++t)
            if (tile_of(t, 0) < ntiles) load_x(t, tile_of(t, 0));
    }
    for (int q = tid; q < 4 * M4_SLOTS * NN; q += blockDim.x) reinterpret_cast<float *>(smem + sh.o_dwout)[q] = 0.0f;
    __syncthreads();
    tc::mbar_wait(&bar_w, 0);
    if (warp == 0) tc::tmem_alloc(&tmem_base_sh, sh.t_alloc);
    tc::fence_proxy_async();
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tmem_base_sh;
    // zero the dW accumulators (every dW MMA then accumulates, so the issuer warps' chains into
    // one dW_j may interleave: the tensor pipe serialises their read-modify-writes,
    // tools/micro/mma_shared_acc.cu) -- the 16 epilogue warps, lane quarter x column group
    if (warp < 4 * M4_SLOTS) {
        const int q = warp & 3, grp = warp >> 2;
        const uint32_t dw0 = (uint32_t)S * sh.accw, ncol = (uint32_t)(NINP + (NH - 1) * NN);
        const uint32_t z = 0;
        for (uint32_t c = (uint32_t)grp * 8; c < ncol; c += 8 * M4_SLOTS)
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(
                             tmem + ((uint32_t)(q * 32) << 16) + dw0 + c), "r"(z)
                         : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // h_j (j >= 1: the scratch written by the forward epilogue; j = 0: the X hi tile) -> Q[t]
    auto load_h = [&](int t, int64_t tile, int j) {
        const uint8_t *src = j == 0 ? xtiles + tile * xtile_bytes : hscratch + tile * hs_tile + (int64_t)(j - 1) * sh.h_tile_bytes;
        const uint32_t bytes = j == 0 ? sh.xhalf : (uint32_t)sh.h_tile_bytes;
        tc::mbar_arrive_expect_tx(&bar_h[t], bytes);
        tc::bulk_g2s(smem + sh.o_q[t], src, bytes, &bar_h[t]);
    };
    const int nph = 2 * NH;

    if (warp >= 4 * M4_SLOTS) {
        // ================================================================ MMA issuers (round-robin over their slots)
        // The whole warp runs the loop converged, every decision is a warp vote and every
        // operand address is computed arithmetically from kernel parameters, so the state and
        // the descriptors stay warp-uniform (uniform registers): one elected lane issues each
        // phase's tcgen05.mma chain without per-instruction register->uniform moves.
        const uint32_t tmem_u = __shfl_sync(0xffffffffu, tmem, 0);
        const uint32_t sbase = tc::smem_u32(smem);
        const uint32_t w1 = 4u * NN * NINP, wst = 4u * NN * NN, wlo1 = 2u * NN * NN;  // o_w / o_wl by layer
        const uint32_t dw0 = (uint32_t)S * sh.accw;
        const int mw = warp - 4 * M4_SLOTS, nmw = (int)(blockDim.x >> 5) - 4 * M4_SLOTS;  // issuer mw of nmw
        uint32_t par_x = 0, par_h = 0, par_op = 0, started = 0, done = 0;
        int64_t kt[M4_SLOTS];
        int ph[M4_SLOTS];
#pragma unroll
        for (int t = 0; t < M4_SLOTS; ++t) {
            kt[t] = 0;
            ph[t] = 0;
            if (t >= S || t % nmw != mw || tile_of(t, 0) >= ntiles) done |= 1u << t;
        }
        const uint32_t idesc_f = tc::make_idesc(128, NN, 0, 0);
#ifdef NVOL_TIMELINE
        int mma_n = 0;
        if (lane == 0) TL(4000, gtime());
#endif
        while (done != (1u << M4_SLOTS) - 1u) {
            bool issued = false;
#pragma unroll
            for (int t = 0; t < M4_SLOTS; ++t) {
                if ((done >> t) & 1u) continue;
                const int p = ph[t];
                bool ok = true;
                if (sh.rr) {  // slots progress in lockstep: wait (suspended) for this one instead of polling all
                    if ((started >> t) & 1u) tc::mbar_wait_sleep(&bar_op[t], (par_op >> t) & 1u);
                    if (p == 0) tc::mbar_wait_sleep(&bar_x[t], (par_x >> t) & 1u);
                    if (p >= NH) tc::mbar_wait_sleep(&bar_h[t], (par_h >> t) & 1u);
                } else {
                    if ((started >> t) & 1u) ok = mbar_test(&bar_op[t], (par_op >> t) & 1u);
                    if (ok && p == 0) ok = mbar_test(&bar_x[t], (par_x >> t) & 1u);
                    if (ok && p >= NH) ok = mbar_test(&bar_h[t], (par_h >> t) & 1u);
                }
                if (!__all_sync(0xffffffffu, ok)) continue;
                if ((started >> t) & 1u) par_op ^= 1u << t;
                if (p == 0) par_x ^= 1u << t;
                if (p >= NH) par_h ^= 1u << t;
                started |= 1u << t;
                tc::fence_after();
#ifdef NVOL_TIMELINE
                if (lane == 0) TL(2 * ((2 * mma_n + mw) & 511), gtime());
#endif
                const uint32_t acc = tmem_u + (uint32_t)t * sh.accw;
                const uint32_t pb = sbase + sh.o_p[0] + 2u * (uint32_t)t * sh.half_bytes, qb = pb + sh.half_bytes;
                if (p < NH) {
                    // forward layer i: hi*W_hi + lo*W_hi + hi*W_lo into one accumulator
                    const int i = p, win = (i == 0) ? NINP : NN;
                    const uint32_t sbo = (win / 8) * 128;
                    const uint32_t ow = i == 0 ? 0u : w1 + (uint32_t)(i - 1) * wst;
                    const uint32_t owl = ow + (i == 0 ? 2u * NN * NINP : wlo1);
                    const uint64_t ah = tc::make_desc(pb, 128, sbo), al = tc::make_desc(qb, 128, sbo);
                    const uint64_t bh = tc::make_desc(sbase + ow, 128, sbo), bl = tc::make_desc(sbase + owl, 128, sbo);
                    if (elect_one()) {
                        for (int k = 0; k < win / 16; ++k) {
                            const uint64_t dk = (uint64_t)(k * 16);
                            tc::mma_f16(acc, ah + dk, bh + dk, idesc_f, k > 0);
                            if (sh.split) {
                                tc::mma_f16(acc, al + dk, bh + dk, idesc_f, 1);
                                tc::mma_f16(acc, ah + dk, bl + dk, idesc_f, 1);
                            }
                        }
                        tc::mma_commit(&bar_acc[t]);
                    }
                } else {
                    // backward layer j: dW_j += delta^T h_j (P^T x Q), dX = delta W_j (P x W_j)
                    const int j = nph - 1 - p, win = (j == 0) ? NINP : NN;
                    const uint32_t ow = j == 0 ? 0u : w1 + (uint32_t)(j - 1) * wst;
                    const uint32_t tdw = tmem_u + dw0 + (j == 0 ? 0u : (uint32_t)NINP + (uint32_t)(j - 1) * NN);
                    const uint32_t id1 = tc::make_idesc(128, win, 1, 1), id2 = tc::make_idesc(128, win, 0, 1);
                    const uint64_t ad1 = tc::make_desc(pb, (NN / 8) * 128, 128);
                    const uint64_t bd1 = tc::make_desc(qb, (win / 8) * 128, 128);
                    const uint64_t ad2 = tc::make_desc(pb, 128, (NN / 8) * 128);
                    const uint64_t bd2 = tc::make_desc(sbase + ow, (win / 8) * 128, 128);
                    if (elect_one()) {
                        for (int k = 0; k < TILE / 16; ++k)  // dW_j was zeroed in the prologue: always accumulate
                            tc::mma_f16(tdw, ad1 + (uint64_t)(k * 2 * (NN / 8) * 8), bd1 + (uint64_t)(k * 2 * (win / 8) * 8), id1, 1);
                        for (int k = 0; k < NN / 16; ++k)
                            tc::mma_f16(acc, ad2 + (uint64_t)(k * 16), bd2 + (uint64_t)(k * 2 * (win / 8) * 8), id2, k > 0);
                        tc::mma_commit(&bar_acc[t]);
                    }
                }
                __syncwarp();
                issued = true;
#ifdef NVOL_TIMELINE
                if (lane == 0)
                    TL(2 * ((2 * mma_n + mw) & 511) + 1, ((unsigned long long)t << 60) | ((unsigned long long)p << 52) | (gtime() & ((1ull << 52) - 1)));
                ++mma_n;
#endif
                if (p + 1 == nph) {
                    ph[t] = 0;
                    ++kt[t];
                    if (tile_of(t, kt[t]) >= ntiles) done |= 1u << t;
                } else {
                    ph[t] = p + 1;
                }
            }
            // nothing ready: back off instead of stealing issue slots from the epilogue
            // warps that share this warp's scheduler
            if (!issued) __nanosleep(64);
        }
    } else if ((warp >> 2) < S) {
        // ================================================================ epilogue: slot t, TMEM lane quarter q, row s
        const int t = warp >> 2, q = warp & 3;
        const int s = q * 32 + lane;
        const uint32_t tacc = tmem + ((uint32_t)(q * 32) << 16) + sh.t_acc[t];
        uint8_t *pbuf = smem + sh.o_p[t];
        uint8_t *qbuf = smem + sh.o_q[t];
        const float *s_wout = reinterpret_cast<const float *>(smem + sh.o_wout);
        float *s_dwout = reinterpret_cast<float *>(smem + sh.o_dwout);
        const bool leader = q == 0 && lane == 0;
        uint32_t par_acc = 0;
        double lsum = 0.0;
#ifdef NVOL_TIMELINE
        int epi_n = 0;
#endif
        auto release = [&]() {
            tc::fence_before();
            tc::fence_proxy_async();  // shared operands -> the tensor cores
            __syncwarp();
#ifdef NVOL_TIMELINE
            if (leader) TL(1024 + t * 256 + 2 * (epi_n & 127) + 1, gtime());
            if (lane == 0 && t < 2 && epi_n < 8) TL(3200 + t * 64 + epi_n * 4 + q, gtime());  // per-warp release
            ++epi_n;
#endif
            if (lane == 0) mbar_arrive(&bar_op[t]);
        };
        auto wait_acc = [&]() {
            tc::mbar_wait_sleep(&bar_acc[t], par_acc);
            par_acc ^= 1u;
            tc::fence_after();
#ifdef NVOL_TIMELINE
            if (leader) TL(1024 + t * 256 + 2 * (epi_n & 127), gtime());
#endif
        };
        for (int64_t k = 0;; ++k) {
            const int64_t tile = tile_of(t, k);
            if (tile >= ntiles) break;
            const int64_t row = tile * TILE + s;
            const bool valid = row < b;
            const float tgt = valid ? __ldg(targets + row) : 0.0f;
            uint8_t *hs = hscratch + tile * hs_tile;
            uint32_t mlo[MAX_NH + 1], mhi[MAX_NH + 1];  // ReLU masks of h_1..h_NH (64 columns = 2 words)
            // ---- forward epilogues 0 .. NH-2: h_{i+1} = relu(acc) -> P (hi), Q (lo), scratch (hi)
            for (int i = 0; i < NH - 1; ++i) {
                wait_acc();
                uint32_t bl = 0, bh = 0;
                for (int c = 0; c < NN; c += 16) {
                    float v[16];
                    tc::tmem_ld16(tacc + c, v);
                    tc::tmem_wait_ld();
                    uint32_t bits = 0;
#pragma unroll
                    for (int e = 0; e < 16; ++e) {
                        v[e] = relu_nan(v[e]);
                        bits |= (v[e] > 0.0f ? 1u : 0u) << e;
                    }
                    if (c < 32) bl |= bits << c; else bh |= bits << (c - 32);
                    uint4 h0, h1, l0, l1;
                    split_row16(v, h0, h1, l0, l1);
                    const uint32_t o0 = tc::tile_off(s, c, NN), o1 = tc::tile_off(s, c + 8, NN);
                    *reinterpret_cast<uint4 *>(pbuf + o0) = h0;
                    *reinterpret_cast<uint4 *>(pbuf + o1) = h1;
                    if (sh.split) {
                        *reinterpret_cast<uint4 *>(qbuf + o0) = l0;
                        *reinterpret_cast<uint4 *>(qbuf + o1) = l1;
                    }
                    uint8_t *g = hs + (int64_t)i * sh.h_tile_bytes;
                    st_global_v4(g + o0, h0);
                    st_global_v4(g + o1, h1);
                }
                mlo[i + 1] = bl;
                mhi[i + 1] = bh;
                release();
            }
            // ---- last forward epilogue: h_NH, output layer, loss gradient, delta_NH, dW_out
            wait_acc();
            // the slot's 4 warps wrote h_1..h_{NH-1} to the scratch (generic stores): proxy fence, then
            // order them before the bulk copies that stream them back (bar.sync: CTA memory barrier).
            // Done once per tile, phases after the stores, so the fence finds them retired.
#ifdef NVOL_TIMELINE
            if (leader && k == 0) TL(3000 + t * 8 + 0, gtime());
#endif
            fence_proxy_async_global();
            named_sync(1 + t, 128);
#ifdef NVOL_TIMELINE
            if (leader && k == 0) TL(3000 + t * 8 + 1, gtime());
#endif
            if (leader) load_h(t, tile, NH - 1);  // Q (h_{NH-1} lo) is free: stream h_{NH-1} back for dW_{NH-1}
            float outp = 0.0f;
            for (int c = 0; c < NN; c += 16) {
                float v[16];
                tc::tmem_ld16(tacc + c, v);
                tc::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; e += 4) {  // (16-byte shared loads: s_wout is 128-byte aligned)
                    const float4 w4 = *reinterpret_cast<const float4 *>(s_wout + c + e);
                    outp += w4.x * relu_nan(v[e]);
                    outp += w4.y * relu_nan(v[e + 1]);
                    outp += w4.z * relu_nan(v[e + 2]);
                    outp += w4.w * relu_nan(v[e + 3]);
                }
            }
#ifdef NVOL_TIMELINE
            if (leader && k == 0) TL(3000 + t * 8 + 2, gtime());
#endif
            const float o = outp * (1.0f / tc::kActScale);
            const float pred = sh.relu_out ? relu_nan(o) : o;
            if (dbg_pred && valid) dbg_pred[row] = pred;  // parity hook (nvol_train_tc_debug)
            const double d = (double)pred - (double)tgt;
            double gg, sl;
            if (sh.loss_kind == 0) {
                sl = fabs(d);
                gg = (d > 0.0 ? 1.0 : (d < 0.0 ? -1.0 : (d == d ? 0.0 : d))) * inv_bglobal;  // np.sign(NaN) = NaN
            } else {
                sl = d * d;
                gg = 2.0 * d * inv_bglobal;
            }
            float gf = (float)gg;
            if (sh.relu_out && !(pred > 0.0f)) gf *= 0.0f;  // d * (act > 0): a NaN d stays NaN (numpy)
            if (!valid) {
                gf = 0.0f;
                sl = 0.0;
            }
            lsum += sl;
            const float gd = gf * dscale;
#ifdef NVOL_TIMELINE
            if (leader && k == 0) TL(3000 + t * 8 + 3, gtime());
#endif
            for (int c = 0; c < NN; c += 16) {
                float v[16], dv[16], wv[16];
#pragma unroll
                for (int e = 0; e < 16; e += 4) {  // (issued ahead of the TMEM load's latency)
                    const float4 w4 = *reinterpret_cast<const float4 *>(s_wout + c + e);
                    wv[e] = w4.x;
                    wv[e + 1] = w4.y;
                    wv[e + 2] = w4.z;
                    wv[e + 3] = w4.w;
                }
                tc::tmem_ld16(tacc + c, v);
                tc::tmem_wait_ld();
#pragma unroll
                for (int e = 0; e < 16; ++e) {
                    v[e] = relu_nan(v[e]);
                    const float x = gd * wv[e];
                    dv[e] = v[e] > 0.0f ? x : x * 0.0f;
                }
                store_row_f16(pbuf, s, c, NN, dv, false);
                // dW_out[c + e] += sum over the warp's rows of gd * h: transpose-reduce 16 columns over 32 lanes
                float x[16];
#pragma unroll
                for (int e = 0; e < 16; ++e) x[e] = gd * v[e];
#pragma unroll
                for (int w = 8; w >= 1; w >>= 1) {
                    const bool up = (lane & (2 * w)) != 0;  // lane bit 4, 3, 2, 1 for w = 8, 4, 2, 1
#pragma unroll
                    for (int e = 0; e < w; ++e) {
                        const float send = up ? x[e] : x[e + w];
                        const float keep = up ? x[e + w] : x[e];
                        x[e] = keep + __shfl_xor_sync(0xffffffffu, send, 2 * w);
                    }
                }
                const float z = x[0] + __shfl_xor_sync(0xffffffffu, x[0], 1);
                const int col = ((lane >> 4) & 1) * 8 + ((lane >> 3) & 1) * 4 + ((lane >> 2) & 1) * 2 + ((lane >> 1) & 1);
                if ((lane & 1) == 0) s_dwout[warp * NN + c + col] += z;  // this warp's row: one owner lane per column
            }
            release();
            // ---- backward epilogues
            for (int j = NH - 1; j >= 0; --j) {
                wait_acc();
                if (j > 0) {
                    if (leader) load_h(t, tile, j - 1);  // Q (h_j) was read by dW_j: stream h_{j-1} back
                    for (int64_t ln = s; ln * 128 < sh.h_tile_bytes; ln += TILE)  // h_j's scratch is dead
                        discard_l2(hs + (int64_t)(j - 1) * sh.h_tile_bytes + ln * 128);
                    for (int c = 0; c < NN; c += 16) {
                        float v[16];
                        tc::tmem_ld16(tacc + c, v);
                        tc::tmem_wait_ld();
                        const uint32_t bits = (c < 32 ? mlo[j] >> c : mhi[j] >> (c - 32)) & 0xffffu;
#pragma unroll
                        for (int e = 0; e < 16; ++e) v[e] = ((bits >> e) & 1u) ? v[e] : v[e] * 0.0f;
                        store_row_f16(pbuf, s, c, NN, v, false);
                    }
                } else {
                    // the slot's buffers are free once dW_0 / dX_0 completed: next X tile
                    if (leader && tile_of(t, k + 1) < ntiles) load_x(t, tile_of(t, k + 1));
                    for (int64_t ln = s; ln * 128 < xtile_bytes; ln += TILE)  // this X tile is dead
                        discard_l2(xtiles + tile * xtile_bytes + ln * 128);
                    for (int c = 0; c < NINP; c += 16) {
                        float v[16];
                        tc::tmem_ld16(tacc + c, v);
                        tc::tmem_wait_ld();
                        if (valid) {
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                if (c + e < NIN) {
                                    const float dv = v[e] * (1.0f / dscale);
                                    if (isnan(dv)) nan_at = 0;  // the encoder group (group 0) gets a NaN gradient
                                    dfeat[(int64_t)(c + e) * stride + row] = dv;
                                }
                        }
                    }
                }
                release();
            }
        }
        for (int o2 = 16; o2 > 0; o2 >>= 1) lsum += __shfl_xor_sync(0xffffffffu, lsum, o2);
        if (lane == 0) s_loss[warp] = lsum;
    } else if (warp < 4 * M4_SLOTS && lane == 0) {
        s_loss[warp] = 0.0;  // slots this shape has no room for
    }
    __syncthreads();
    if (tid == 0) {
        double l = 0.0;
        for (int w = 0; w < 4 * M4_SLOTS; ++w) l += s_loss[w];
        atomicAdd(loss_sum, l);
    }
    // ---- flush dW_0..dW_{nh-1} (TMEM) and dW_out (shared) once per CTA: vector REDs into the gradient
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
#ifdef NVOL_TIMELINE
    if (threadIdx.x == 0) TL(4003, gtime());
#endif
    const float unscale = 1.0f / (dscale * tc::kActScale);  // dW = (dscale*delta)^T (kActScale*H)
    // dw_part: this CTA's dW as plain stores into its own partial row (summed in CTA order by
    // scatter_kernel's prologue); every CTA REDing into the same 57 KB of gradient at once
    // serialises on a few L2 slices (in-step MLP 37.9 -> 33.8 us, tools/gpu_r3t.sh)
    float *const dw_out = dw_part ? dw_part + (int64_t)blockIdx.x * sh.w_floats : dw_grads;
    if (warp < 4 * M4_SLOTS) {
        const int q = warp & 3, grp = warp >> 2;
        const int o = q * 32 + lane;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        int64_t base = 0;
        for (int j = 0; j < NH; ++j) {
            const int win = (j == 0) ? NIN : NN;
            const int wacc = (j == 0) ? NINP : NN;
            int c0, nc;
            group_cols(wacc, grp, 4, c0, nc);
            if (q * 32 < NN) {  // warp-uniform: lanes of quarters past nn hold no dW rows
                for (int c = c0; c < c0 + nc; c += 16) {
                    float v[16];
                    tc::tmem_ld16(tmem + lane_base + sh.t_dw[j] + c, v);
                    tc::tmem_wait_ld();
                    if (o < NN) {
#pragma unroll
                        for (int e = 0; e < 16; ++e)
                            if (c + e < win && isnan(v[e])) nan_at = min(nan_at, woff + base);  // W_j's group
                        float *g = dw_out + base + (int64_t)o * win + c;
                        if (c + 16 <= win && (reinterpret_cast<uintptr_t>(g) & 15) == 0) {
#pragma unroll
                            for (int e = 0; e < 16; e += 4) {
                                const float4 w4 = make_float4(v[e] * unscale, v[e + 1] * unscale, v[e + 2] * unscale,
                                                              v[e + 3] * unscale);
                                if (dw_part)
                                    *reinterpret_cast<float4 *>(g + e) = w4;
                                else
                                    atomicAdd(reinterpret_cast<float4 *>(g + e), w4);
                            }
                        } else {
#pragma unroll
                            for (int e = 0; e < 16; ++e)
                                if (c + e < win) {
                                    if (dw_part)
                                        g[e] = v[e] * unscale;
                                    else
                                        atomicAdd(g + e, v[e] * unscale);
                                }
                        }
                    }
                }
            }
            base += (int64_t)NN * win;
        }
#ifdef NVOL_TIMELINE
        if (lane == 0) TL(3600 + warp, gtime());  // per warp: dW rows out of TMEM and stored
#endif
        if (tid < NN) {
            float v = 0.0f;
            for (int w = 0; w < 4 * M4_SLOTS; ++w) v += reinterpret_cast<const float *>(smem + sh.o_dwout)[w * NN + tid];
            if (isnan(v)) nan_at = min(nan_at, woff + base);
            if (dw_part)
                dw_out[base + tid] = v * unscale;
            else
                atomicAdd(dw_grads + base + tid, v * unscale);
        }
    }
    if (nan_at != kNanNone) nan_mark(nan_state, nan_at);
    tc::fence_before();
    __syncthreads();
#ifdef NVOL_TIMELINE
    if (tid == 0) TL(4001, gtime());
#endif
    if (warp == 0) tc::tmem_dealloc(tmem, sh.t_alloc);
}

// ============================================================================ 3. scatter
// mlp_tc4_kernel's per-CTA weight-gradient partials [n_part][w_floats] (dw_part), summed in CTA
// order into the flat gradient (dw[q] += sum_r part[r][q]) by dw_reduce_kernel, which runs on a side
// stream beside the scatter (its 256-thread CTAs fit in the registers the scatter leaves free):
// each CTA owns DWR_Q consecutive q, its warps split the partial rows into DWR_G groups (128-byte
// loads), the group sums are folded in group order.  A NaN in a sum marks its parameter group
// (W_0 .. W_{nh-1}, W_out) as the MLP kernel's own flush would have.
struct DwPartials {
    const float *part;  // nullptr: the MLP kernel REDs its dW itself
    float *dw;          // the flat gradient's MLP weights (grads + woff)
    int n_part, w_floats, nin, nn, nh;
    int64_t woff;
};
constexpr int DWR_Q = 32, DWR_G = 8;

__global__ void __launch_bounds__(DWR_Q * DWR_G) dw_reduce_kernel(const DwPartials d, int64_t *__restrict__ nan_state) {
    if (nan_halted(nan_state)) return;
    __shared__ float s_red[DWR_G][DWR_Q];
    const int ql = threadIdx.x % DWR_Q, grp = threadIdx.x / DWR_Q;
    const int q = (int)blockIdx.x * DWR_Q + ql;
    const int rpg = (d.n_part + DWR_G - 1) / DWR_G;
    float acc = 0.0f;
    if (q < d.w_floats) {
        const int r1 = min(d.n_part, (grp + 1) * rpg);
#pragma unroll 4
        for (int r = grp * rpg; r < r1; ++r) acc += __ldcg(d.part + (int64_t)r * d.w_floats + q);
    }
    s_red[grp][ql] = acc;
    __syncthreads();
    if (threadIdx.x < DWR_Q && q < d.w_floats) {
        float v = 0.0f;
#pragma unroll
        for (int g2 = 0; g2 < DWR_G; ++g2) v += s_red[g2][ql];
        d.dw[q] += v;
        if (isnan(v)) {
            const int a = d.nn * d.nin, hid = a + (d.nh - 1) * d.nn * d.nn;
            const int start = q < a ? 0 : (q < hid ? a + ((q - a) / (d.nn * d.nn)) * d.nn * d.nn : hid);
            nan_mark(nan_state, d.woff + start);
        }
    }
}

template <int NF>
__global__ void __launch_bounds__(SC_THREADS, 1) scatter_kernel(const float *__restrict__ coords,
                                                                const float *__restrict__ dfeat, int64_t b,
                                                                int64_t stride,
                                                                const GridTables tab, int n_coarse, int coarse_floats,
                                                                float *__restrict__ grads,
                                                                const int64_t *__restrict__ nan_state,
                                                                int discard_dfeat, int rep_floats, int rep) {
    if (nan_halted(nan_state)) return;
    extern __shared__ float acc_s[];
    const uint64_t keep = l2_evict_last();
    // the most contended coarse levels (the first rep_floats accumulators: a 125-entry level 0
    // takes every sample's 8 corners) are replicated rep times, lane & (rep - 1) picking the copy,
    // which divides the collisions of the shared-memory CAS loops (fp32 shared atomics are CAS)
    const int rep_total = rep * rep_floats;
    const int smem_floats = rep_total + (coarse_floats - rep_floats);
    for (int q = threadIdx.x; q < smem_floats; q += SC_THREADS) acc_s[q] = 0.0f;
    __syncthreads();
    float *const acc_rep = acc_s + ((threadIdx.x & 31) & (rep - 1)) * rep_floats;
    // One item = one sample x SC_LG consecutive levels (level-group-major, so a
    // warp shares its level constants): the coordinates and the group's
    // dL/dfeat are loaded once up front and the group's REDs issue back to
    // back (fire-and-forget), which keeps many L2 reductions in flight.
    const int m = tab.n_levels;
    const int ngrp = (m + SC_LG - 1) / SC_LG;
    const int64_t items = b * ngrp;
    for (int64_t t = (int64_t)blockIdx.x * SC_THREADS + threadIdx.x; t < items; t += (int64_t)gridDim.x * SC_THREADS) {
        const int grp = (int)(t / b);
        const int64_t i = t - (int64_t)grp * b;
        const float px = __ldg(coords + 3 * i), py = __ldg(coords + 3 * i + 1), pz = __ldg(coords + 3 * i + 2);
        float dg[SC_LG][NF];
#pragma unroll
        for (int u = 0; u < SC_LG; ++u) {
            const int l = grp * SC_LG + u;
#pragma unroll
            for (int f = 0; f < NF; ++f) dg[u][f] = l < m ? __ldg(dfeat + (int64_t)(l * NF + f) * stride + i) : 0.0f;
        }
        if (discard_dfeat && (threadIdx.x & 31) == 0) {
            // the step's dL/dfeat scratch: this warp was the only reader of these lines
            // (32 consecutive samples of one level group, b % 32 == 0)
#pragma unroll
            for (int u = 0; u < SC_LG; ++u)
#pragma unroll
                for (int f = 0; f < NF; ++f)
                    if (grp * SC_LG + u < m) discard_l2(dfeat + (int64_t)((grp * SC_LG + u) * NF + f) * stride + i);
        }
#pragma unroll
        for (int u = 0; u < SC_LG; ++u) {
            const int l = grp * SC_LG + u;
            if (l >= m) break;
            const float *d = dg[u];
            const int32_t res = tab.res[l];
            const uint32_t r1 = (uint32_t)res + 1, mask = (uint32_t)(tab.entries[l] - 1);
            const bool dense = tab.dense[l] != 0;
            const Cell32 c = cell32(px, py, pz, res);
            if (l < n_coarse) {
                // shared-typed accumulators of the dense coarse levels
                const int o = (int)tab.offset[l];
                float *gs = o < rep_floats ? acc_rep + o : acc_s + rep_total + (o - rep_floats);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t slot = slot32(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), r1, mask,
                                                 dense);
                    const float w = cw32(c, k);
#pragma unroll
                    for (int f = 0; f < NF; ++f) atomicAdd(gs + (size_t)slot * NF + f, w * d[f]);
                }
                continue;
            }
            float *gl = grads + tab.offset[l];
            if constexpr (NF == 2) {
                // x-adjacent corner pairs in one aligned 16-byte entry pair go
                // out as a single float4 RED
                // entry pair {lo, lo+1} is 16-byte aligned iff (address of entry 0) / 8 + lo is even
                const uint32_t par = (uint32_t)((reinterpret_cast<uintptr_t>(gl) >> 3) & 1u);
#pragma unroll
                for (int k = 0; k < 8; k += 2) {
                    const uint32_t yo = (k >> 1) & 1, zo = (k >> 2) & 1;
                    const uint32_t s0 = slot32(c.cx, c.cy + yo, c.cz + zo, r1, mask, dense);
                    const uint32_t s1 = slot32(c.cx + 1, c.cy + yo, c.cz + zo, r1, mask, dense);
                    const float w0 = cw32(c, k), w1 = cw32(c, k + 1);
                    const uint32_t lo = min(s0, s1);
                    if (max(s0, s1) == lo + 1 && ((lo + par) & 1u) == 0u) {  // adjacent and 16-byte aligned
                        const float4 q = s0 == lo ? make_float4(w0 * d[0], w0 * d[1], w1 * d[0], w1 * d[1])
                                                  : make_float4(w1 * d[0], w1 * d[1], w0 * d[0], w0 * d[1]);
                        red_add4(gl + 2 * (size_t)lo, q, keep);
                    } else {
                        red_add2(gl + 2 * (size_t)s0, w0 * d[0], w0 * d[1], keep);
                        red_add2(gl + 2 * (size_t)s1, w1 * d[0], w1 * d[1], keep);
                    }
                }
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const uint32_t slot = slot32(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), r1, mask,
                                                 dense);
                    const float w = cw32(c, k);
                    float *g = gl + (size_t)slot * NF;
                    if constexpr (NF == 4 || NF == 8) {
#pragma unroll
                        for (int q = 0; q < NF / 4; ++q)
                            red_add4(g + 4 * q,
                                     make_float4(w * d[4 * q], w * d[4 * q + 1], w * d[4 * q + 2], w * d[4 * q + 3]),
                                     keep);
                    } else {
                        red_add(g, w * d[0], keep);
                    }
                }
            }
        }
    }
    __syncthreads();
    // coarse levels: one vector RED per 16-byte-aligned float quad per CTA (the flat
    // buffer may start 4/8/12 bytes past a 16-byte boundary: scalar head and tail)
    auto cval = [&](int q) -> float {  // the CTA's sum of coarse accumulator q (copies in a fixed order)
        if (q >= rep_floats) return acc_s[rep_total + (q - rep_floats)];
        float v = 0.0f;
        for (int c = 0; c < rep; ++c) v += acc_s[c * rep_floats + q];
        return v;
    };
    const int head = min(coarse_floats, (int)(((16 - (reinterpret_cast<uintptr_t>(grads) & 15)) & 15) >> 2));
    const int n4 = (coarse_floats - head) >> 2;
    for (int q = threadIdx.x; q < n4; q += SC_THREADS) {
        const int q0 = head + 4 * q;
        const float4 v = make_float4(cval(q0), cval(q0 + 1), cval(q0 + 2), cval(q0 + 3));
        if (v.x != 0.0f || v.y != 0.0f || v.z != 0.0f || v.w != 0.0f) red_add4(grads + q0, v, keep);
    }
    for (int q = threadIdx.x; q < head; q += SC_THREADS) red_add(grads + q, cval(q), keep);
    for (int q = head + 4 * n4 + threadIdx.x; q < coarse_floats; q += SC_THREADS) red_add(grads + q, cval(q), keep);
}

// ============================================================================ host side
// The batch is processed in `nchunks` row chunks on three streams so the
// L2-bound encode / scatter kernels of one chunk overlap the tensor-core
// MLP kernel of another (encode(c+1) || mlp(c) || scatter(c-1)); all of it
// is ordinary stream fork/join, so it captures into the step's CUDA graph.
constexpr int MAX_CHUNKS = 4;

struct TcPlan {
    TcShape sh;
    Tc4Shape sh4;
    bool v4;  // mlp_tc4_kernel (four slots, folded split-fp16 accumulator) takes this shape
    int grid_mlp, grid_sc, n_coarse, coarse_floats, nchunks, rep_floats, rep;
    size_t sc_smem() const { return (size_t)(rep * rep_floats + (coarse_floats - rep_floats)) * 4; }
    int64_t ntiles, chunk_tiles, off_x, off_dfeat, off_h, off_img, off_dwp, total;
    float lo_scale() const { return v4 ? 1.0f : tc::kLoScale; }
};

static bool mlp4_enabled() {
    static int on = -1;  // NVOL_MLP4=0 selects the two-slot mlp_tc_kernel (A/B measurements)
    if (on < 0) {
        const char *e = getenv("NVOL_MLP4");
        on = (e && e[0] == '0') ? 0 : 1;
    }
    return on == 1;
}

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
    p.v4 = mlp4_enabled() && build_shape4(p.sh4, tab.n_levels, tab.n_feat, nn, nh, relu_out, loss_kind);
    for (int l = 0; l < tab.n_levels; ++l)
        if (tab.entries[l] >= (1ll << 31)) return 0;
    const int sms = num_sms();
    p.ntiles = (b + TILE - 1) / TILE;
    // Row chunks on three streams (encode(c+1) || mlp(c) || scatter(c-1)).
    // Measured on B200 at cfg2: each kernel's cost is dominated by its fixed
    // per-launch latency (weight-image load, tail), so two half-size chunks
    // cost ~2x one full chunk; default is one chunk, NVOL_TRAIN_CHUNKS=n
    // (1..4) re-enables the overlap schedule.
    static int env_chunks = -1;
    if (env_chunks < 0) {
        const char *e = getenv("NVOL_TRAIN_CHUNKS");
        env_chunks = e ? atoi(e) : 1;
    }
    p.nchunks = env_chunks;
    p.nchunks = p.nchunks < 1 ? 1 : (p.nchunks > MAX_CHUNKS ? MAX_CHUNKS : p.nchunks);
    if (p.nchunks > p.ntiles) p.nchunks = (int)p.ntiles;
    p.chunk_tiles = (p.ntiles + p.nchunks - 1) / p.nchunks;
    p.nchunks = (int)((p.ntiles + p.chunk_tiles - 1) / p.chunk_tiles);  // every chunk non-empty
    p.grid_mlp = (int)(p.chunk_tiles < sms ? p.chunk_tiles : sms);
    p.grid_sc = sms;
    p.n_coarse = 0;
    p.coarse_floats = 0;
    static int max_coarse = -1;  // NVOL_SC_COARSE: cap on shared-memory levels (experiments)
    if (max_coarse < 0) {
        const char *e = getenv("NVOL_SC_COARSE");
        max_coarse = e ? atoi(e) : 64;
    }
    for (int l = 0; l < tab.n_levels && l < max_coarse; ++l) {
        int64_t end = tab.offset[l] + tab.entries[l] * tab.n_feat;
        if (!tab.dense[l] || end * 4 > (int64_t)COARSE_BYTES) break;
        p.n_coarse = l + 1;
        p.coarse_floats = (int)end;
    }
    // replicated coarse levels (NVOL_SC_REP copies of the first NVOL_SC_REP_LEVELS levels)
    static int rep_env = -1, rep_lv = -1;
    if (rep_env < 0) {
        const char *e = getenv("NVOL_SC_REP");
        const char *f = getenv("NVOL_SC_REP_LEVELS");
        rep_env = e ? atoi(e) : 4;
        rep_lv = f ? atoi(f) : 2;
        if (rep_env < 1) rep_env = 1;
        while (rep_env & (rep_env - 1)) rep_env &= rep_env - 1;  // power of two
        if (rep_env > 32) rep_env = 32;
    }
    p.rep = 1;
    p.rep_floats = 0;
    for (int l = 0; l < p.n_coarse && l < rep_lv; ++l) {
        const int end = (int)(tab.offset[l] + tab.entries[l] * tab.n_feat);
        if ((size_t)(rep_env * end + (p.coarse_floats - end)) * 4 > 200 * 1024) break;
        p.rep_floats = end;
        p.rep = rep_env;
    }
    auto al = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
    p.off_x = 0;
    p.off_dfeat = al(p.ntiles * TILE * p.sh.ninp * 4);  // hi + lo fp16 tiles
    p.off_h = p.off_dfeat + al(b * p.sh.nin * 4);      // mlp_tc4_kernel's activation scratch h_1..h_{nh-1}
    p.off_img = p.off_h + (p.v4 ? al(p.ntiles * (int64_t)(nh - 1) * p.sh4.h_tile_bytes) : 0);  // packed weights
    p.off_dwp = p.off_img + (p.v4 ? al(p.sh4.img_bytes) : 0);  // mlp_tc4_kernel's per-CTA dW partials
    p.total = p.off_dwp + (p.v4 ? al((int64_t)p.grid_mlp * p.sh4.w_floats * 4) : 0) + 256;
    return 1;
}

int64_t train_tc_workspace(int64_t b, int m, int n, int nn, int nh) {
    TcPlan p;
    if (!build_shape(p.sh, m, n, nn, nh, 1, 0)) return 0;
    const bool v4 = mlp4_enabled() && build_shape4(p.sh4, m, n, nn, nh, 1, 0);
    int64_t ntiles = (b + TILE - 1) / TILE;
    auto al = [](int64_t x) { return (x + 255) & ~(int64_t)255; };
    // (the same regions make_plan lays out; the dW partials sized for the largest MLP grid)
    return al(ntiles * TILE * p.sh.ninp * 4) + al(b * p.sh.nin * 4) +
           (v4 ? al(ntiles * (int64_t)(nh - 1) * p.sh4.h_tile_bytes) + al(p.sh4.img_bytes) +
                     al((int64_t)num_sms() * p.sh4.w_floats * 4)
               : 0) +
           256;
}

static cudaEvent_t g_stage_events[8];
// nvol_set_fork_event: recorded on the encoder's stream right after the step's encode launch, so a
// caller can start side work (the next step's sampling) beside the MLP instead of the encoder
static thread_local cudaEvent_t g_fork_event = nullptr;
// Parity hooks (nvol_train_tc_debug): the hot kernels additionally write the fp32 features
// (encode_tiles_kernel), the per-sample prediction (mlp_tc_kernel) and a copy of the
// feature-major dL/dfeat; all null in production.
struct TcDebug {
    float *feat = nullptr, *pred = nullptr, *dfeat = nullptr;
};
static TcDebug g_dbg;
static int g_stage_events_n = 0;

struct SideStreams {
    cudaStream_t enc = nullptr, sc = nullptr, pk = nullptr, red = nullptr;
    cudaEvent_t fork, join_enc, join_sc, enc_done[MAX_CHUNKS], mlp_done[MAX_CHUNKS], fork_pk, packed, fork_red,
        red_done;
};

static SideStreams &side_streams() {
    static SideStreams ss;
    if (ss.enc == nullptr) {
        cudaStreamCreateWithFlags(&ss.enc, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&ss.sc, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&ss.pk, cudaStreamNonBlocking);
        cudaStreamCreateWithFlags(&ss.red, cudaStreamNonBlocking);
        cudaEventCreateWithFlags(&ss.fork_red, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss.red_done, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss.fork_pk, cudaEventDisableTiming);
        cudaEventCreateWithFlags(&ss.packed, cudaEventDisableTiming);
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
                    double *loss_sum, void *workspace, int64_t ws_bytes, int flags, int64_t *nan_state,
                    cudaStream_t s) {
    TcPlan p;
    if (!make_plan(p, b, tab, nn, nh, relu_out, loss_kind)) {
        set_error("MLP / grid shape not supported by the tcgen05 path");
        return NVOL_EINVAL;
    }
    NVOL_REQUIRE(ws_bytes >= p.total, "workspace too small for the tcgen05 pipeline");
    uint8_t *ws = reinterpret_cast<uint8_t *>(workspace);
    uint8_t *xt = ws + p.off_x;
    float *dfeat = reinterpret_cast<float *>(ws + p.off_dfeat);
    int64_t enc = 0;
    for (int l = 0; l < tab.n_levels; ++l) enc = max(enc, tab.offset[l] + tab.entries[l] * tab.n_feat);
    const int64_t woff = flat_weight_offset(params, enc);
    int st = NVOL_OK;
    if (p.v4)
        cudaFuncSetAttribute(mlp_tc4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p.sh4.smem_bytes);
    else
        cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, p.sh.smem_bytes);
    const size_t csm = p.sc_smem();
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
    // flags: 16 = the tile buffer already holds this batch's encoding (written by
    // nvol_adam_encode_step), 32 = encode only
    const bool pre = (flags & 16) != 0, only = (flags & 32) != 0;
    const int nc = (prof || flags) ? 1 : p.nchunks;
    if (prof) cudaEventRecord(pev[0], s);
    SideStreams &ss = side_streams();
    cudaStream_t se = nc > 1 ? ss.enc : s, sc = nc > 1 ? ss.sc : s;
    if (p.v4 && !only) {
        // the step's packed MLP weight image (pack_w4), on a side stream beside the encode: 8 small
        // blocks in the shadow of the encoder kernel, joined before the MLP
        cudaEventRecord(ss.fork_pk, s);
        cudaStreamWaitEvent(ss.pk, ss.fork_pk, 0);
        pack_w4_kernel<<<PACK_BLOCKS, 256, 0, ss.pk>>>(params + woff, tab.n_levels * tab.n_feat, p.sh.ninp, nn, nh,
                                                      ws + p.off_img);
        cudaEventRecord(ss.packed, ss.pk);
    }
    if (nc > 1) {
        cudaEventRecord(ss.fork, s);
        cudaStreamWaitEvent(ss.enc, ss.fork, 0);
        cudaStreamWaitEvent(ss.sc, ss.fork, 0);
    }
    const int64_t tile_bytes = 2 * TILE * p.sh.ninp * 2;
    // one MLP launch (no chunking): its per-CTA dW partials are folded by the scatter's prologue
    // (NVOL_DW_PARTIALS=0: the MLP kernel REDs its dW into the gradient itself)
    static int dwp_env = -1;
    if (dwp_env < 0) {
        const char *e = getenv("NVOL_DW_PARTIALS");
        dwp_env = (e && e[0] == '0') ? 0 : 1;
    }
    DwPartials dwp{};
    if (p.v4 && nc == 1 && !only && dwp_env) {
        dwp.part = reinterpret_cast<const float *>(ws + p.off_dwp);
        dwp.dw = grads + woff;
        dwp.w_floats = (int)p.sh4.w_floats;
        dwp.nin = p.sh4.nin;
        dwp.nn = nn;
        dwp.nh = nh;
        dwp.woff = woff;
    }
    for (int c = 0; c < nc; ++c) {
        const int64_t t0 = c * p.chunk_tiles;
        const int64_t r0 = t0 * TILE;
        if (r0 >= b) break;
        const int64_t nb = (r0 + p.chunk_tiles * TILE < b ? p.chunk_tiles * TILE : b - r0);
        const unsigned egrid = grid_for(nb * tab.n_levels, 256);
        uint8_t *xtc = xt + t0 * tile_bytes;
        const float *cc = coords + 3 * r0;
        float *dfe = g_dbg.feat ? g_dbg.feat + r0 * (int64_t)tab.n_levels * tab.n_feat : nullptr;
        if (!pre) {
            if (nb % TILE)  // rows past the batch must be zero (0 x garbage could be NaN in dW)
                cudaMemsetAsync(xtc + (nb / TILE) * tile_bytes, 0, (size_t)tile_bytes, se);
            switch (tab.n_feat) {
                case 1: encode_tiles_kernel<1><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc, p.lo_scale(), dfe, nan_state); break;
                case 2: encode_tiles_kernel<2><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc, p.lo_scale(), dfe, nan_state); break;
                case 4: encode_tiles_kernel<4><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc, p.lo_scale(), dfe, nan_state); break;
                default: encode_tiles_kernel<8><<<egrid, 256, 0, se>>>(cc, nb, params, tab, p.sh.ninp, xtc, p.lo_scale(), dfe, nan_state); break;
            }
            st = check_launch("encode_tiles_kernel");
            if (st) return st;
        }
        if (c == 0 && g_fork_event) cudaEventRecord(g_fork_event, se);
        if (only) return NVOL_OK;
        if (nc > 1) {
            cudaEventRecord(ss.enc_done[c], se);
            cudaStreamWaitEvent(s, ss.enc_done[c], 0);
        }
        if (prof) cudaEventRecord(pev[1], s);
        const int64_t ct = (nb + TILE - 1) / TILE;
        const int gm = (int)(ct < p.grid_mlp ? ct : p.grid_mlp);
        if (p.v4) {
            const int64_t h_tile = (int64_t)(nh - 1) * p.sh4.h_tile_bytes;
            if (c == 0) cudaStreamWaitEvent(s, ss.packed, 0);  // the weight image (forked before the encode)
            static int nmw = -1;  // MMA-issuing warps (NVOL_MMA_WARPS=1: one issuer for all slots)
            if (nmw < 0) {
                const char *e = getenv("NVOL_MMA_WARPS");
                nmw = e ? atoi(e) : M4_MMA_WARPS;
                nmw = nmw < 1 ? 1 : (nmw > M4_MMA_WARPS ? M4_MMA_WARPS : nmw);
            }
            mlp_tc4_kernel<<<gm, (4 * M4_SLOTS + nmw) * 32, p.sh4.smem_bytes, s>>>(
                xtc, targets + r0, nb, 1.0 / (double)b_global, dscale, p.sh4, params + woff, loss_sum, dfeat + r0, b,
                grads + woff, ws + p.off_h + t0 * h_tile, g_dbg.pred ? g_dbg.pred + r0 : nullptr, nan_state, woff,
                ws + p.off_img, dwp.part ? const_cast<float *>(dwp.part) : nullptr);
            if (dwp.part) {  // the partials are folded beside the scatter (launched after it, below)
                dwp.n_part = gm;
                cudaEventRecord(ss.fork_red, s);
            }
        } else {
            mlp_tc_kernel<<<gm, PP_THREADS, p.sh.smem_bytes, s>>>(xtc, targets + r0, nb, 1.0 / (double)b_global, dscale,
                                                                  p.sh, params + woff, loss_sum, dfeat + r0, b,
                                                                  grads + woff, g_dbg.pred ? g_dbg.pred + r0 : nullptr,
                                                                  nan_state, woff);
        }
        st = check_launch("mlp_tc_kernel");
        if (st) return st;
        if (g_dbg.dfeat)
            cudaMemcpy2DAsync(g_dbg.dfeat + r0, (size_t)b * 4, dfeat + r0, (size_t)b * 4, (size_t)nb * 4,
                              (size_t)p.sh.nin, cudaMemcpyDeviceToDevice, s);
        if (nc > 1) {
            cudaEventRecord(ss.mlp_done[c], s);
            cudaStreamWaitEvent(sc, ss.mlp_done[c], 0);
        }
        if (prof) cudaEventRecord(pev[2], s);
        switch (tab.n_feat) {
#define LAUNCH_SC(NFV)                                                                                             \
    case NFV:                                                                                                      \
        scatter_kernel<NFV><<<p.grid_sc, SC_THREADS, csm, sc>>>(cc, dfeat + r0, nb, b, tab, p.n_coarse,            \
                                                                p.coarse_floats, grads, nan_state,             \
                                                                (nb % 32 == 0 && b % 32 == 0) ? 1 : 0,         \
                                                                p.rep_floats, p.rep);                          \
        break;
            LAUNCH_SC(1)
            LAUNCH_SC(2)
            LAUNCH_SC(4)
            LAUNCH_SC(8)
#undef LAUNCH_SC
        }
        st = check_launch("scatter_kernel");
        if (st) return st;
        if (dwp.part) {
            // after the scatter's launch, so its one-per-SM CTAs are placed first and the small
            // reduction CTAs fill the registers they leave free
            cudaStreamWaitEvent(ss.red, ss.fork_red, 0);
            dw_reduce_kernel<<<(unsigned)((dwp.w_floats + DWR_Q - 1) / DWR_Q), DWR_Q * DWR_G, 0, ss.red>>>(dwp,
                                                                                                  nan_state);
            st = check_launch("dw_reduce_kernel");
            if (st) return st;
            cudaEventRecord(ss.red_done, ss.red);
            cudaStreamWaitEvent(s, ss.red_done, 0);  // the weight gradient is complete
        }
        if (prof) cudaEventRecord(pev[3], s);
    }
    if (nc > 1) {
        cudaEventRecord(ss.join_enc, ss.enc);
        cudaEventRecord(ss.join_sc, ss.sc);
        cudaStreamWaitEvent(s, ss.join_enc, 0);
        cudaStreamWaitEvent(s, ss.join_sc, 0);
    }
    return NVOL_OK;
}

}  // namespace nvol

extern "C" int nvol_set_fork_event(void *event) {
    nvol::g_fork_event = reinterpret_cast<cudaEvent_t>(event);
    return NVOL_OK;
}

// Profiling hook: with >= 4 events set, nvol_train_fwd_bwd (mode 1) runs as a
// single chunk on the caller's stream and records events[0..3] before encode,
// after encode, after pack+MLP and after scatter.  n = 0 disables.
extern "C" int nvol_set_stage_events(void *const *events, int32_t n) {
    n = n > 8 ? 8 : (n < 0 ? 0 : n);
    for (int i = 0; i < n; ++i) nvol::g_stage_events[i] = reinterpret_cast<cudaEvent_t>(events[i]);
    nvol::g_stage_events_n = n;
    return NVOL_OK;
}

#ifdef NVOL_TIMELINE
extern "C" int nvol_debug_timeline(unsigned long long *host, int32_t n) {
    cudaDeviceSynchronize();
    return cudaMemcpyFromSymbol(host, nvol::g_tl, sizeof(unsigned long long) * (n > 4096 ? 4096 : n)) == cudaSuccess
               ? 0 : 2;
}
#endif

extern "C" int nvol_train_tc_debug(float *feat, float *pred, float *dfeat) {
    nvol::g_dbg.feat = feat;
    nvol::g_dbg.pred = pred;
    nvol::g_dbg.dfeat = dfeat;
    return NVOL_OK;
}

// The training step's encoder-backward kernel (scatter_kernel) on its own, fed a
// caller-provided feature-major dL/dfeat [n_levels*n_feat][stride] -- exactly the
// launch nvol_train_fwd_bwd (mode 1) makes after the MLP.
extern "C" int nvol_train_tc_scatter(const float *coords, const float *dfeat, int64_t b, int64_t stride,
                                     const int64_t *level_off, const int64_t *level_res,
                                     const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels,
                                     int32_t n_feat, float *grads, void *stream) {
    using namespace nvol;
    NVOL_REQUIRE(coords && dfeat && grads && b >= 1 && stride >= b, "bad arguments");
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    TcPlan p;
    // the scatter's coarse-level plan does not depend on the MLP shape: any supported one
    if (!make_plan(p, b, tab, 64, 1, 1, 0) && !make_plan(p, b, tab, 16, 1, 1, 0)) {
        set_error("grid shape not supported by the tcgen05 path");
        return NVOL_EINVAL;
    }
    const size_t csm = p.sc_smem();
    cudaStream_t s = as_stream(stream);
    switch (n_feat) {
#define LAUNCH_SC1(NFV)                                                                                          \
    case NFV:                                                                                                    \
        cudaFuncSetAttribute(scatter_kernel<NFV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);        \
        scatter_kernel<NFV><<<p.grid_sc, SC_THREADS, csm, s>>>(coords, dfeat, b, stride, tab, p.n_coarse,      \
                                                               p.coarse_floats, grads, nullptr, 0, p.rep_floats, \
                                                               p.rep);                                          \
        break;
        LAUNCH_SC1(1)
        LAUNCH_SC1(2)
        LAUNCH_SC1(4)
        LAUNCH_SC1(8)
#undef LAUNCH_SC1
        default: set_error("n_feat must be 1, 2, 4 or 8"); return NVOL_EINVAL;
    }
    return check_launch("scatter_kernel");
}

extern "C" int64_t nvol_l2_persist(int64_t bytes) {
    int dev = 0, maxp = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev);
    size_t want = (size_t)(bytes < 0 ? 0 : bytes);
    if (want > (size_t)maxp) want = (size_t)maxp;
    if (cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want) != cudaSuccess) {
        cudaGetLastError();
        return -1;
    }
    size_t got = 0;
    cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize);
    return (int64_t)got;
}

extern "C" int nvol_train_tc_supported(int32_t n_levels, int32_t n_feat, int32_t n_neurons, int32_t n_hidden) {
    nvol::TcShape sh;
    return nvol::build_shape(sh, n_levels, n_feat, n_neurons, n_hidden, 1, 0) ? 1 : 0;
}

extern "C" int nvol_has_tcgen05(int device) {
    int major = 0, minor = 0;
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
    cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, device);
    return major == 10 && minor == 0;
}

// Step tail fused with the next step's encoder forward (adam_encode_kernel):
// nvol_adam_train_step's update + bookkeeping, and the encoding of next_coords
// into the tcgen05 tile buffer of `workspace`, so the next
// nvol_train_fwd_bwd(mode 1 | NVOL_TRAIN_PREENCODED) skips its encode kernel.
extern "C" int nvol_adam_encode_step(float *p, float *g, float *m, float *v, int64_t n, const float *sched,
                                     int64_t sched_len, int64_t *step_counter, float beta1, float one_minus_beta1,
                                     float beta2, float one_minus_beta2, float eps, float l2, int64_t *nan_state,
                                     double *loss_acc, double *losses, int64_t t0, int64_t cap, double inv_b,
                                     uint32_t *work, const float *next_coords, int64_t b, const int64_t *level_off,
                                     const int64_t *level_res, const int64_t *level_entries,
                                     const uint8_t *level_dense, int32_t n_levels, int32_t n_feat, int32_t n_neurons,
                                     int32_t n_hidden, void *workspace, int64_t workspace_bytes, void *stream) {
    using namespace nvol;
    NVOL_REQUIRE(p && g && m && v && sched && step_counter && work && sched_len >= 1, "null pointer");
    NVOL_REQUIRE(next_coords && workspace && b >= 1, "null pointer");
    NVOL_REQUIRE(((uintptr_t)p & 127) == ((uintptr_t)g & 127) && ((uintptr_t)p & 127) == ((uintptr_t)m & 127) &&
                     ((uintptr_t)p & 127) == ((uintptr_t)v & 127) && ((uintptr_t)p & 3) == 0,
                 "flat Adam buffers must share their alignment modulo 128 bytes");
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    TcPlan pl;
    if (!make_plan(pl, b, tab, n_neurons, n_hidden, 1, 0)) {
        set_error("MLP / grid shape not supported by the tcgen05 path");
        return NVOL_EINVAL;
    }
    NVOL_REQUIRE(workspace_bytes >= pl.total, "workspace too small for the tcgen05 pipeline");
    for (int l = 0; l < n_levels; ++l)
        NVOL_REQUIRE(level_off[l] >= 0 && level_off[l] + level_entries[l] * n_feat <= n, "table outside the flat buffer");
    cudaStream_t s = as_stream(stream);
    uint8_t *xt = reinterpret_cast<uint8_t *>(workspace) + pl.off_x;
    const int64_t tile_bytes = 2 * TILE * pl.sh.ninp * 2;
    if (b % TILE) cudaMemsetAsync(xt + (b / TILE) * tile_bytes, 0, (size_t)tile_bytes, s);
    AdamArgs a{p,    g,    m,    v,        n,        sched,  sched_len, step_counter, beta1, one_minus_beta1,
               beta2, one_minus_beta2, eps, l2, nan_state, loss_acc, losses, t0, cap, inv_b};
    // flat layout: scalar head up to the next 128-byte boundary, float4 body in warp chunks, scalar tail
    const int64_t head = std::min(n, (int64_t)(((128 - ((uintptr_t)p & 127)) & 127) >> 2));
    const int64_t n4 = (n - head) >> 2;
    const int64_t nch = std::max((int64_t)1, (n4 + AE_WARP_F4 - 1) / AE_WARP_F4);
    auto chunk_of = [&](int64_t idx) -> int64_t {
        return idx < head ? 0 : std::min((idx - head) / (4 * AE_WARP_F4), nch - 1);
    };
    NVOL_REQUIRE(nch < (1ll << 31), "flat buffer too large");
    LevelChunks lc;
    for (int l = 0; l < n_levels; ++l) {
        lc.lo[l] = (int32_t)chunk_of(level_off[l]);
        lc.hi[l] = (int32_t)chunk_of(level_off[l] + level_entries[l] * n_feat - 1);
    }
    auto launch = [&](auto kern) {
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, AE_THREADS, 0);
        if (per_sm < 1) per_sm = 1;
        kern<<<per_sm * num_sms(), AE_THREADS, 0, s>>>(a, head, n4, nch, lc, next_coords, b, tab, pl.sh.ninp, xt, work,
                                                       pl.lo_scale());
    };
    switch (n_feat) {
        case 1: launch(adam_encode_kernel<1>); break;
        case 2: launch(adam_encode_kernel<2>); break;
        case 4: launch(adam_encode_kernel<4>); break;
        default: launch(adam_encode_kernel<8>); break;
    }
    return check_launch("adam_encode_kernel");
}
