// Exact fused field evaluation (encode + MLP per sample) and full-grid decode.
//
// Reference: _kernels.py:95-176 (_mlp_row, _field_one, field_eval_model ==
// NeuralModel.eval_fused, model.py:184-198) and trainer.py:80-106 (decode).
// One thread per sample, float32 throughout, each dot product folded in k
// order without FMA contraction: bit-identical to the reference's numba
// evaluator.  Weights are staged once per CTA in shared memory, transposed
// (k-major) so the inner j loop reads a broadcast float4.
#include "common.cuh"
#include "field_exact.cuh"

namespace nvol {


// mode: 0 = explicit coords, 1 = decode brick (voxel centres of rows [z0, z0+nz)).
template <int NN>
__global__ void __launch_bounds__(FE_THREADS) field_exact_kernel(
    const float *__restrict__ coords, int64_t b, const float *__restrict__ params, const GridTables tab,
    const float *__restrict__ weights, const MlpShape sh, int decode, int64_t dx, int64_t dy, int64_t dz,
    int64_t z0, double lo, double scale, float *__restrict__ out, int maxw) {
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    // transposed weights: layer li occupies widths[li]*widths[li+1] floats, k-major
    int wtotal = 0;
    for (int li = 0; li < sh.n_layers; ++li) wtotal += sh.widths[li] * sh.widths[li + 1];
    float *wt = smem;
    {
        const float *src = weights;
        float *dst = wt;
        for (int li = 0; li < sh.n_layers; ++li) {
            int win = sh.widths[li], wout = sh.widths[li + 1];
            for (int q = threadIdx.x; q < win * wout; q += blockDim.x) {
                int j = q / win, k = q % win;  // src row-major (j, k)
                dst[k * wout + j] = src[q];
            }
            src += win * wout;
            dst += win * wout;
        }
    }
    float *h0 = wt + ((wtotal + 3) & ~3);
    float *h1 = h0 + maxw * FE_THREADS;
    __syncthreads();
    for (int64_t base = (int64_t)blockIdx.x * FE_THREADS; base < b; base += (int64_t)gridDim.x * FE_THREADS) {
        int64_t i = base + threadIdx.x;
        if (i >= b) continue;
        float x, y, z;
        if (decode) {
            int64_t ix = i % dx, iy = (i / dx) % dy, iz = z0 + i / (dx * dy);
            if (decode == 2) {  // macrocell.py:90-94: centres in float64, then cast
                x = (float)(((double)ix + 0.5) / (double)dx);
                y = (float)(((double)iy + 0.5) / (double)dy);
                z = (float)(((double)iz + 0.5) / (double)dz);
            } else {            // trainer.py:86-92: float32 arithmetic
                x = xdiv(xadd((float)ix, 0.5f), (float)dx);
                y = xdiv(xadd((float)iy, 0.5f), (float)dy);
                z = xdiv(xadd((float)iz, 0.5f), (float)dz);
            }
        } else {
            x = coords[3 * i];
            y = coords[3 * i + 1];
            z = coords[3 * i + 2];
        }
        float *col0 = h0 + threadIdx.x, *col1 = h1 + threadIdx.x;
        encode_exact(x, y, z, params, tab, col0);
        float v;
        if constexpr (NN > 0) {
            v = mlp_exact_reg<NN>(col0, tab.n_levels * tab.n_feat, wt, sh);
        } else {
            v = mlp_exact_smem(col0, col1, wt, sh);
        }
        if (decode == 1)
            out[i] = (float)__dadd_rn(__dmul_rn((double)v, scale), lo);
        else
            out[i] = v;
    }
}

template <int NN>
__global__ void __launch_bounds__(FE_THREADS, 4) field_exact_col_kernel(
    const float *__restrict__ coords, int64_t b, const float *__restrict__ params, const GridTables tab,
    const float *__restrict__ wt, const MlpShape sh, int decode, int64_t dx, int64_t dy, int64_t dz, int64_t z0,
    double lo, double scale, float *__restrict__ out) {
    extern __shared__ float4 smem4[];
    float *col = reinterpret_cast<float *>(smem4) + threadIdx.x;
    for (int64_t base = (int64_t)blockIdx.x * FE_THREADS; base < b; base += (int64_t)gridDim.x * FE_THREADS) {
        const int64_t i = base + threadIdx.x;
        if (i >= b) continue;
        float x, y, z;
        if (decode) {
            int64_t ix = i % dx, iy = (i / dx) % dy, iz = z0 + i / (dx * dy);
            if (decode == 2) {  // macrocell.py:90-94: centres in float64, then cast
                x = (float)(((double)ix + 0.5) / (double)dx);
                y = (float)(((double)iy + 0.5) / (double)dy);
                z = (float)(((double)iz + 0.5) / (double)dz);
            } else {            // trainer.py:86-92: float32 arithmetic
                x = xdiv(xadd((float)ix, 0.5f), (float)dx);
                y = xdiv(xadd((float)iy, 0.5f), (float)dy);
                z = xdiv(xadd((float)iz, 0.5f), (float)dz);
            }
        } else {
            x = coords[3 * i];
            y = coords[3 * i + 1];
            z = coords[3 * i + 2];
        }
        encode_exact(x, y, z, params, tab, col);
        const float v = mlp_exact_col<NN, true>(col, tab.n_levels * tab.n_feat, wt, sh);
        if (decode == 1)
            out[i] = (float)__dadd_rn(__dmul_rn((double)v, scale), lo);
        else
            out[i] = v;
    }
}

// row-major (out x in) layers -> k-major (in x out), layer by layer
__global__ void transpose_layers_kernel(const float *__restrict__ w, const MlpShape sh, float *__restrict__ wt) {
    int off = 0;
    for (int li = 0; li < sh.n_layers; ++li) {
        const int win = sh.widths[li], wout = sh.widths[li + 1];
        for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < win * wout; q += gridDim.x * blockDim.x) {
            const int j = q / win, k = q % win;
            wt[off + k * wout + j] = w[off + q];
        }
        off += win * wout;
    }
}

int field_exact_launch(const float *coords, int64_t b, const float *params, const GridTables &tab,
                       const float *weights, const int32_t *widths, int32_t n_layers, int32_t relu_out,
                       int decode, int64_t dx, int64_t dy, int64_t dz, int64_t z0, double lo, double scale,
                       float *out, cudaStream_t s) {
    NVOL_REQUIRE(n_layers >= 1 && n_layers <= 11, "MLP depth out of range");
    MlpShape sh;
    sh.n_layers = n_layers;
    sh.relu_out = relu_out ? 1 : 0;
    int maxw = 0, wtotal = 0;
    for (int i = 0; i <= n_layers; ++i) {
        sh.widths[i] = widths[i];
        maxw = max(maxw, (int)widths[i]);
    }
    for (int i = 0; i < n_layers; ++i) wtotal += widths[i] * widths[i + 1];
    NVOL_REQUIRE(widths[0] == tab.n_levels * tab.n_feat, "MLP input width != encoder width");
    NVOL_REQUIRE(widths[n_layers] == 1, "output width must be 1");
    // register path: uniform hidden width NN in {16,32,64}
    int nn = n_layers >= 2 ? widths[1] : 0;
    bool uniform = n_layers >= 2;
    for (int i = 1; i < n_layers; ++i) uniform &= widths[i] == nn;
    // the register path (uniform NN) keeps only the feature columns in shared memory: 3 CTAs / SM at cfg2
    // instead of 1 with the generic path's two maxw-wide ping-pong columns
    const bool regpath = uniform && (nn == 16 || nn == 32 || nn == 64);
    size_t smem = sizeof(float) * (((wtotal + 3) & ~3) + (regpath ? (size_t)widths[0] : 2 * (size_t)maxw) * FE_THREADS);
    NVOL_REQUIRE(smem <= 220 * 1024, "MLP too large for the exact evaluator");
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (b + FE_THREADS - 1) / FE_THREADS;
    unsigned grid = (unsigned)max((int64_t)1, min(blocks, (int64_t)sms * 16));
    if (regpath && widths[0] <= nn) {
        // column kernel: per-thread activation columns in shared memory, k-major weights via L1
        // transposed-weight scratch: grow-only, per host thread and device (a per-call
        // stream-ordered allocation went back to the driver at every host sync of the
        // render loop and cost milliseconds)
        struct WtScratch {
            float *p = nullptr;
            size_t n = 0;
        };
        static thread_local WtScratch scratch[64];
        NVOL_REQUIRE(dev >= 0 && dev < 64, "device index out of range");
        WtScratch &ws = scratch[dev];
        if (ws.n < (size_t)wtotal) {
            if (ws.p) {
                cudaStreamSynchronize(s);  // the previous scratch may still be read by queued work
                cudaFree(ws.p);
            }
            ws.p = nullptr;
            ws.n = 0;
            if (cudaMalloc((void **)&ws.p, sizeof(float) * (size_t)wtotal) != cudaSuccess)
                return check_launch("exact evaluator weights");
            ws.n = (size_t)wtotal;
        }
        float *wt = ws.p;
        transpose_layers_kernel<<<16, 256, 0, s>>>(weights, sh, wt);
        const size_t csm = sizeof(float) * (size_t)nn * FE_THREADS;
        auto go = [&](auto kern) {
            cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)csm);
            cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 60);
            kern<<<grid, FE_THREADS, csm, s>>>(coords, b, params, tab, wt, sh, decode, dx, dy, dz, z0, lo, scale, out);
        };
        if (nn == 16) go(field_exact_col_kernel<16>);
        else if (nn == 32) go(field_exact_col_kernel<32>);
        else go(field_exact_col_kernel<64>);
        return check_launch("field_eval_exact");
    }
#define LAUNCH_FE(NNV)                                                                                      \
    do {                                                                                                    \
        cudaFuncSetAttribute(field_exact_kernel<NNV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
        field_exact_kernel<NNV><<<grid, FE_THREADS, smem, s>>>(coords, b, params, tab, weights, sh, decode, dx, \
                                                               dy, dz, z0, lo, scale, out, maxw);           \
    } while (0)
    if (uniform && nn == 16)
        LAUNCH_FE(16);
    else if (uniform && nn == 32)
        LAUNCH_FE(32);
    else if (uniform && nn == 64)
        LAUNCH_FE(64);
    else
        LAUNCH_FE(0);
#undef LAUNCH_FE
    return check_launch("field_eval_exact");
}

int nvol_decode_tc(const float *params, const GridTables &tab, const float *weights, const int32_t *widths,
                   int32_t n_layers, int32_t relu_out, int64_t dx, int64_t dy, int64_t dz, int64_t z0,
                   int64_t nz, double lo, double scale, float *out, void *mlp_image, cudaStream_t s);

}  // namespace nvol

using namespace nvol;

extern "C" {

int nvol_field_eval_exact(const float *coords, int64_t b, const float *params, const int64_t *level_off,
                          const int64_t *level_res, const int64_t *level_entries, const uint8_t *level_dense,
                          int32_t n_levels, int32_t n_feat, const float *weights, const int32_t *widths,
                          int32_t n_layers, int32_t relu_out, float *out, void *stream) {
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    if (b == 0) return NVOL_OK;
    NVOL_REQUIRE(coords && params && weights && widths && out, "null pointer");
    return field_exact_launch(coords, b, params, tab, weights, widths, n_layers, relu_out, 0, 0, 0, 0, 0, 0.0,
                              1.0, out, as_stream(stream));
}

int nvol_decode(const float *params, const int64_t *level_off, const int64_t *level_res,
                const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels, int32_t n_feat,
                const float *weights, const int32_t *widths, int32_t n_layers, int32_t relu_out, int64_t dx,
                int64_t dy, int64_t dz, int64_t z0, int64_t nz, double lo, double hi, float *out, int32_t mode,
                void *mlp_image, void *stream) {
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    NVOL_REQUIRE(dx >= 1 && dy >= 1 && dz >= 1 && z0 >= 0 && nz >= 0 && z0 + nz <= dz, "bad decode brick");
    NVOL_REQUIRE(params && weights && widths && out, "null pointer");
    if (nz == 0) return NVOL_OK;
    double scale = hi - lo;
    if (mode == 1) return nvol_decode_tc(params, tab, weights, widths, n_layers, relu_out, dx, dy, dz, z0, nz, lo,
                                         scale, out, mlp_image, as_stream(stream));
    // mode 0: trainer.decode semantics (float32 centres, denormalised);
    // mode 2: macrocell_from_model semantics (float64 centres, raw Phi)
    return field_exact_launch(nullptr, dx * dy * nz, params, tab, weights, widths, n_layers, relu_out,
                              mode == 2 ? 2 : 1, dx, dy, dz, z0, lo, scale, out, as_stream(stream));
}

}  // extern "C"
