// tcgen05 field inference: fused encode + MLP forward for decode and render.
//
// Reference: trainer.py:80-106 (decode: Phi at voxel centres, denormalised)
// and _kernels.py:154-176 / model.py:178-198 (batched Phi evaluation, the
// renderers' phi_eval_staged, _render_kernels.py:518-540).
// Persistent CTAs (two per SM, 128 TMEM columns each) walk 128-sample tiles:
// bit-exact fp32 hash-grid encode -> split-fp16 (hi + lo) feature tiles in
// smem -> per hidden layer one tcgen05.mma chain (hi*hi into one TMEM
// accumulator, lo*hi + hi*lo into a second, see tc.cuh) -> ReLU epilogue
// re-splitting the activations -> output layer on CUDA cores (fp32).  The
// split forward keeps outputs within the north-star 1e-2 relative bar even
// where plain fp16 rounding flips ReLU masks; the exact evaluator
// (field.cu) remains available as infer_mode "exact".
#include <cuda_fp16.h>

#include <cstdlib>

#include "common.cuh"
#include "infer_tile.cuh"
#include "tc.cuh"

namespace nvol {

template <int NF, bool PAIR>
__global__ void __launch_bounds__(IT_THREADS, 2) infer_tc_kernel(
    const float *__restrict__ coords, int64_t b, const float *__restrict__ params, const GridTables tab,
    const InferShape sh, const uint8_t *__restrict__ wimg, int decode, int64_t dx, int64_t dy, int64_t dz, int64_t z0,
    double lo, double scale, float *__restrict__ out, const int32_t *__restrict__ b_dev) {
    if (b_dev) b = *b_dev;  // sample count produced on the device (render loop), b was its upper bound
    if ((int64_t)blockIdx.x * IT_TILE >= b) return;  // no tile for this CTA: skip the weight load / TMEM
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    infer_prologue(smem, sh, wimg, &mbar, &tmem_base_sh);
    const int s = threadIdx.x & (IT_TILE - 1), h = threadIdx.x >> 7;
    const uint32_t tmem = tmem_base_sh;
    uint32_t phase = 0;
    const int64_t ntiles = (b + IT_TILE - 1) / IT_TILE;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t i = tile * IT_TILE + s;
        const bool valid = i < b;
        float x = 0.f, y = 0.f, z = 0.f;
        if (valid) {
            if (decode) {
                int64_t ix = i % dx, iy = (i / dx) % dy, iz = z0 + i / (dx * dy);
                x = xdiv(xadd((float)ix, 0.5f), (float)dx);
                y = xdiv(xadd((float)iy, 0.5f), (float)dy);
                z = xdiv(xadd((float)iz, 0.5f), (float)dz);
            } else {
                x = coords[3 * i];
                y = coords[3 * i + 1];
                z = coords[3 * i + 2];
            }
        }
        const float o = infer_tile<NF, PAIR>(smem, sh, tab, params, x, y, z, valid, tmem, &mbar, phase);
        if (h == 0 && valid) out[i] = decode ? (float)__dadd_rn(__dmul_rn((double)o, scale), lo) : o;
    }
    infer_teardown(tmem, sh);
}

int pack_mlp_image(const float *wflat, int nin, int ninp, int nn, int nh, const uint32_t *o_w, uint32_t o_wout,
                   uint8_t *image, cudaStream_t s, const uint32_t *o_wlo);

int infer_tc_launch(const float *coords, int64_t b, const float *params, const GridTables &tab, const float *wflat,
                    uint8_t *wimg, int nn, int nh, int relu_out, int decode, int64_t dx, int64_t dy, int64_t dz,
                    int64_t z0, double lo, double scale, float *out, cudaStream_t s, bool pack = true,
                    const int32_t *b_dev = nullptr) {
    InferShape sh;
    if (!build_infer_shape(sh, tab.n_levels, tab.n_feat, nn, nh, relu_out)) {
        set_error("MLP shape not supported by the tcgen05 inference path");
        return NVOL_EINVAL;
    }
    for (int l = 0; l < tab.n_levels; ++l)
        NVOL_REQUIRE(tab.entries[l] < (1ll << 31), "level too large for the tcgen05 inference path");
    NVOL_REQUIRE(wimg, "tcgen05 inference needs an mlp_image scratch buffer (nvol_mlp_image_bytes)");
    if (pack) {  // callers that launch repeatedly on unchanged weights (the render loop) pack once
        int st = pack_mlp_image(wflat, sh.nin, sh.ninp, nn, nh, sh.o_w, sh.o_wout, wimg, s, sh.o_wlo);
        if (st) return st;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t ntiles = (b + IT_TILE - 1) / IT_TILE;
    int64_t cap = (int64_t)sms * 2;
    int grid = (int)(ntiles < cap ? ntiles : cap);
    if (grid < 1) return NVOL_OK;
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem_bytes);
        kern<<<grid, IT_THREADS, sh.smem_bytes, s>>>(coords, b, params, tab, sh, wimg, decode, dx, dy, dz, z0, lo,
                                                     scale, out, b_dev);
    };
    switch (tab.n_feat) {
        case 1: decode ? go(infer_tc_kernel<1, false>) : go(infer_tc_kernel<1, true>); break;
        case 2: decode ? go(infer_tc_kernel<2, false>) : go(infer_tc_kernel<2, true>); break;
        case 4: decode ? go(infer_tc_kernel<4, false>) : go(infer_tc_kernel<4, true>); break;
        default: decode ? go(infer_tc_kernel<8, false>) : go(infer_tc_kernel<8, true>); break;
    }
    return check_launch("infer_tc_kernel");
}

static int mlp_dims(const int32_t *widths, int32_t n_layers, const GridTables &tab, int &nn, int &nh) {
    NVOL_REQUIRE(n_layers >= 2 && widths[n_layers] == 1, "MLP must have >= 1 hidden layer and output width 1");
    NVOL_REQUIRE(widths[0] == tab.n_levels * tab.n_feat, "MLP input width != encoder width");
    nn = widths[1];
    for (int i = 1; i < n_layers; ++i) NVOL_REQUIRE(widths[i] == nn, "tcgen05 path needs a uniform hidden width");
    nh = n_layers - 1;
    return NVOL_OK;
}

int nvol_decode_tc(const float *params, const GridTables &tab, const float *weights, const int32_t *widths,
                   int32_t n_layers, int32_t relu_out, int64_t dx, int64_t dy, int64_t dz, int64_t z0, int64_t nz,
                   double lo, double scale, float *out, void *mlp_image, cudaStream_t s) {
    int nn, nh;
    int st = mlp_dims(widths, n_layers, tab, nn, nh);
    if (st) return st;
    return infer_tc_launch(nullptr, dx * dy * nz, params, tab, weights, (uint8_t *)mlp_image, nn, nh, relu_out, 1, dx,
                           dy, dz, z0, lo, scale, out, s);
}

}  // namespace nvol

using namespace nvol;

extern "C" int64_t nvol_mlp_image_bytes(int32_t n_levels, int32_t n_feat, int32_t n_neurons, int32_t n_hidden) {
    InferShape sh;
    if (!build_infer_shape(sh, n_levels, n_feat, n_neurons, n_hidden, 1)) return 0;
    return sh.o_x;
}

extern "C" int nvol_field_eval_tc(const float *coords, int64_t b, const float *params, const int64_t *level_off,
                                  const int64_t *level_res, const int64_t *level_entries,
                                  const uint8_t *level_dense, int32_t n_levels, int32_t n_feat,
                                  const float *weights, const int32_t *widths, int32_t n_layers, int32_t relu_out,
                                  void *mlp_image, float *out, void *stream) {
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    if (b == 0) return NVOL_OK;
    NVOL_REQUIRE(coords && params && weights && widths && out, "null pointer");
    int nn, nh;
    st = mlp_dims(widths, n_layers, tab, nn, nh);
    if (st) return st;
    return infer_tc_launch(coords, b, params, tab, weights, (uint8_t *)mlp_image, nn, nh, relu_out, 0, 0, 0, 0, 0, 0.0,
                           1.0, out, as_stream(stream));
}
