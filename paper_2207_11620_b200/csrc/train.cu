// Training step forward + backward over a flat parameter buffer.
//
// Reference: model.py:154-174 NeuralModel.train_step = encode (_kernels.py:31)
// -> Mlp.forward (network.py:61) -> loss_and_grad (network.py:96) ->
// Mlp.backward (network.py:76) -> grid_encode_bwd (_kernels.py:82); Adam is
// launched separately (nvol_adam_flat_dev) so a data-parallel caller can
// all-reduce the gradient buffer in between.
//
// mode 0 composes the generic kernels (SIMT fp32); mode 1 is the fused
// tcgen05 tile pipeline in train_tc.cu.
#include "common.cuh"

namespace nvol {

struct Ws {
    char *p;
    int64_t used;
    template <typename T>
    T *take(int64_t n) {
        T *r = reinterpret_cast<T *>(p + used);
        used += ((n * (int64_t)sizeof(T)) + 255) & ~(int64_t)255;
        return r;
    }
};

static int64_t ws_simt(int64_t b, int m, int n, int nn, int nh) {
    Ws w{nullptr, 0};
    int maxw = max(m * n, nn);
    w.take<float>(b * m * n);           // feats
    for (int i = 0; i < nh; ++i) w.take<float>(b * nn);  // hidden activations
    w.take<float>(b);                   // pred
    w.take<float>(b);                   // dl/dpred
    w.take<float>(b * maxw);            // scratch 0
    w.take<float>(b * maxw);            // scratch 1
    w.take<float>(b * m * n);           // dl/dfeat
    return w.used;
}

int train_tc_launch(const float *coords, const float *targets, int64_t b, int64_t b_global, const float *params,
                    float *grads, const GridTables &tab, int nn, int nh, int relu_out, int loss_kind,
                    double *loss_sum, void *workspace, int64_t ws_bytes, int flags, int64_t *nan_state,
                    cudaStream_t s);
int64_t train_tc_workspace(int64_t b, int m, int n, int nn, int nh);

// [b][w] -> [w][b] (the hot scatter reads dL/dfeat feature-major)
__global__ void transpose_kernel(const float *__restrict__ in, float *__restrict__ out, int64_t b, int w) {
    __shared__ float t[32][33];
    const int64_t r0 = (int64_t)blockIdx.x * 32;
    const int c0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int64_t r = r0 + k;
        const int c = c0 + threadIdx.x;
        t[k][threadIdx.x] = (r < b && c < w) ? in[r * w + c] : 0.0f;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int c = c0 + k;
        const int64_t r = r0 + threadIdx.x;
        if (c < w && r < b) out[(int64_t)c * b + r] = t[threadIdx.x][k];
    }
}

}  // namespace nvol

using namespace nvol;

extern "C" {

int nvol_loss_and_grad_scaled(const void *, const void *, int64_t, int64_t, int32_t, void *, double *, int32_t,
                              void *);
int nvol_mlp_forward(int64_t, int32_t, const int32_t *, const void *const *, void *const *, int32_t, int32_t, void *);
int nvol_mlp_backward(int64_t, int32_t, const int32_t *, const void *const *, const void *const *, const void *,
                      void *const *, void *, void *, void *, int32_t, int32_t, void *);
int nvol_nan_scan(const float *, int64_t, const int64_t *, int32_t, int64_t *, void *);
int nvol_train_tc_scatter(const float *, const float *, int64_t, int64_t, const int64_t *, const int64_t *,
                          const int64_t *, const uint8_t *, int32_t, int32_t, float *, void *);

int64_t nvol_train_workspace_bytes(int64_t b, int32_t n_levels, int32_t n_feat, int32_t n_neurons, int32_t n_hidden,
                                   int32_t mode) {
    if (mode == 1) return train_tc_workspace(b, n_levels, n_feat, n_neurons, n_hidden);
    return ws_simt(b, n_levels, n_feat, n_neurons, n_hidden);
}

int nvol_train_fwd_bwd(const float *coords, const float *targets, int64_t b, int64_t b_global, const float *params,
                       float *grads, const int64_t *level_off, const int64_t *level_res,
                       const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels, int32_t n_feat,
                       int32_t n_neurons, int32_t n_hidden, int32_t relu_out, int32_t loss_kind, double *loss_sum,
                       void *workspace, int64_t workspace_bytes, int32_t mode, int64_t *nan_state,
                       void *stream) {
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    const int flags = mode & ~15;  // NVOL_TRAIN_PREENCODED / NVOL_TRAIN_ENCODE_ONLY (tcgen05 engine)
    mode &= 15;
    NVOL_REQUIRE(flags == 0 || mode == 1, "encode flags need the tcgen05 engine (mode 1)");
    NVOL_REQUIRE(b >= 1 && b_global >= b, "bad batch");
    NVOL_REQUIRE(n_hidden >= 1 && n_hidden <= 10, "n_hidden_layers out of range");
    NVOL_REQUIRE(loss_kind == 0 || loss_kind == 1, "loss kind must be L1 or L2");
    NVOL_REQUIRE(coords && targets && params && grads && loss_sum && workspace, "null pointer");
    NVOL_REQUIRE(workspace_bytes >= nvol_train_workspace_bytes(b, n_levels, n_feat, n_neurons, n_hidden, mode),
                 "workspace too small");
    cudaStream_t s = as_stream(stream);
    if (mode == 1)
        return train_tc_launch(coords, targets, b, b_global, params, grads, tab, n_neurons, n_hidden, relu_out,
                               loss_kind, loss_sum, workspace, workspace_bytes, flags, nan_state, s);
    const int m = n_levels, n = n_feat, nn = n_neurons, nh = n_hidden;
    const int nl = nh + 1;
    Ws w{(char *)workspace, 0};
    float *feats = w.take<float>(b * m * n);
    float *acts[12];
    acts[0] = feats;
    for (int i = 0; i < nh; ++i) acts[i + 1] = w.take<float>(b * nn);
    float *pred = w.take<float>(b);
    acts[nl] = pred;
    float *dpred = w.take<float>(b);
    int maxw = max(m * n, nn);
    float *s0 = w.take<float>(b * maxw);
    float *s1 = w.take<float>(b * maxw);
    float *dfeat = w.take<float>(b * m * n);
    (void)maxw;
    int32_t widths[12];
    widths[0] = m * n;
    for (int i = 1; i <= nh; ++i) widths[i] = nn;
    widths[nl] = 1;
    const void *wptr[12];
    void *gptr[12];
    int64_t off = 0;
    for (int l = 0; l < m; ++l) off = max(off, tab.offset[l] + tab.entries[l] * n);
    off = flat_weight_offset(params, off);  // W_0 starts 16-byte aligned (see nvol.h, flat layout)
    int64_t starts[16];  // parameter-group starts in the flat buffer (encoder, W_0, ...)
    starts[0] = 0;
    for (int i = 0; i < nl; ++i) {
        if (i + 1 < 16) starts[i + 1] = off;
        wptr[i] = params + off;
        gptr[i] = grads + off;
        off += (int64_t)widths[i] * widths[i + 1];
    }
    st = nvol_grid_encode_fwd(coords, b, params, level_off, level_res, level_entries, level_dense, m, n, nullptr,
                              nullptr, feats, 4, stream);
    if (st) return st;
    st = nvol_mlp_forward(b, nl, widths, wptr, (void *const *)acts, relu_out, 4, stream);
    if (st) return st;
    st = nvol_loss_and_grad_scaled(pred, targets, b, b_global, loss_kind, dpred, loss_sum, 4, stream);
    if (st) return st;
    st = nvol_mlp_backward(b, nl, widths, wptr, (const void *const *)acts, dpred, gptr, dfeat, s0, s1, relu_out, 4,
                           stream);
    if (st) return st;
    st = NVOL_EINVAL;
    if (!g_deterministic) {
        // float-atomic mode: the training engine's scatter (shared-memory coarse levels, merged
        // corner pairs) on the transposed dL/dfeat; shapes it does not take fall through
        transpose_kernel<<<dim3((unsigned)((b + 31) / 32), (unsigned)((m * n + 31) / 32)), dim3(32, 8), 0, s>>>(
            dfeat, s0, b, m * n);
        st = nvol_train_tc_scatter(coords, s0, b, b, level_off, level_res, level_entries, level_dense, m, n, grads,
                                   stream);
    }
    if (st != NVOL_OK)  // ordered mode: the sort-based fold, bit-identical to the reference's serial scatter
        st = nvol_grid_encode_bwd_coords(coords, dfeat, b, level_off, level_res, level_entries, level_dense, m, n,
                                         grads, 4, g_deterministic, stream);
    if (st == NVOL_OK && nan_state) st = nvol_nan_scan(grads, off, starts, nl + 1 < 16 ? nl + 1 : 16, nan_state, stream);
    (void)s;
    return st;
}

}  // extern "C"
