// Multi-resolution grid encoder: forward gather and backward scatter.
//
// Reference: _kernels.py:31-92 (grid_encode_fwd / grid_encode_bwd) and
// encoding.py:145-226 (GridEncoder).  One thread per (sample, level): the m
// threads of a sample write its contiguous m*n feature row, each issuing 8
// independent n-wide vector gathers (float2 for n = 2) so a warp keeps 8x32
// table reads in flight against the L2-resident tables.
#include <cub/cub.cuh>

#include "common.cuh"

namespace nvol {

template <typename T, int N>
struct FeatVec {
    T v[N];
};

template <typename T, int N>
__device__ __forceinline__ FeatVec<T, N> load_feat(const T *__restrict__ p) {
    FeatVec<T, N> r;
    if constexpr (sizeof(T) == 4 && N == 2) {
        float2 a = __ldg(reinterpret_cast<const float2 *>(p));
        r.v[0] = a.x;
        r.v[1] = a.y;
    } else if constexpr (sizeof(T) == 4 && N == 4) {
        float4 a = __ldg(reinterpret_cast<const float4 *>(p));
        r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
    } else if constexpr (sizeof(T) == 4 && N == 8) {
        float4 a = __ldg(reinterpret_cast<const float4 *>(p));
        float4 b = __ldg(reinterpret_cast<const float4 *>(p) + 1);
        r.v[0] = a.x; r.v[1] = a.y; r.v[2] = a.z; r.v[3] = a.w;
        r.v[4] = b.x; r.v[5] = b.y; r.v[6] = b.z; r.v[7] = b.w;
    } else {
#pragma unroll
        for (int f = 0; f < N; ++f) r.v[f] = __ldg(p + f);
    }
    return r;
}

template <typename T, int N>
__global__ void __launch_bounds__(256) grid_encode_fwd_kernel(
    const T *__restrict__ coords, int64_t b, const T *__restrict__ params, const GridTables tab,
    int64_t *__restrict__ idx_cache, T *__restrict__ w_cache, T *__restrict__ out) {
    const int m = tab.n_levels;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b * m) return;
    int64_t i = t / m;
    int l = (int)(t - i * m);
    T x = coords[3 * i], y = coords[3 * i + 1], z = coords[3 * i + 2];
    const int32_t res = tab.res[l];
    const bool dense = tab.dense[l] != 0;
    const int64_t entries = tab.entries[l], loff = tab.offset[l];
    Cell<T> c = cell_of<T>(x, y, z, res);
    int64_t base[8];
    T w[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int64_t slot = vertex_slot(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), res,
                                   entries, dense);
        base[k] = loff + slot * N;
        w[k] = corner_weight<T>(c, k);
    }
    FeatVec<T, N> g[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) g[k] = load_feat<T, N>(params + base[k]);
    T acc[N];
#pragma unroll
    for (int f = 0; f < N; ++f) acc[f] = (T)0;
#pragma unroll
    for (int k = 0; k < 8; ++k)
#pragma unroll
        for (int f = 0; f < N; ++f) acc[f] = xadd(acc[f], xmul(w[k], g[k].v[f]));
    T *o = out + i * (int64_t)m * N + (int64_t)l * N;
#pragma unroll
    for (int f = 0; f < N; ++f) o[f] = acc[f];
    if (idx_cache) {
        int64_t *ic = idx_cache + (i * m + l) * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) ic[k] = base[k];
    }
    if (w_cache) {
        T *wc = w_cache + (i * m + l) * 8;
#pragma unroll
        for (int k = 0; k < 8; ++k) wc[k] = w[k];
    }
}

template <typename T, int N>
__device__ __forceinline__ void scatter_add(T *__restrict__ grad, const T (&v)[N]) {
    if constexpr (sizeof(T) == 4 && N == 2) {
        atomicAdd(reinterpret_cast<float2 *>(grad), make_float2(v[0], v[1]));
    } else if constexpr (sizeof(T) == 4 && (N == 4 || N == 8)) {
#pragma unroll
        for (int q = 0; q < N / 4; ++q)
            atomicAdd(reinterpret_cast<float4 *>(grad) + q,
                      make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]));
    } else {
#pragma unroll
        for (int f = 0; f < N; ++f) atomicAdd(grad + f, v[f]);
    }
}

template <typename T, int N>
__global__ void __launch_bounds__(256) grid_encode_bwd_cache_kernel(
    const T *__restrict__ dl, const int64_t *__restrict__ idx_cache, const T *__restrict__ w_cache,
    int64_t b, int m, T *__restrict__ grad) {
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b * m * 8) return;
    int64_t il = t >> 3;  // (i*m + l)
    int64_t i = il / m;
    int l = (int)(il - i * m);
    T w = w_cache[t];
    const T *d = dl + i * (int64_t)m * N + (int64_t)l * N;
    T v[N];
#pragma unroll
    for (int f = 0; f < N; ++f) v[f] = xmul(w, d[f]);
    scatter_add<T, N>(grad + idx_cache[t], v);
}

template <typename T, int N>
__global__ void __launch_bounds__(256) grid_encode_bwd_coords_kernel(
    const T *__restrict__ coords, const T *__restrict__ dl, int64_t b, const GridTables tab,
    T *__restrict__ grad) {
    const int m = tab.n_levels;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b * m) return;
    int64_t i = t / m;
    int l = (int)(t - i * m);
    const int32_t res = tab.res[l];
    Cell<T> c = cell_of<T>(coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], res);
    const T *d = dl + i * (int64_t)m * N + (int64_t)l * N;
    T dv[N];
#pragma unroll
    for (int f = 0; f < N; ++f) dv[f] = d[f];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int64_t slot = vertex_slot(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), res,
                                   tab.entries[l], tab.dense[l] != 0);
        T w = corner_weight<T>(c, k);
        T v[N];
#pragma unroll
        for (int f = 0; f < N; ++f) v[f] = xmul(w, dv[f]);
        scatter_add<T, N>(grad + tab.offset[l] + slot * N, v);
    }
}

// ----------------------------------------------------------------------------- deterministic scatter
// Bit-exact replica of the serial scatter (_kernels.py:82-92): every table
// row must fold its contributions in (sample, corner) order, starting from
// its current value.  Keys = global row index of each (i, l, c) corner; a
// stable radix sort keeps equal keys in (i, l, c) order, then one thread per
// run folds its run sequentially.  A correctness mode (reference-exact,
// run-to-run reproducible), not the fast path.
__global__ void det_keys_kernel(const float *__restrict__ coords, int64_t b, const GridTables tab,
                                uint32_t *__restrict__ keys, uint32_t *__restrict__ ids) {
    const int m = tab.n_levels;
    int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= b * m) return;
    int64_t i = t / m;
    int l = (int)(t - i * m);
    const int32_t res = tab.res[l];
    Cell<float> c = cell_of<float>(coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], res);
    int64_t row0 = tab.offset[l] / tab.n_feat;
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        int64_t slot = vertex_slot(c.cx + (k & 1), c.cy + ((k >> 1) & 1), c.cz + ((k >> 2) & 1), res,
                                   tab.entries[l], tab.dense[l] != 0);
        keys[t * 8 + k] = (uint32_t)(row0 + slot);
        ids[t * 8 + k] = (uint32_t)(t * 8 + k);
    }
}

// the contribution w_k * dL/dfeat of every sorted (i, l, c) corner, in sorted order (parallel;
// the same xmul the serial scatter does)
template <int N>
__global__ void det_values_kernel(const float *__restrict__ coords, const float *__restrict__ dl, int64_t total,
                                  const GridTables tab, const uint32_t *__restrict__ ids, float *__restrict__ vals) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= total) return;
    const int m = tab.n_levels;
    const uint32_t id = ids[q];
    const int k = id & 7;
    const int64_t il = id >> 3;
    const int64_t i = il / m;
    const int l = (int)(il - i * m);
    const Cell<float> c = cell_of<float>(coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], tab.res[l]);
    const float w = corner_weight<float>(c, k);
    const float *d = dl + i * (int64_t)m * N + (int64_t)l * N;
#pragma unroll
    for (int f = 0; f < N; ++f) vals[q * N + f] = xmul(w, d[f]);
}

constexpr int DET_LONG = 32;  // runs longer than this are folded by a warp (det_fold_long_kernel)

// one thread per run head: fold the run's contributions in order into its row (short runs);
// long runs go to a list for det_fold_long_kernel
template <int N>
__global__ void det_fold_kernel(int64_t total, const uint32_t *__restrict__ keys, const float *__restrict__ vals,
                                float *__restrict__ grad, uint32_t *__restrict__ long_heads,
                                uint32_t *__restrict__ n_long) {
    const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= total) return;
    const uint32_t key = keys[p];
    if (p > 0 && keys[p - 1] == key) return;  // not the head of a run
    if (p + DET_LONG < total && keys[p + DET_LONG] == key) {
        long_heads[atomicAdd(n_long, 1u)] = (uint32_t)p;
        return;
    }
    float acc[N];
    float *g = grad + (int64_t)key * N;
#pragma unroll
    for (int f = 0; f < N; ++f) acc[f] = g[f];
    for (int64_t q = p; q < total && keys[q] == key; ++q)
#pragma unroll
        for (int f = 0; f < N; ++f) acc[f] = xadd(acc[f], vals[q * N + f]);
#pragma unroll
    for (int f = 0; f < N; ++f) g[f] = acc[f];
}

// one warp per long run: the lanes load 32 contributions at a time (coalesced) and lane 0 folds
// them in order through shuffles -- the same sequence of xadds as the serial scatter
template <int N>
__global__ void det_fold_long_kernel(int64_t total, const uint32_t *__restrict__ keys, const float *__restrict__ vals,
                                     float *__restrict__ grad, const uint32_t *__restrict__ long_heads,
                                     const uint32_t *__restrict__ n_long) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = (int64_t)gridDim.x * (blockDim.x >> 5);
    const uint32_t cnt = *n_long;
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < cnt; w += nw) {
        const int64_t p = long_heads[w];
        const uint32_t key = keys[p];
        float acc[N];
        float *g = grad + (int64_t)key * N;
#pragma unroll
        for (int f = 0; f < N; ++f) acc[f] = g[f];
        // 8 chunks of 32 contributions per round trip: the loads of a round are all in flight at once
        constexpr int CH = 8;
        bool more = true;
        for (int64_t q0 = p; more; q0 += 32 * CH) {
            bool in[CH];
            float v[CH][N];
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int64_t q = q0 + c * 32 + lane;
                in[c] = q < total && keys[q] == key;
#pragma unroll
                for (int f = 0; f < N; ++f) v[c][f] = in[c] ? vals[q * N + f] : 0.0f;
            }
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                if (!more) break;
                const int nin = __popc(__ballot_sync(0xffffffffu, in[c]));  // a prefix of the chunk
                for (int j = 0; j < nin; ++j)
#pragma unroll
                    for (int f = 0; f < N; ++f) acc[f] = xadd(acc[f], __shfl_sync(0xffffffffu, v[c][f], j));
                if (nin < 32) more = false;
            }
        }
        if (lane == 0)
#pragma unroll
            for (int f = 0; f < N; ++f) g[f] = acc[f];
    }
}

static int launch_bwd_serial(const float *coords, const float *dl, int64_t b, const GridTables &tab,
                             float *grad, cudaStream_t s) {
    int64_t total = b * tab.n_levels * 8;
    int64_t rows = (tab.offset[tab.n_levels - 1] / tab.n_feat) + tab.entries[tab.n_levels - 1];
    NVOL_REQUIRE(total < (1ll << 32) && rows < (1ll << 32), "deterministic scatter: batch too large");
    int key_bits = 1;
    while ((1ll << key_bits) < rows) ++key_bits;
    uint32_t *buf = nullptr;
    size_t temp_bytes = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, (uint32_t *)nullptr, (uint32_t *)nullptr,
                                    (uint32_t *)nullptr, (uint32_t *)nullptr, (int)total, 0, key_bits, s);
    const int nf = tab.n_feat;
    size_t bytes = (5 + (size_t)nf) * (size_t)total * 4 + 256 + temp_bytes;
    if (cudaMallocAsync((void **)&buf, bytes, s) != cudaSuccess) return check_launch("det scatter alloc");
    uint32_t *k0 = buf, *v0 = buf + total, *k1 = buf + 2 * total, *v1 = buf + 3 * total;
    uint32_t *heads = buf + 4 * total;
    float *vals = reinterpret_cast<float *>(buf + 5 * total);
    uint32_t *n_long = buf + (5 + nf) * total;
    void *temp = n_long + 64;
    cudaMemsetAsync(n_long, 0, 4, s);
    det_keys_kernel<<<grid_for(b * tab.n_levels, 256), 256, 0, s>>>(coords, b, tab, k0, v0);
    cub::DeviceRadixSort::SortPairs(temp, temp_bytes, k0, k1, v0, v1, (int)total, 0, key_bits, s);
    unsigned grid = grid_for(total, 256);
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    switch (nf) {
#define DET_FOLD(NFV)                                                                                         \
    case NFV:                                                                                                 \
        det_values_kernel<NFV><<<grid, 256, 0, s>>>(coords, dl, total, tab, v1, vals);                       \
        det_fold_kernel<NFV><<<grid, 256, 0, s>>>(total, k1, vals, grad, heads, n_long);                      \
        det_fold_long_kernel<NFV><<<(unsigned)(sms * 8), 256, 0, s>>>(total, k1, vals, grad, heads, n_long);  \
        break;
        DET_FOLD(1)
        DET_FOLD(2)
        DET_FOLD(4)
        default: DET_FOLD(8)
#undef DET_FOLD
    }
    cudaFreeAsync(buf, s);
    return check_launch("grid_encode_bwd_deterministic");
}

template <typename T>
static int launch_fwd(const void *coords, int64_t b, const void *params, const GridTables &tab,
                      int64_t *idx, void *w, void *out, cudaStream_t s) {
    int64_t n = b * tab.n_levels;
    unsigned grid = grid_for(n, 256);
    const T *c = (const T *)coords;
    const T *p = (const T *)params;
    switch (tab.n_feat) {
        case 1: grid_encode_fwd_kernel<T, 1><<<grid, 256, 0, s>>>(c, b, p, tab, idx, (T *)w, (T *)out); break;
        case 2: grid_encode_fwd_kernel<T, 2><<<grid, 256, 0, s>>>(c, b, p, tab, idx, (T *)w, (T *)out); break;
        case 4: grid_encode_fwd_kernel<T, 4><<<grid, 256, 0, s>>>(c, b, p, tab, idx, (T *)w, (T *)out); break;
        default: grid_encode_fwd_kernel<T, 8><<<grid, 256, 0, s>>>(c, b, p, tab, idx, (T *)w, (T *)out); break;
    }
    return check_launch("grid_encode_fwd");
}

template <typename T>
static int launch_bwd_cache(const void *dl, const int64_t *idx, const void *w, int64_t b, int m,
                            int n, void *grad, cudaStream_t s) {
    unsigned grid = grid_for(b * m * 8, 256);
    const T *d = (const T *)dl;
    switch (n) {
        case 1: grid_encode_bwd_cache_kernel<T, 1><<<grid, 256, 0, s>>>(d, idx, (const T *)w, b, m, (T *)grad); break;
        case 2: grid_encode_bwd_cache_kernel<T, 2><<<grid, 256, 0, s>>>(d, idx, (const T *)w, b, m, (T *)grad); break;
        case 4: grid_encode_bwd_cache_kernel<T, 4><<<grid, 256, 0, s>>>(d, idx, (const T *)w, b, m, (T *)grad); break;
        default: grid_encode_bwd_cache_kernel<T, 8><<<grid, 256, 0, s>>>(d, idx, (const T *)w, b, m, (T *)grad); break;
    }
    return check_launch("grid_encode_bwd");
}

template <typename T>
static int launch_bwd_coords(const void *coords, const void *dl, int64_t b, const GridTables &tab,
                             void *grad, cudaStream_t s) {
    unsigned grid = grid_for(b * tab.n_levels, 256);
    const T *c = (const T *)coords;
    const T *d = (const T *)dl;
    switch (tab.n_feat) {
        case 1: grid_encode_bwd_coords_kernel<T, 1><<<grid, 256, 0, s>>>(c, d, b, tab, (T *)grad); break;
        case 2: grid_encode_bwd_coords_kernel<T, 2><<<grid, 256, 0, s>>>(c, d, b, tab, (T *)grad); break;
        case 4: grid_encode_bwd_coords_kernel<T, 4><<<grid, 256, 0, s>>>(c, d, b, tab, (T *)grad); break;
        default: grid_encode_bwd_coords_kernel<T, 8><<<grid, 256, 0, s>>>(c, d, b, tab, (T *)grad); break;
    }
    return check_launch("grid_encode_bwd_coords");
}

}  // namespace nvol

using namespace nvol;

extern "C" {

int nvol_grid_encode_fwd(const void *coords, int64_t b, const void *params, const int64_t *level_off,
                         const int64_t *level_res, const int64_t *level_entries,
                         const uint8_t *level_dense, int32_t n_levels, int32_t n_feat,
                         int64_t *idx_cache, void *w_cache, void *out, int32_t dtype_bytes,
                         void *stream) {
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    NVOL_REQUIRE(b >= 0, "negative batch");
    NVOL_REQUIRE(dtype_bytes == 4 || dtype_bytes == 8, "dtype must be float32 or float64");
    if (b == 0) return NVOL_OK;
    NVOL_REQUIRE(coords && params && out, "null pointer");
    if (dtype_bytes == 4)
        return launch_fwd<float>(coords, b, params, tab, idx_cache, w_cache, out, as_stream(stream));
    return launch_fwd<double>(coords, b, params, tab, idx_cache, w_cache, out, as_stream(stream));
}

int nvol_grid_encode_bwd(const void *dl_dfeat, const int64_t *idx_cache, const void *w_cache,
                         int64_t b, int32_t n_levels, int32_t n_feat, void *grad_out,
                         int32_t dtype_bytes, void *stream) {
    NVOL_REQUIRE(n_levels >= 1 && n_levels <= NVOL_MAX_LEVELS, "n_levels must be in [1, 32]");
    NVOL_REQUIRE(n_feat == 1 || n_feat == 2 || n_feat == 4 || n_feat == 8, "bad n_feat");
    NVOL_REQUIRE(dtype_bytes == 4 || dtype_bytes == 8, "dtype must be float32 or float64");
    if (b == 0) return NVOL_OK;
    NVOL_REQUIRE(dl_dfeat && idx_cache && w_cache && grad_out, "null pointer");
    if (dtype_bytes == 4)
        return launch_bwd_cache<float>(dl_dfeat, idx_cache, w_cache, b, n_levels, n_feat, grad_out,
                                       as_stream(stream));
    return launch_bwd_cache<double>(dl_dfeat, idx_cache, w_cache, b, n_levels, n_feat, grad_out,
                                    as_stream(stream));
}

int nvol_grid_encode_bwd_coords(const void *coords, const void *dl_dfeat, int64_t b,
                                const int64_t *level_off, const int64_t *level_res,
                                const int64_t *level_entries, const uint8_t *level_dense,
                                int32_t n_levels, int32_t n_feat, void *grad_out,
                                int32_t dtype_bytes, int32_t deterministic, void *stream) {
    GridTables tab;
    int st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
    if (st) return st;
    NVOL_REQUIRE(dtype_bytes == 4 || dtype_bytes == 8, "dtype must be float32 or float64");
    if (b == 0) return NVOL_OK;
    NVOL_REQUIRE(coords && dl_dfeat && grad_out, "null pointer");
    if (deterministic) {
        NVOL_REQUIRE(dtype_bytes == 4, "deterministic scatter is float32 only");
        return launch_bwd_serial((const float *)coords, (const float *)dl_dfeat, b, tab,
                                 (float *)grad_out, as_stream(stream));
    }
    if (dtype_bytes == 4)
        return launch_bwd_coords<float>(coords, dl_dfeat, b, tab, grad_out, as_stream(stream));
    return launch_bwd_coords<double>(coords, dl_dfeat, b, tab, grad_out, as_stream(stream));
}

}  // extern "C"
