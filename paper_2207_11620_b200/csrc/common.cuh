// Shared device helpers for libnvol (sm_100a).
//
// Exactness discipline: every arithmetic step that must reproduce the
// reference's float32/float64 rounding goes through the explicit
// round-to-nearest intrinsics below, which nvcc never contracts into FMA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/nvol.h"

namespace nvol {

// ----------------------------------------------------------------------------- status
void set_error(const char *msg);
int check_launch(const char *what);

#define NVOL_REQUIRE(cond, msg)          \
    do {                                 \
        if (!(cond)) {                   \
            ::nvol::set_error(msg);      \
            return NVOL_EINVAL;          \
        }                                \
    } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

extern int g_deterministic;  // nvol_set_deterministic

inline unsigned grid_for(int64_t n, int block) {
    int64_t g = (n + block - 1) / block;
    return (unsigned)(g < 1 ? 1 : g);
}

// ----------------------------------------------------------------------------- exact arithmetic
__device__ __forceinline__ float xmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float xadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float xsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ float xdiv(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ float xsqrt(float a) { return __fsqrt_rn(a); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double xdiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double xsqrt(double a) { return __dsqrt_rn(a); }

// Adam update of one parameter: network.py:172-182, operation for operation.
template <typename T>
__device__ __forceinline__ void adam_one(T &p, T &g, T &m, T &v, T lr, T b1, T omb1, T b2, T omb2, T c1,
                                         T c2, T eps, T l2) {
    T geff = xadd(g, xmul(l2, p));
    T mj = xadd(xmul(m, b1), xmul(omb1, geff));
    T vj = xadd(xmul(v, b2), xmul(omb2, xmul(geff, geff)));
    T mhat = xdiv(mj, c1);
    T vhat = xdiv(vj, c2);
    p = xsub(p, xdiv(xmul(lr, mhat), xadd(xsqrt(vhat), eps)));
    m = mj;
    v = vj;
    g = (T)0;
}

// ----------------------------------------------------------------------------- NaN contract
// The training pipeline's device NaN state (int64[2], nvol.h "NaN state"):
// [0] = flat index where the first parameter group holding a NaN gradient starts
// (kNanNone: none), [1] = halted.  network.py:167-171 checks each group for NaN
// BEFORE updating it, so the groups in front of the offending one are updated
// and the rest are not; the flat buffer keeps the groups in order, so "update
// q < state[0]" is exactly that prefix.  The step's last Adam block then sets
// halted and every later kernel of the pipeline returns at entry (the
// reference raises and stops; t is not advanced).
constexpr int64_t kNanNone = 0x7fffffffffffffffll;

__device__ __forceinline__ bool nan_halted(const int64_t *ns) {
    return ns != nullptr && *reinterpret_cast<const volatile int64_t *>(ns + 1) != 0;
}
__device__ __forceinline__ int64_t nan_limit(const int64_t *ns) {
    return ns != nullptr ? *reinterpret_cast<const volatile int64_t *>(ns) : kNanNone;
}
__device__ __forceinline__ void nan_mark(int64_t *ns, int64_t group_start) {
    if (ns != nullptr) atomicMin(reinterpret_cast<long long *>(ns), (long long)group_start);
}

// ----------------------------------------------------------------------------- grid tables
// GridEncoder.kernel_tables() (encoding.py:174-177) packed by value.
struct GridTables {
    int32_t n_levels;
    int32_t n_feat;
    int32_t res[NVOL_MAX_LEVELS];
    int32_t dense[NVOL_MAX_LEVELS];
    int64_t entries[NVOL_MAX_LEVELS];
    int64_t offset[NVOL_MAX_LEVELS];
};

int pack_tables(GridTables &t, const int64_t *level_off, const int64_t *level_res,
                const int64_t *level_entries, const uint8_t *level_dense, int32_t n_levels,
                int32_t n_feat);

// _kernels.py:22-28 _vertex_slot.  Hashed levels always have entries = 2^k
// (encoding.py:160-164), so masking the u32-wrapped XOR is exact.
__device__ __forceinline__ int64_t vertex_slot(int64_t vx, int64_t vy, int64_t vz, int32_t res,
                                               int64_t entries, bool dense) {
    if (dense) {
        int64_t r1 = (int64_t)res + 1;
        return (vz * r1 + vy) * r1 + vx;
    }
    uint32_t h = ((uint32_t)vx) ^ ((uint32_t)vy * 2654435761u) ^ ((uint32_t)vz * 805459861u);
    return (int64_t)(h & (uint32_t)(entries - 1));
}

// One level's cell decomposition (_kernels.py:51-66 / encoding.py:179-185):
// s = p*R (one rounding), cell = clamp(floor(s), 0, R-1), fr = s - cell.
template <typename T>
struct Cell {
    int64_t cx, cy, cz;
    T fx, fy, fz;
};

template <typename T>
__device__ __forceinline__ Cell<T> cell_of(T x, T y, T z, int32_t res) {
    Cell<T> c;
    T r = (T)res;
    T sx = xmul(x, r), sy = xmul(y, r), sz = xmul(z, r);
    int64_t hi = (int64_t)res - 1;
    c.cx = min(max((int64_t)floor(sx), (int64_t)0), hi);
    c.cy = min(max((int64_t)floor(sy), (int64_t)0), hi);
    c.cz = min(max((int64_t)floor(sz), (int64_t)0), hi);
    c.fx = xsub(sx, (T)c.cx);
    c.fy = xsub(sy, (T)c.cy);
    c.fz = xsub(sz, (T)c.cz);
    return c;
}

// Corner weight in the reference order: w = wx; w *= wy; w *= wz (_kernels.py:59-61).
template <typename T>
__device__ __forceinline__ T corner_weight(const Cell<T> &c, int corner) {
    const T one = (T)1;
    T w = (corner & 1) ? c.fx : xsub(one, c.fx);
    w = xmul(w, (corner & 2) ? c.fy : xsub(one, c.fy));
    w = xmul(w, (corner & 4) ? c.fz : xsub(one, c.fz));
    return w;
}

// Flat parameter layout (include/nvol.h): the buffer may start 4*pad bytes past
// a 16-byte boundary (pad = (address / 4) % 4, chosen by the host so that the
// hashed levels' entry pairs are 16-byte aligned); W_0 starts at the first
// 16-byte-aligned float at or after the end of the encoder table.
inline int64_t flat_weight_offset(const float *flat, int64_t enc_floats) {
    const int64_t pad = (int64_t)((reinterpret_cast<uintptr_t>(flat) >> 2) & 3);
    return ((pad + enc_floats + 3) & ~(int64_t)3) - pad;
}

// ----------------------------------------------------------------------------- L2 residency hints
// The flat gradient (48.7 MB at cfg2) is kept L2-resident across a training
// step: Adam zeroes it with evict_last stores and the encoder-backward REDs
// carry the same policy, so the scatter's random read-modify-writes hit L2
// while Adam's p/m/v stream through with evict_first.
__device__ __forceinline__ uint64_t l2_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void red_add(float *a, float v, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}
__device__ __forceinline__ void red_add2(float *a, float x, float y, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.v2.f32 [%0], {%1, %2}, %3;" ::"l"(a), "f"(x), "f"(y), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ void red_add4(float *a, float4 v, uint64_t pol) {
    asm volatile("red.global.add.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}
__device__ __forceinline__ float4 ld4_hint(const float4 *a, uint64_t pol) {
    float4 v;
    asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "l"(a), "l"(pol));
    return v;
}
__device__ __forceinline__ void st4_hint(float4 *a, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z),
                 "f"(v.w), "l"(pol)
                 : "memory");
}

// ----------------------------------------------------------------------------- PCG64
// numpy.random.PCG64 (numpy 2.3.5): 128-bit LCG stepped before output, XSL-RR.
struct U128 {
    uint64_t hi, lo;
};

__device__ __forceinline__ U128 u128_mul(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
    return r;
}
__device__ __forceinline__ U128 u128_add(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}

__device__ __forceinline__ U128 pcg_mult() { return U128{0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull}; }

// Jump-ahead by delta steps (Brown's algorithm).
__device__ __forceinline__ U128 pcg_advance(U128 state, U128 inc, uint64_t delta) {
    U128 acc_mult{0, 1}, acc_plus{0, 0}, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult = u128_mul(acc_mult, cur_mult);
            acc_plus = u128_add(u128_mul(acc_plus, cur_mult), cur_plus);
        }
        cur_plus = u128_mul(u128_add(cur_mult, U128{0, 1}), cur_plus);
        cur_mult = u128_mul(cur_mult, cur_mult);
        delta >>= 1;
    }
    return u128_add(u128_mul(acc_mult, state), acc_plus);
}

__device__ __forceinline__ uint64_t pcg_output(U128 s) {
    uint64_t x = s.hi ^ s.lo;
    unsigned rot = (unsigned)(s.hi >> 58);
    return (x >> rot) | (x << ((64 - rot) & 63));
}

__device__ __forceinline__ float u32_to_f32(uint32_t u) {
    return __fmul_rn((float)(u >> 8), 1.0f / 16777216.0f);
}

// Sequential float32 reader of the u32 stream starting at global u32 index g.
struct PcgF32Stream {
    U128 state, inc;
    uint64_t g;
    uint64_t word;
    __device__ __forceinline__ void init(U128 s0, U128 inc_, uint64_t g0) {
        inc = inc_;
        g = g0;
        state = pcg_advance(s0, inc, g0 >> 1);
        if (g & 1) {  // the first draw is the high half of an already-started u64
            state = u128_add(u128_mul(state, pcg_mult()), inc);
            word = pcg_output(state);
        }
    }
    __device__ __forceinline__ float next() {
        if ((g & 1) == 0) {
            state = u128_add(u128_mul(state, pcg_mult()), inc);
            word = pcg_output(state);
        }
        uint32_t u = (g & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
        ++g;
        return u32_to_f32(u);
    }
};

__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ float ldg_hint(const float *a, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}

// volume.py:148-164 _gather_corners at one point (float32 throughout).  EVICT_FIRST:
// the training sampler's volume reads must not push the L2-resident tables and
// gradient out (they are touched once per step, the tables every kernel).
template <bool EVICT_FIRST = false>
__device__ __forceinline__ float trilinear_at(const float *__restrict__ vol, int64_t dx, int64_t dy,
                                              int64_t dz, float px, float py, float pz) {
    const uint64_t pol = EVICT_FIRST ? l2_evict_first() : 0ull;
    float sx = xsub(xmul(px, (float)dx), 0.5f);
    float sy = xsub(xmul(py, (float)dy), 0.5f);
    float sz = xsub(xmul(pz, (float)dz), 0.5f);
    int64_t x0 = (int64_t)floorf(sx), y0 = (int64_t)floorf(sy), z0 = (int64_t)floorf(sz);
    float fx = xsub(sx, (float)x0), fy = xsub(sy, (float)y0), fz = xsub(sz, (float)z0);
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        int ox = c & 1, oy = (c >> 1) & 1, oz = (c >> 2) & 1;
        int64_t ix = min(max(x0 + ox, (int64_t)0), dx - 1);
        int64_t iy = min(max(y0 + oy, (int64_t)0), dy - 1);
        int64_t iz = min(max(z0 + oz, (int64_t)0), dz - 1);
        float w = ox ? fx : xsub(1.0f, fx);
        w = xmul(w, oy ? fy : xsub(1.0f, fy));
        w = xmul(w, oz ? fz : xsub(1.0f, fz));
        const float *a = vol + (iz * dy + iy) * dx + ix;
        acc = xadd(acc, xmul(w, EVICT_FIRST ? ldg_hint(a, pol) : __ldg(a)));
    }
    return acc;
}

}  // namespace nvol
