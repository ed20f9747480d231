// Ray-marched volume rendering with macro-cell empty-space skipping (sm_100a).
//
// Reference: render.py:201-454 (scene setup, render_reference,
// render_wavefront), _render_kernels.py:52-563 (slab test, macro-cell DDA,
// adaptive step, the ray-march state machine, TF lookup, opacity
// correction, compositing, shadow phase), camera.py:117-143 (pixel rays),
// macrocell.py:63-156 (bordered ranges, exact majorants).
//
// Two schedules, as in the reference:
//  * in-shader (render_reference / rm_reference): one thread per ray runs its
//    state machine to completion and evaluates Phi inline (exact evaluator);
//  * sample streaming (render_wavefront): per iteration, rm_step_kernel
//    composites the previous samples of each alive ray (rm_shade) and stages up
//    to K new ones (rm_coord), appending them densely; one batched Phi
//    evaluation runs over all staged samples (exact or tcgen05) and a stable
//    CUB selection keeps the list of alive ray ids contiguous.
// Geometry (DDA, clocks, coordinates) is float64/float32 with the reference's
// operation order and no FMA contraction (file compiled with -fmad=false).
// pow is evaluated in float64 and rounded, which matches the reference's
// glibc powf in all but ~0.1% of inputs (1 ulp); images agree to float
// rounding, not bitwise.
#include <cub/cub.cuh>

#include <cmath>
#include <cstdlib>

#include <algorithm>

#include "common.cuh"
#include "field_exact.cuh"
#include "infer_tile.cuh"

namespace nvol {

constexpr int MAX_TF = 16;

struct TfTables {
    int ncv, nov;
    float cv[MAX_TF], crgb[3 * MAX_TF], ov[MAX_TF], oa[MAX_TF];
};

struct RmScene {
    int mode_shadow, use_mc, skip_empty, k_batch;
    float s1, s2, pexp, term, ka, ds;
    int64_t gx, gy, gz;
    double ng;
    float sd[3], bg[3];
    double hx, hy, hz;
    double ihx, ihy, ihz, ing;  // exact reciprocals of power-of-two extents / cell size, else 0
    TfTables tf;
    // path tracing (render.py mode "pathtrace", _render_kernels.py:566-878)
    int pathtrace, rr_depth;
    uint64_t seed, frame;
    float light[3];
    double mu_glob;
};

// 192 bytes, 16-byte aligned so a ray loads / stores as 12 vector accesses.
// pend / mdone carry one wavefront iteration's staging (count, march-ended
// flag) from the sampling half of rm_step_kernel to the next call's shading half.
struct alignas(16) RayState {
    float T, r, g, b, clock, sbar, best_w, best_t, Tsh, o[3], d[3], muc;
    double cell_exit, march_end, tm[3], td[3], t0;  // t0: float64 slab entry (path tracing starts there)
    int32_t pixel, phase, in_cell, pend;
    int32_t c[3], st[3], mdone, pad0;
};

// pow in float64, rounded.  x^1 = x, 1^y = 1 and x^2 = x*x (a float64 product of
// two floats is exact) are the values every faithful pow returns: taken directly.
__device__ __forceinline__ float powd(float x, float y) {
    if (y == 1.0f) return x;
    if (x == 1.0f) return 1.0f;
    if (y == 2.0f) return (float)((double)x * (double)x);
    return (float)pow((double)x, (double)y);
}

// x / h, as a multiply when h is a power of two (ih = 1 / h exactly, else 0): bit-identical
__device__ __forceinline__ double div_h(double x, double h, double ih) { return ih != 0.0 ? x * ih : x / h; }

__device__ __forceinline__ int64_t clampl(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

// _render_kernels.py:244-253
__device__ __forceinline__ float adaptive(float muc, float s1, float s2, float pexp) {
    float m = muc > 1.0f ? 1.0f : muc;
    float gap = 1.0f - m;
    float s = s1 + (s2 - s1) * powd(gap, pexp);
    return s < s1 ? s1 : s;
}

__device__ __forceinline__ float mu_read(const RmScene &S, const float *__restrict__ mu, int64_t cx, int64_t cy,
                                         int64_t cz) {
    int64_t ix = clampl(cx, 0, S.gx - 1), iy = clampl(cy, 0, S.gy - 1), iz = clampl(cz, 0, S.gz - 1);
    return __ldg(mu + (iz * S.gy + iy) * S.gx + ix);
}

// _render_kernels.py:92-138 _dda_enter + 268-305 _rm_cell_entry
__device__ void cell_entry(const RmScene &S, const float *__restrict__ mu, RayState &R) {
    const double t1 = R.march_end;
    if (!S.use_mc) {
        R.cell_exit = t1;
        R.sbar = S.s1;
        R.muc = 1.0f;
        R.in_cell = 1;
        return;
    }
    const double t0 = (double)R.clock, ng = S.ng;
    const int64_t gd[3] = {S.gx, S.gy, S.gz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double o = (double)R.o[a], d = (double)R.d[a];
        double p = o + t0 * d;
        int64_t c = clampl((int64_t)floor(div_h(p, ng, S.ing)), 0, gd[a] - 1);
        R.c[a] = c;
        if (d > 0.0) {
            R.st[a] = 1;
            R.tm[a] = t0 + ((double)(c + 1) * ng - p) / d;
            R.td[a] = ng / d;
        } else if (d < 0.0) {
            R.st[a] = -1;
            R.tm[a] = t0 + ((double)c * ng - p) / d;
            R.td[a] = -ng / d;
        } else {
            R.st[a] = 0;
            R.tm[a] = INFINITY;
            R.td[a] = INFINITY;
        }
    }
    double se = R.tm[0];
    if (R.tm[1] < se) se = R.tm[1];
    if (R.tm[2] < se) se = R.tm[2];
    if (se > t1) se = t1;
    R.cell_exit = se;
    R.muc = mu_read(S, mu, R.c[0], R.c[1], R.c[2]);
    R.sbar = adaptive(R.muc, S.s1, S.s2, S.pexp);
    R.in_cell = 1;
}

// _render_kernels.py:308-333
__device__ void cell_advance(const RmScene &S, const float *__restrict__ mu, RayState &R) {
    const double t1 = R.march_end;
    if (R.tm[0] <= R.tm[1] && R.tm[0] <= R.tm[2]) {
        R.c[0] += R.st[0];
        R.tm[0] = R.tm[0] + R.td[0];
    } else if (R.tm[1] <= R.tm[2]) {
        R.c[1] += R.st[1];
        R.tm[1] = R.tm[1] + R.td[1];
    } else {
        R.c[2] += R.st[2];
        R.tm[2] = R.tm[2] + R.td[2];
    }
    double se = R.tm[0];
    if (R.tm[1] < se) se = R.tm[1];
    if (R.tm[2] < se) se = R.tm[2];
    if (se > t1) se = t1;
    R.cell_exit = se;
    R.muc = mu_read(S, mu, R.c[0], R.c[1], R.c[2]);
    R.sbar = adaptive(R.muc, S.s1, S.s2, S.pexp);
}

// _render_kernels.py:336-361 _rm_next (returns the sample t or -1 at march end)
__device__ float rm_next(const RmScene &S, const float *__restrict__ mu, RayState &R) {
    const double t1 = R.march_end;
    if (R.in_cell == 0) cell_entry(S, mu, R);
    for (;;) {
        const float sbar = R.sbar;
        const double se = R.cell_exit;
        if (S.use_mc && S.skip_empty && R.muc <= 0.0f) {
            float t = R.clock;
            while ((double)(t + 0.5f * sbar) < se) t = t + sbar;
            R.clock = t;
        } else {
            float ts = R.clock + 0.5f * sbar;
            if ((double)ts < se) {
                R.clock = R.clock + sbar;
                return ts;
            }
        }
        if (se >= t1) return -1.0f;
        cell_advance(S, mu, R);
    }
}

__device__ float tf_alpha(const TfTables &T, float v) {
    float x = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
    int n = T.nov;
    if (x <= T.ov[0]) return T.oa[0];
    if (x >= T.ov[n - 1]) return T.oa[n - 1];
    int i = 1;
    while (T.ov[i] < x) ++i;
    float w = (x - T.ov[i - 1]) / (T.ov[i] - T.ov[i - 1]);
    return T.oa[i - 1] + w * (T.oa[i] - T.oa[i - 1]);
}

__device__ void tf_rgb(const TfTables &T, float v, float &r, float &g, float &b) {
    float x = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
    int n = T.ncv;
    const float *c = T.crgb;
    if (x <= T.cv[0]) {
        r = c[0], g = c[1], b = c[2];
        return;
    }
    if (x >= T.cv[n - 1]) {
        r = c[3 * (n - 1)], g = c[3 * (n - 1) + 1], b = c[3 * (n - 1) + 2];
        return;
    }
    int i = 1;
    while (T.cv[i] < x) ++i;
    float w = (x - T.cv[i - 1]) / (T.cv[i] - T.cv[i - 1]);
    r = c[3 * (i - 1)] + w * (c[3 * i] - c[3 * (i - 1)]);
    g = c[3 * (i - 1) + 1] + w * (c[3 * i + 1] - c[3 * (i - 1) + 1]);
    b = c[3 * (i - 1) + 2] + w * (c[3 * i + 2] - c[3 * (i - 1) + 2]);
}

// _render_kernels.py:364-392 (true when the current march just ended)
__device__ bool rm_consume(const RmScene &S, RayState &R, float v, float ts, float sbar) {
    float a = tf_alpha(S.tf, v) * S.ds;
    if (a < 0.0f) a = 0.0f;
    if (a > 1.0f) a = 1.0f;
    float abar = 1.0f - powd(1.0f - a, sbar / S.s1);
    if (R.phase == 0) {
        float T = R.T;
        float w = T * abar;
        if (S.mode_shadow && w > R.best_w) {
            R.best_w = w;
            R.best_t = ts;
        }
        float cr, cg, cb;
        tf_rgb(S.tf, v, cr, cg, cb);
        R.r += w * cr;
        R.g += w * cg;
        R.b += w * cb;
        T = T * (1.0f - abar);
        R.T = T;
        return T < S.term;
    }
    float Tsh = R.Tsh * (1.0f - abar);
    R.Tsh = Tsh;
    return Tsh < S.term;
}

// _render_kernels.py:54-89
__device__ bool isect(double ox, double oy, double oz, double dx, double dy, double dz, double hx, double hy,
                      double hz, double &t0o, double &t1o) {
    double t0 = -INFINITY, t1 = INFINITY;
    const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz}, h[3] = {hx, hy, hz};
    for (int a = 0; a < 3; ++a) {
        if (d[a] != 0.0) {
            double ta = (0.0 - o[a]) / d[a], tb = (h[a] - o[a]) / d[a];
            if (ta > tb) {
                double t = ta;
                ta = tb;
                tb = t;
            }
            t0 = t0 > ta ? t0 : ta;
            t1 = t1 < tb ? t1 : tb;
        } else if (o[a] < 0.0 || o[a] > h[a]) {
            return false;
        }
    }
    t0 = t0 > 0.0 ? t0 : 0.0;
    if (t1 <= t0) return false;
    t0o = t0;
    t1o = t1;
    return true;
}

// _render_kernels.py:395-420 (true = ray done)
__device__ bool rm_phase_end(const RmScene &S, RayState &R) {
    if (!S.mode_shadow || R.phase != 0) return true;
    R.phase = 1;
    if (R.r == 0.0f && R.g == 0.0f && R.b == 0.0f) return true;
    double bt = (double)R.best_t;
    double bx = (double)R.o[0] + bt * (double)R.d[0];
    double by = (double)R.o[1] + bt * (double)R.d[1];
    double bz = (double)R.o[2] + bt * (double)R.d[2];
    double t0s, t1s;
    if (!isect(bx, by, bz, (double)S.sd[0], (double)S.sd[1], (double)S.sd[2], S.hx, S.hy, S.hz, t0s, t1s)) return true;
    R.o[0] = (float)bx;
    R.o[1] = (float)by;
    R.o[2] = (float)bz;
    R.d[0] = S.sd[0];
    R.d[1] = S.sd[1];
    R.d[2] = S.sd[2];
    R.clock = (float)t0s;
    R.march_end = t1s;
    R.in_cell = 0;
    return false;
}

// _render_kernels.py:423-432
__device__ void rm_final(const RmScene &S, const RayState &R, float *__restrict__ img) {
    float scale = 1.0f;
    if (S.mode_shadow) scale = S.ka + (1.0f - S.ka) * R.Tsh;
    float T = R.T;
    int64_t p = R.pixel;
    img[3 * p] = R.r * scale + T * S.bg[0];
    img[3 * p + 1] = R.g * scale + T * S.bg[1];
    img[3 * p + 2] = R.b * scale + T * S.bg[2];
}

// _render_kernels.py:435-452
__device__ void coord_at(const RmScene &S, const RayState &R, float ts, float &x, float &y, float &z) {
    const float one_below = 0.99999994f;
    const double h[3] = {S.hx, S.hy, S.hz}, ih[3] = {S.ihx, S.ihy, S.ihz};
    float c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float v = (float)div_h((double)R.o[a] + (double)ts * (double)R.d[a], h[a], ih[a]);
        if (v < 0.0f) v = 0.0f;
        if (v >= 1.0f) v = one_below;
        c[a] = v;
    }
    x = c[0];
    y = c[1];
    z = c[2];
}

// ----------------------------------------------------------------------------- ray generation
struct CamParams {
    float eye[3];
    double fwd[3], right[3], up[3];
    double tan_half, aspect;
    int64_t width, height;
    int64_t row0, nrows;  // image tile: rows [row0, row0 + nrows) of the width x height frame
};

// camera.py:117-143 (float64, cast to float32) + render.py:225-243 slab test:
// the ray of tile pixel p and whether it hits the volume box
__device__ __forceinline__ bool make_ray(const CamParams &cam, const RmScene &S, int64_t p, RayState &R) {
    const int64_t pf = p + cam.row0 * cam.width;  // pixel index in the full frame (camera.py:117-125)
    double ii = (double)(pf % cam.width), jj = floor((double)pf / (double)cam.width);
    double nx = ((ii + 0.5) / (double)cam.width * 2.0 - 1.0) * (cam.tan_half * cam.aspect);
    double ny = (1.0 - (jj + 0.5) / (double)cam.height * 2.0) * cam.tan_half;
    double d[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) d[a] = cam.fwd[a] + nx * cam.right[a] + ny * cam.up[a];
    double nrm = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    memset(&R, 0, sizeof(R));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        R.d[a] = (float)(d[a] / nrm);
        R.o[a] = cam.eye[a];
    }
    // vectorised slab test of render.py:225-243 on the float32 ray, in float64
    const double h[3] = {S.hx, S.hy, S.hz};
    double lo = -INFINITY, up = INFINITY;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double o = (double)R.o[a], dd = (double)R.d[a];
        double l, u;
        if (dd == 0.0) {
            bool inside = (o >= 0.0) && (o <= h[a]);
            l = inside ? -INFINITY : INFINITY;
            u = inside ? INFINITY : -INFINITY;
        } else {
            double ta = (0.0 - o) / dd, tb = (h[a] - o) / dd;
            l = fmin(ta, tb);
            u = fmax(ta, tb);
        }
        lo = fmax(lo, l);
        up = fmin(up, u);
    }
    double t0 = fmax(lo, 0.0), t1 = up;
    R.T = 1.0f;
    R.clock = (float)t0;
    R.t0 = t0;
    R.Tsh = 1.0f;
    R.march_end = t1;
    R.pixel = (int32_t)p;
    return t1 > t0;
}

// background into every pixel of the tile + the hit flags (the stable selection
// of hit pixel ids then orders the rays as the reference's boolean gather does)
__global__ void ray_hits_kernel(const CamParams cam, const RmScene S, uint8_t *__restrict__ hit,
                                float *__restrict__ img) {
    int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // pixel within the tile
    const int64_t n = cam.width * cam.nrows;
    if (p >= n) return;
    img[3 * p] = S.bg[0];
    img[3 * p + 1] = S.bg[1];
    img[3 * p + 2] = S.bg[2];
    RayState R;
    hit[p] = make_ray(cam, S, p, R) ? 1 : 0;
}

__global__ void set_count_kernel(int64_t *__restrict__ c, int64_t v) { *c = v; }

__global__ void iota_kernel(int32_t *__restrict__ ids, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) ids[i] = (int32_t)i;
}

// the initial state of hit ray i (pixel ids[i]), staged through shared memory so
// the 192-byte records leave as coalesced 16-byte stores
constexpr int RG_THREADS = 128;
__global__ void __launch_bounds__(RG_THREADS) raygen_kernel(const CamParams cam, const RmScene S,
                                                            const int32_t *__restrict__ ids, int64_t n,
                                                            RayState *__restrict__ rays) {
    __shared__ RayState st[RG_THREADS];
    const int64_t i0 = (int64_t)blockIdx.x * RG_THREADS, i = i0 + threadIdx.x;
    if (i < n) make_ray(cam, S, ids[i], st[threadIdx.x]);
    __syncthreads();
    const int64_t cnt = min((int64_t)RG_THREADS, n - i0);
    const uint4 *src = reinterpret_cast<const uint4 *>(st);
    uint4 *dst = reinterpret_cast<uint4 *>(rays + i0);
    constexpr int Q = (int)(sizeof(RayState) / 16);
    for (int64_t q = threadIdx.x; q < cnt * Q; q += RG_THREADS) dst[q] = src[q];
}

// ----------------------------------------------------------------------------- field for the in-shader marcher
struct FieldDesc {
    int use_grid;
    const float *norm;
    int64_t ndx, ndy, ndz;
    const float *params;
    const float *weights;
};

// render_reference / rm_reference (_render_kernels.py:455-488): one thread per
// ray to completion, Phi inline (exact evaluator, shared-memory feature column).
template <int NN>
__global__ void __launch_bounds__(FE_THREADS) rm_mega_kernel(RayState *__restrict__ rays, int64_t n, const RmScene S,
                                                             const float *__restrict__ mu, const FieldDesc F,
                                                             const GridTables tab, const MlpShape sh, int maxw,
                                                             float *__restrict__ img,
                                                             unsigned long long *__restrict__ evals) {
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    float *wt = smem;
    int wsz = F.use_grid ? 0 : stage_weights_t(F.weights, sh, wt);
    float *h0 = wt + wsz, *h1 = h0 + maxw * FE_THREADS;
    __syncthreads();
    int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    RayState R = rays[r];
    unsigned long long ev = 0;
    float *col0 = h0 + threadIdx.x, *col1 = h1 + threadIdx.x;
    for (;;) {
        float ts = rm_next(S, mu, R);
        if (ts < 0.0f) {
            if (rm_phase_end(S, R)) {
                rm_final(S, R, img);
                break;
            }
            continue;
        }
        float x, y, z;
        coord_at(S, R, ts, x, y, z);
        float v;
        if (F.use_grid) {
            v = trilinear_at(F.norm, F.ndx, F.ndy, F.ndz, x, y, z);
        } else {
            encode_exact(x, y, z, F.params, tab, col0);
            if constexpr (NN > 0)
                v = mlp_exact_col<NN, false>(col0, tab.n_levels * tab.n_feat, wt, sh);
            else
                v = mlp_exact_smem(col0, col1, wt, sh);
        }
        ++ev;
        if (rm_consume(S, R, v, ts, R.sbar)) {
            if (rm_phase_end(S, R)) {
                rm_final(S, R, img);
                break;
            }
        }
    }
    atomicAdd(evals, ev);
}

// render_reference / rm_reference with the tcgen05 evaluator: the in-shader marcher on the tensor
// cores.  Persistent CTAs (two per SM); each CTA keeps 256 rays in flight, one per thread, and pulls
// new hit rays from a global queue as its rays finish.  A round: every ray marches to its next
// sample (rm_next / coord_at, ending and replacing rays as the reference's loop does), the CTA
// evaluates the 256 samples as two tensor-core tiles (infer_tile: the encode and split-fp16 MLP of
// the batched evaluator, bit-identical values), and every ray composites its own value
// (rm_consume) -- the reference's per-ray sequence sample -> Phi -> consume, so images equal the
// wavefront's bit for bit, with no ray records, staging or compaction in global memory.
template <int NF>
__global__ void __launch_bounds__(IT_THREADS, 2) rm_tc_kernel(const int32_t *__restrict__ hitpix, int64_t n,
                                                              int32_t *__restrict__ queue, const CamParams cam,
                                                              const RmScene S, const float *__restrict__ mu,
                                                              const float *__restrict__ params, const GridTables tab,
                                                              const InferShape sh, const uint8_t *__restrict__ wimg,
                                                              float *__restrict__ img,
                                                              unsigned long long *__restrict__ evals) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base_sh;
    __shared__ float s_xyz[3 * IT_THREADS], s_val[IT_THREADS];
    __shared__ uint8_t s_ok[IT_THREADS];
    infer_prologue(smem, sh, wimg, &mbar, &tmem_base_sh);
    const int tid = threadIdx.x, s = tid & (IT_TILE - 1), h = tid >> 7;
    const uint32_t tmem = tmem_base_sh;
    uint32_t phase = 0;
    RayState R;
    bool have = false, drained = false;
    float ts = 0.0f;
    unsigned long long ev = 0;
    for (;;) {
        bool staged = false;
        float x = 0.5f, y = 0.5f, z = 0.5f;
        while (!drained) {
            if (!have) {
                const int32_t q = atomicAdd(queue, 1);
                if (q >= n) {
                    drained = true;
                    break;
                }
                make_ray(cam, S, hitpix[q], R);  // a hit ray (ray_hits_kernel + selection)
                have = true;
            }
            const float t = rm_next(S, mu, R);
            if (t < 0.0f) {
                if (rm_phase_end(S, R)) {
                    rm_final(S, R, img);
                    have = false;
                }
                continue;
            }
            ts = t;
            coord_at(S, R, t, x, y, z);
            staged = true;
            break;
        }
        s_xyz[3 * tid] = x;
        s_xyz[3 * tid + 1] = y;
        s_xyz[3 * tid + 2] = z;
        s_ok[tid] = staged ? 1 : 0;
        if (!__syncthreads_or(staged ? 1 : 0)) break;  // (also publishes s_xyz / s_ok)
        for (int half = 0; half < 2; ++half) {         // the rays of threads [128 half, 128 half + 128)
            const int r = half * IT_TILE + s;
            const float v = infer_tile<NF, true>(smem, sh, tab, params, s_xyz[3 * r], s_xyz[3 * r + 1],
                                                 s_xyz[3 * r + 2], s_ok[r] != 0, tmem, &mbar, phase);
            if (h == 0) s_val[r] = v;
        }
        __syncthreads();
        if (staged) {
            ++ev;
            if (rm_consume(S, R, s_val[tid], ts, R.sbar) && rm_phase_end(S, R)) {
                rm_final(S, R, img);
                have = false;
            }
        }
    }
    for (int o = 16; o > 0; o >>= 1) ev += __shfl_down_sync(0xffffffffu, ev, o);
    if ((tid & 31) == 0 && ev) atomicAdd(evals, ev);
    infer_teardown(tmem, sh);
}

// ----------------------------------------------------------------------------- wavefront stages
// One wavefront iteration per alive ray (rays[ids[pos]]): the shading half of
// the previous iteration (_render_kernels.py:543-563 rm_shade: composite the
// evaluated staged samples, end the march / phase, write the pixel) followed by
// the sampling half of this one (_render_kernels.py:491-515 rm_coord: stage up
// to K samples).  Fusing the two halves touches each ray record once per
// iteration.  Staging is addressed by ray (ray * K + c); counts / keep by
// position for the compaction that follows.
__global__ void __launch_bounds__(128) rm_step_kernel(const int32_t *__restrict__ ids, int64_t n,
                                                      const int64_t *__restrict__ n_dev,
                                                      RayState *__restrict__ rays, const RmScene S,
                                                      const float *__restrict__ mu, int shade,
                                                      const float *__restrict__ values, float *__restrict__ sxyz,
                                                      float *__restrict__ sts, float *__restrict__ ssbar,
                                                      uint8_t *__restrict__ keep,
                                                      float *__restrict__ img, unsigned long long *__restrict__ evals,
                                                      int32_t *__restrict__ coord_rays, const CamParams cam,
                                                      const int32_t *__restrict__ hitpix, float *__restrict__ dxyz,
                                                      int32_t *__restrict__ dray, int32_t *__restrict__ dcount) {
    const int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int c = 0, marched = 0;
    int64_t ray = 0;
    // n_dev: the alive count produced on the device; n is then only its upper bound
    // (launch size), and positions in [*n_dev, n) stage nothing and keep nothing
    const int64_t nact = n_dev ? *n_dev : n;
    if (pos < n && pos >= nact) {
        keep[pos] = 0;
    } else if (pos < n) {
        ray = ids[pos];
        RayState R;
        if (hitpix)
            make_ray(cam, S, hitpix[ray], R);  // first iteration: the ray is generated here, not loaded
        else
            R = rays[ray];
        const int K = S.k_batch;
        bool alive = true;
        if (shade) {
            bool ended = false;
            for (int q = 0; q < R.pend; ++q) {
                const int64_t i = ray * K + q;
                if (rm_consume(S, R, values[i], sts[i], ssbar[i])) {
                    ended = true;
                    break;
                }
            }
            if (!ended && R.mdone) ended = true;
            if (ended && rm_phase_end(S, R)) {
                rm_final(S, R, img);
                alive = false;
            }
        }
        if (alive) {
            marched = 1;
            int done = 0;
            while (c < K) {
                float ts = rm_next(S, mu, R);
                if (ts < 0.0f) {
                    done = 1;
                    break;
                }
                float x, y, z;
                coord_at(S, R, ts, x, y, z);
                const int64_t i = ray * K + c;
                sxyz[3 * i] = x;
                sxyz[3 * i + 1] = y;
                sxyz[3 * i + 2] = z;
                sts[i] = ts;
                ssbar[i] = R.sbar;
                ++c;
            }
            R.pend = c;
            R.mdone = done;
            rays[ray] = R;
        }
        keep[pos] = alive ? 1 : 0;
    }
    // the staged samples go densely to dxyz (one atomic per warp; evaluation order does not
    // matter: every sample is evaluated independently), with their (ray, slot) for the scatter back
    {
        const int lane = threadIdx.x & 31;
        int incl = c;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        const int wtot = __shfl_sync(0xffffffffu, incl, 31);
        int base = 0;
        if (lane == 31 && wtot) base = atomicAdd(dcount, wtot);
        base = __shfl_sync(0xffffffffu, base, 31) + incl - c;
        const int K = S.k_batch;
        for (int j = 0; j < c; ++j) {
            const int64_t i = ray * K + j;
            const int64_t d = (int64_t)base + j;
            dxyz[3 * d] = sxyz[3 * i];
            dxyz[3 * d + 1] = sxyz[3 * i + 1];
            dxyz[3 * d + 2] = sxyz[3 * i + 2];
            dray[d] = (int32_t)i;
        }
    }
    // phi_eval_staged evaluates exactly the staged samples (_render_kernels.py:518-540)
    unsigned long long tot = (unsigned long long)c;
    int m = marched;
    for (int o = 16; o > 0; o >>= 1) {
        tot += __shfl_down_sync(0xffffffffu, tot, o);
        m += __shfl_down_sync(0xffffffffu, m, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (tot) atomicAdd(evals, tot);
        if (m) atomicAdd(coord_rays, m);
    }
}

// evaluated dense samples back to their (ray, slot): values[dray[i]] = dvals[i], i < *count
__global__ void scatter_dense_kernel(const float *__restrict__ dvals, const int32_t *__restrict__ dray,
                                     const int32_t *__restrict__ count, int64_t bound, float *__restrict__ values) {
    const int64_t n = min(bound, (int64_t)*count);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        values[dray[i]] = dvals[i];
}

static unsigned dense_grid(int64_t n) {  // grid-stride launches sized for a device-side count <= n
    const int64_t b = (n + 255) / 256;
    return (unsigned)(b < 1 ? 1 : (b > 148 * 8 ? 148 * 8 : b));
}

// Path tracing's position-indexed staging (one slot per ray): compacted with the
// exclusive scan offs, evaluated densely, scattered back.
__global__ void compact_staged_kernel(const float *__restrict__ sxyz, const int32_t *__restrict__ counts,
                                      const int32_t *__restrict__ offs, int64_t n, int K, float *__restrict__ dxyz,
                                      int32_t *__restrict__ total) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int c = counts[r], o = offs[r];
    for (int j = 0; j < c; ++j) {
        const int64_t i = r * K + j;
        dxyz[3 * (int64_t)(o + j)] = sxyz[3 * i];
        dxyz[3 * (int64_t)(o + j) + 1] = sxyz[3 * i + 1];
        dxyz[3 * (int64_t)(o + j) + 2] = sxyz[3 * i + 2];
    }
    if (r == n - 1) *total = o + c;
}

__global__ void scatter_staged_kernel(const float *__restrict__ dvals, const int32_t *__restrict__ counts,
                                      const int32_t *__restrict__ offs, int64_t n, int K, float *__restrict__ values) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const int c = counts[r], o = offs[r];
    for (int j = 0; j < c; ++j) values[r * K + j] = dvals[o + j];
}

// ----------------------------------------------------------------------------- macro-cells
// macrocell.py:63-76: per cell min/max over its voxels plus a one-voxel border
// (optionally clipping the values to [0,1] first, macrocell.py:97).
__global__ void mc_ranges_kernel(const float *__restrict__ vals, int64_t dx, int64_t dy, int64_t dz, int64_t ng,
                                 int64_t gx, int64_t gy, int64_t gz, int clip, float *__restrict__ lo,
                                 float *__restrict__ hi) {
    int64_t cell = blockIdx.x;
    if (cell >= gx * gy * gz) return;
    int64_t cx = cell % gx, cy = (cell / gx) % gy, cz = cell / (gx * gy);
    int64_t x0 = max(cx * ng - 1, (int64_t)0), x1 = min((cx + 1) * ng + 1, dx);
    int64_t y0 = max(cy * ng - 1, (int64_t)0), y1 = min((cy + 1) * ng + 1, dy);
    int64_t z0 = max(cz * ng - 1, (int64_t)0), z1 = min((cz + 1) * ng + 1, dz);
    int64_t nxv = x1 - x0, nyv = y1 - y0, nzv = z1 - z0, tot = nxv * nyv * nzv;
    float mn = INFINITY, mx = -INFINITY;
    for (int64_t q = threadIdx.x; q < tot; q += blockDim.x) {
        int64_t x = x0 + q % nxv, y = y0 + (q / nxv) % nyv, z = z0 + q / (nxv * nyv);
        float v = vals[(z * dy + y) * dx + x];
        if (clip) v = fminf(fmaxf(v, 0.0f), 1.0f);
        mn = fminf(mn, v);
        mx = fmaxf(mx, v);
    }
    __shared__ float smn[32], smx[32];
    for (int o = 16; o > 0; o >>= 1) {
        mn = fminf(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    if ((threadIdx.x & 31) == 0) {
        smn[threadIdx.x >> 5] = mn;
        smx[threadIdx.x >> 5] = mx;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mn = fminf(mn, smn[w]);
            mx = fmaxf(mx, smx[w]);
        }
        if (tot > 0) {
            lo[cell] = mn;
            hi[cell] = mx;
        }
    }
}

// numpy.interp (the reference's np.interp in macrocell.py:148-149), float64
__device__ double interp_np(double x, const double *xp, const double *fp, int n) {
    if (x < xp[0]) return fp[0];
    if (x > xp[n - 1]) return fp[n - 1];
    if (x == xp[n - 1]) return fp[n - 1];
    int j = 0;
    while (j < n - 2 && xp[j + 1] <= x) ++j;
    if (x == xp[j]) return fp[j];
    double slope = (fp[j + 1] - fp[j]) / (xp[j + 1] - xp[j]);
    double r = slope * (x - xp[j]) + fp[j];
    if (isnan(r)) r = slope * (x - xp[j + 1]) + fp[j + 1];
    return r;
}

struct OpacityPts {
    int n;
    double v[MAX_TF], a[MAX_TF];
};

// macrocell.py:136-156 macrocell_set_tf: exact max opacity over [lo, hi]
__global__ void mc_set_tf_kernel(const float *__restrict__ lo_a, const float *__restrict__ hi_a, int64_t ncell,
                                 const OpacityPts P, double density_scale, float *__restrict__ mu) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= ncell) return;
    float lf = lo_a[i], hf = hi_a[i];
    bool touched = lf <= hf;
    double lo = fmin(fmax((double)lf, 0.0), 1.0), hi = fmin(fmax((double)hf, 0.0), 1.0);
    double best = fmax(interp_np(lo, P.v, P.a, P.n), interp_np(hi, P.v, P.a, P.n));
    for (int q = 0; q < P.n; ++q)
        if (P.v[q] > lo && P.v[q] < hi) best = fmax(best, P.a[q]);
    mu[i] = touched ? (float)(best * density_scale) : 0.0f;
}

// ----------------------------------------------------------------------------- host helpers
static int fill_scene(RmScene &S, const double *rp, const float *tf_cv, const float *tf_crgb, int ncv,
                      const float *tf_ov, const float *tf_oa, int nov, int64_t gx, int64_t gy, int64_t gz) {
    NVOL_REQUIRE(ncv >= 1 && ncv <= MAX_TF && nov >= 1 && nov <= MAX_TF, "transfer function has too many points");
    // rp: mode_shadow, use_mc, skip_empty, k_batch, s1, s2, pexp, term, ka, ds, ng,
    //     sd[3], bg[3], hx, hy, hz, then the path-tracing block below
    S.mode_shadow = (int)rp[0];
    S.use_mc = (int)rp[1];
    S.skip_empty = (int)rp[2];
    S.k_batch = (int)rp[3];
    S.s1 = (float)rp[4];
    S.s2 = (float)rp[5];
    S.pexp = (float)rp[6];
    S.term = (float)rp[7];
    S.ka = (float)rp[8];
    S.ds = (float)rp[9];
    S.ng = rp[10];
    for (int a = 0; a < 3; ++a) {
        S.sd[a] = (float)rp[11 + a];
        S.bg[a] = (float)rp[14 + a];
    }
    S.hx = rp[17];
    S.hy = rp[18];
    S.hz = rp[19];
    auto exact_inv = [](double h) {
        int e = 0;
        return (h > 0.0 && std::frexp(h, &e) == 0.5) ? 1.0 / h : 0.0;
    };
    S.ihx = exact_inv(S.hx);
    S.ihy = exact_inv(S.hy);
    S.ihz = exact_inv(S.hz);
    S.ing = exact_inv(S.ng);
    // rp[20..28]: pathtrace, seed (low 32 bits, high 32 bits), frame, rr_depth, light radiance[3], mu_glob
    S.pathtrace = (int)rp[20];
    S.seed = (uint64_t)rp[21] | ((uint64_t)rp[22] << 32);
    S.frame = (uint64_t)rp[23];
    S.rr_depth = (int)rp[24];
    for (int a = 0; a < 3; ++a) S.light[a] = (float)rp[25 + a];
    S.mu_glob = rp[28];
    S.gx = gx;
    S.gy = gy;
    S.gz = gz;
    S.tf.ncv = ncv;
    S.tf.nov = nov;
    for (int i = 0; i < ncv; ++i) {
        S.tf.cv[i] = tf_cv[i];
        for (int c = 0; c < 3; ++c) S.tf.crgb[3 * i + c] = tf_crgb[3 * i + c];
    }
    for (int i = 0; i < nov; ++i) {
        S.tf.ov[i] = tf_ov[i];
        S.tf.oa[i] = tf_oa[i];
    }
    return NVOL_OK;
}

// ============================================================================ path tracing
// _render_kernels.py:566-878 (delta / Woodcock tracking with macro-cell
// majorants, next-event estimation toward a directional light, isotropic
// scattering with TF-colour albedo, Russian roulette) + rng.py's counter RNG.
// One tentative collision per ray per wavefront iteration, as pt_coord /
// pt_shade; the mega-kernel runs the same helpers to completion per ray.
struct PtState {
    float thr[3], rad[3], o[3], d[3], cp[3], alb[3], mu_s;         // PTF
    double t, t1, tau, cell_exit, tm[3], td[3];                      // PTD
    int64_t pixel, event, role, bounces, tau_pending, in_cell, c[3], st[3];  // PTI
};

// rng.py / _render_kernels.py:26-49: SplitMix64-style key hash -> float32 in [0,1)
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
__device__ __forceinline__ float u01(uint64_t seed, uint64_t frame, int64_t pixel, int64_t event) {
    uint64_t h = mix64(seed + 0x9E3779B97F4A7C15ull);
    h = mix64(h + frame * 0xD1B54A32D192ED03ull);
    h = mix64(h + (uint64_t)pixel * 0x8CB92BA72F3D8DD7ull);
    h = mix64(h + (uint64_t)event * 0x9E3779B97F4A7C15ull);
    return __fmul_rn((float)(h >> 40), 1.0f / 16777216.0f);
}

// The marcher's step-size and opacity formulas on their own (tracking.py adaptive_step /
// correct_opacity): which = 0: adaptive(x, s1 = a, s2 = b, p = c); which = 1: opacity x
// resampled from step s1 = b to step sbar = a, 1 - (1 - x)^(sbar / s1) -- the device functions
// the ray marcher evaluates (_render_kernels.py:244-253, 364-392).
__global__ void march_formula_kernel(int which, const float *__restrict__ x, int64_t n, float a, float b, float c,
                                     float *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = which == 0 ? adaptive(x[i], a, b, c) : 1.0f - powd(1.0f - x[i], a / b);
}

// The counter stream on its own (rng.py RngStream.uniform): the same u01 the path tracer draws
__global__ void rng_u01_kernel(uint64_t seed, uint64_t frame, const int64_t *__restrict__ pixel,
                               const int64_t *__restrict__ event, int64_t n, float *__restrict__ out) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = u01(seed, frame, pixel[i], event[i]);
}

// macrocell.py:159-181 dda_traverse / _render_kernels.py:153-188 dda_collect: every
// (cell, s_enter, s_exit) the macro-cell DDA walks along [t0, t1] of one float64 ray,
// zero-length grazes dropped (the segments tile the interval); the walk of cell_entry /
// cell_advance in float64 from the caller's origin / direction.  One thread.
__global__ void dda_collect_kernel(double ox, double oy, double oz, double dx, double dy, double dz, double t0,
                                   double t1, double ng, int64_t gx, int64_t gy, int64_t gz, int64_t cap,
                                   int64_t *__restrict__ cells, double *__restrict__ ts, int64_t *__restrict__ count) {
    const double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz};
    const int64_t gd[3] = {gx, gy, gz};
    int64_t c[3], st[3];
    double tm[3], td[3];
    for (int a = 0; a < 3; ++a) {
        const double p = o[a] + t0 * d[a];
        c[a] = clampl((int64_t)floor(p / ng), 0, gd[a] - 1);
        if (d[a] > 0.0) {
            st[a] = 1;
            tm[a] = t0 + ((double)(c[a] + 1) * ng - p) / d[a];
            td[a] = ng / d[a];
        } else if (d[a] < 0.0) {
            st[a] = -1;
            tm[a] = t0 + ((double)c[a] * ng - p) / d[a];
            td[a] = -ng / d[a];
        } else {
            st[a] = 0;
            tm[a] = INFINITY;
            td[a] = INFINITY;
        }
    }
    double cur = t0;
    int64_t k = 0;
    for (;;) {
        double se = tm[0];
        if (tm[1] < se) se = tm[1];
        if (tm[2] < se) se = tm[2];
        if (se > t1) se = t1;
        if (se > cur && k < cap) {
            for (int a = 0; a < 3; ++a) cells[3 * k + a] = clampl(c[a], 0, gd[a] - 1);
            ts[2 * k] = cur;
            ts[2 * k + 1] = se;
            ++k;
            cur = se;
        }
        if (se >= t1 || k >= cap) break;
        if (tm[0] <= tm[1] && tm[0] <= tm[2]) {
            c[0] += st[0];
            tm[0] += td[0];
        } else if (tm[1] <= tm[2]) {
            c[1] += st[1];
            tm[1] += td[1];
        } else {
            c[2] += st[2];
            tm[2] += td[2];
        }
    }
    *count = k;
}

// _render_kernels.py:92-138 _dda_enter for the PT state
__device__ void pt_dda_enter(const RmScene &S, PtState &P) {
    const double t0 = P.t, ng = S.ng;
    const int64_t gd[3] = {S.gx, S.gy, S.gz};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double o = (double)P.o[a], d = (double)P.d[a];
        const double p = o + t0 * d;
        const int64_t c = clampl((int64_t)floor(div_h(p, ng, S.ing)), 0, gd[a] - 1);
        P.c[a] = c;
        if (d > 0.0) {
            P.st[a] = 1;
            P.tm[a] = t0 + ((double)(c + 1) * ng - p) / d;
            P.td[a] = ng / d;
        } else if (d < 0.0) {
            P.st[a] = -1;
            P.tm[a] = t0 + ((double)c * ng - p) / d;
            P.td[a] = -ng / d;
        } else {
            P.st[a] = 0;
            P.tm[a] = INFINITY;
            P.td[a] = INFINITY;
        }
    }
}

__device__ __forceinline__ double pt_cell_exit(const PtState &P) {
    double se = P.tm[0];
    if (P.tm[1] < se) se = P.tm[1];
    if (P.tm[2] < se) se = P.tm[2];
    if (se > P.t1) se = P.t1;
    return se;
}

// _render_kernels.py:582-628 _pt_after_nee (true = ray done)
__device__ bool pt_after_nee(const RmScene &S, PtState &P) {
#pragma unroll
    for (int c = 0; c < 3; ++c) P.thr[c] = P.thr[c] * P.alb[c];
    const float u1 = u01(S.seed, S.frame, P.pixel, P.event++);
    const float u2 = u01(S.seed, S.frame, P.pixel, P.event++);
    const double zz = 1.0 - 2.0 * (double)u1;
    const double rr = sqrt(fmax(0.0, 1.0 - zz * zz));
    const double ph = (2.0 * 3.141592653589793) * (double)u2;
    P.d[0] = (float)(rr * cos(ph));
    P.d[1] = (float)(rr * sin(ph));
    P.d[2] = (float)zz;
#pragma unroll
    for (int a = 0; a < 3; ++a) P.o[a] = P.cp[a];
    double t0, t1;
    if (!isect(P.o[0], P.o[1], P.o[2], P.d[0], P.d[1], P.d[2], S.hx, S.hy, S.hz, t0, t1)) {
#pragma unroll
        for (int c = 0; c < 3; ++c) P.rad[c] = P.rad[c] + P.thr[c] * S.bg[c];
        P.role = 2;
        return true;
    }
    P.t = t0;
    P.t1 = t1;
    P.tau_pending = 0;
    P.in_cell = 0;
    if (P.bounces > S.rr_depth) {
        float q = P.thr[0];
        if (P.thr[1] > q) q = P.thr[1];
        if (P.thr[2] > q) q = P.thr[2];
        if (q > 1.0f) q = 1.0f;
        const float u = u01(S.seed, S.frame, P.pixel, P.event++);
        if (u >= q) {
            P.role = 2;
            return true;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) P.thr[c] = P.thr[c] / q;
    }
    P.role = 0;
    return false;
}

// _render_kernels.py:631-716 _pt_next: track until a tentative collision needs a
// field value (1, P.t set) or the ray resolves (-1)
__device__ float pt_next(const RmScene &S, const float *__restrict__ mu, PtState &P) {
    for (;;) {
        if (P.role == 2) return -1.0f;
        if (P.tau_pending == 0) {
            const float zeta = u01(S.seed, S.frame, P.pixel, P.event++);
            P.tau = -log1p(-(double)zeta);
            P.tau_pending = 1;
        }
        bool escape = false;
        if (S.use_mc) {
            if (P.in_cell == 0) {
                pt_dda_enter(S, P);
                P.cell_exit = pt_cell_exit(P);
                P.in_cell = 1;
            }
            const float muc = mu_read(S, mu, P.c[0], P.c[1], P.c[2]);
            if (muc > 0.0f) {
                const double seg = P.cell_exit - P.t;
                const double tauc = (double)muc * seg;
                if (P.tau <= tauc) {
                    P.t = P.t + P.tau / (double)muc;
                    P.mu_s = muc;
                    return 1.0f;
                }
                P.tau -= tauc;
            }
            if (P.cell_exit >= P.t1) {
                escape = true;
            } else {
                P.t = P.cell_exit;
                if (P.tm[0] <= P.tm[1] && P.tm[0] <= P.tm[2]) {
                    P.c[0] += P.st[0];
                    P.tm[0] = P.tm[0] + P.td[0];
                } else if (P.tm[1] <= P.tm[2]) {
                    P.c[1] += P.st[1];
                    P.tm[1] = P.tm[1] + P.td[1];
                } else {
                    P.c[2] += P.st[2];
                    P.tm[2] = P.tm[2] + P.td[2];
                }
                P.cell_exit = pt_cell_exit(P);
            }
        } else {
            if (S.mu_glob > 0.0) {
                const double seg = P.t1 - P.t;
                const double tauc = S.mu_glob * seg;
                if (P.tau <= tauc) {
                    P.t = P.t + P.tau / S.mu_glob;
                    P.mu_s = (float)S.mu_glob;
                    return 1.0f;
                }
            }
            escape = true;
        }
        if (escape) {
            if (P.role == 0) {
#pragma unroll
                for (int c = 0; c < 3; ++c) P.rad[c] = P.rad[c] + P.thr[c] * S.bg[c];
                P.role = 2;
                return -1.0f;
            }
            // shadow ray reached the light: T_sh = 1, take the NEE contribution
#pragma unroll
            for (int c = 0; c < 3; ++c) P.rad[c] = P.rad[c] + P.thr[c] * P.alb[c] * S.light[c];
            if (pt_after_nee(S, P)) return -1.0f;
        }
    }
}

// _render_kernels.py:719-736 _pt_stage_coord
__device__ void pt_stage_coord(const RmScene &S, const PtState &P, float &x, float &y, float &z) {
    const float one_below = __int_as_float(0x3f7fffff);
    const double h[3] = {S.hx, S.hy, S.hz}, ih[3] = {S.ihx, S.ihy, S.ihz};
    float v[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        float c = (float)div_h((double)P.o[a] + P.t * (double)P.d[a], h[a], ih[a]);
        if (c < 0.0f) c = 0.0f;
        if (c >= 1.0f) c = one_below;
        v[a] = c;
    }
    x = v[0];
    y = v[1];
    z = v[2];
}

// _render_kernels.py:739-780 _pt_consume: accept / reject the tentative collision (true = done)
__device__ bool pt_consume(const RmScene &S, PtState &P, float v, unsigned long long *violations) {
    const float mu = P.mu_s;
    float sig = tf_alpha(S.tf, v) * S.ds;
    if (sig > mu * 1.0001f) {
        atomicAdd(violations, 1ull);
        sig = mu;
    }
    const float xi = u01(S.seed, S.frame, P.pixel, P.event++);
    if (!((double)xi < (double)sig / (double)mu)) {
        P.tau_pending = 0;  // null collision: fresh tau from here
        return false;
    }
    if (P.role == 0) {
        P.bounces += 1;
        const double tc = P.t;
#pragma unroll
        for (int a = 0; a < 3; ++a) P.cp[a] = (float)((double)P.o[a] + tc * (double)P.d[a]);
        tf_rgb(S.tf, v, P.alb[0], P.alb[1], P.alb[2]);  // the collision's value doubles as albedo
        double t0, t1;
        if (!isect(P.cp[0], P.cp[1], P.cp[2], S.sd[0], S.sd[1], S.sd[2], S.hx, S.hy, S.hz, t0, t1)) {
#pragma unroll
            for (int c = 0; c < 3; ++c) P.rad[c] = P.rad[c] + P.thr[c] * P.alb[c] * S.light[c];
            return pt_after_nee(S, P);
        }
        P.role = 1;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            P.o[a] = P.cp[a];
            P.d[a] = S.sd[a];
        }
        P.t = t0;
        P.t1 = t1;
        P.tau_pending = 0;
        P.in_cell = 0;
        return false;
    }
    return pt_after_nee(S, P);  // shadow ray hit something: occluded, no NEE contribution
}

__device__ __forceinline__ void pt_write(const PtState &P, float *__restrict__ img) {
    img[3 * P.pixel] = P.rad[0];
    img[3 * P.pixel + 1] = P.rad[1];
    img[3 * P.pixel + 2] = P.rad[2];
}

// render.py:322-333 pt_state from the raygen / slab-test output
__global__ void pt_init_kernel(const RayState *__restrict__ rays, int64_t n, PtState *__restrict__ pts) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    const RayState R = rays[r];
    PtState P;
    memset(&P, 0, sizeof(P));
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        P.thr[a] = 1.0f;
        P.o[a] = R.o[a];
        P.d[a] = R.d[a];
    }
    P.t = R.t0;
    P.t1 = R.march_end;
    P.pixel = R.pixel;
    pts[r] = P;
}

// pt_coord (_render_kernels.py:830-852): one tentative collision per ray
__global__ void pt_coord_kernel(PtState *__restrict__ pts, int64_t n, const RmScene S, const float *__restrict__ mu,
                                float *__restrict__ sxyz, int32_t *__restrict__ counts, uint8_t *__restrict__ alive,
                                float *__restrict__ img) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    PtState P = pts[r];
    if (pt_next(S, mu, P) < 0.0f) {
        pt_write(P, img);
        counts[r] = 0;
        alive[r] = 0;
    } else {
        pt_stage_coord(S, P, sxyz[3 * r], sxyz[3 * r + 1], sxyz[3 * r + 2]);
        counts[r] = 1;
        alive[r] = 1;
    }
    pts[r] = P;
}

// pt_shade (_render_kernels.py:855-878)
__global__ void pt_shade_kernel(PtState *__restrict__ pts, int64_t n, const RmScene S,
                                const float *__restrict__ values, const int32_t *__restrict__ counts,
                                uint8_t *__restrict__ alive, float *__restrict__ img,
                                unsigned long long *__restrict__ violations) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n || counts[r] == 0) return;
    PtState P = pts[r];
    if (pt_consume(S, P, values[r], violations)) {
        pt_write(P, img);
        alive[r] = 0;
    }
    pts[r] = P;
}

// pt_reference (_render_kernels.py:783-827): the mega-kernel path tracer
template <int NN>
__global__ void __launch_bounds__(FE_THREADS) pt_mega_kernel(PtState *__restrict__ pts, int64_t n, const RmScene S,
                                                             const float *__restrict__ mu, const FieldDesc F,
                                                             const GridTables tab, const MlpShape sh, int maxw,
                                                             float *__restrict__ img,
                                                             unsigned long long *__restrict__ evals,
                                                             unsigned long long *__restrict__ violations) {
    extern __shared__ float4 smem4[];
    float *smem = reinterpret_cast<float *>(smem4);
    float *wt = smem;
    int wsz = F.use_grid ? 0 : stage_weights_t(F.weights, sh, wt);
    float *h0 = wt + wsz, *h1 = h0 + maxw * FE_THREADS;
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= n) return;
    PtState P = pts[r];
    unsigned long long ev = 0;
    float *col0 = h0 + threadIdx.x, *col1 = h1 + threadIdx.x;
    for (;;) {
        if (pt_next(S, mu, P) < 0.0f) break;
        float x, y, z;
        pt_stage_coord(S, P, x, y, z);
        float v;
        if (F.use_grid) {
            v = trilinear_at(F.norm, F.ndx, F.ndy, F.ndz, x, y, z);
        } else {
            encode_exact(x, y, z, F.params, tab, col0);
            if constexpr (NN > 0)
                v = mlp_exact_col<NN, false>(col0, tab.n_levels * tab.n_feat, wt, sh);
            else
                v = mlp_exact_smem(col0, col1, wt, sh);
        }
        ++ev;
        if (pt_consume(S, P, v, violations)) break;
    }
    pt_write(P, img);
    atomicAdd(evals, ev);
}

static void fill_cam(CamParams &C, const double *cp) {
    // cp: eye[3], fwd[3], right[3], up[3], tan_half, aspect, width, height, row0, nrows
    for (int a = 0; a < 3; ++a) {
        C.eye[a] = (float)cp[a];
        C.fwd[a] = cp[3 + a];
        C.right[a] = cp[6 + a];
        C.up[a] = cp[9 + a];
    }
    C.tan_half = cp[12];
    C.aspect = cp[13];
    C.width = (int64_t)cp[14];
    C.height = (int64_t)cp[15];
    C.row0 = (int64_t)cp[16];
    C.nrows = (int64_t)cp[17];
}

constexpr int RM_HIST_CAP = 1 << 16;  // wavefront iterations recorded on the device per frame

struct RenderWs {
    RayState *rays;            // the hit rays, in pixel order (fixed for the frame)
    int32_t *ids[2];           // alive ray indices (ping-pong), then hit pixel ids at setup
    uint8_t *flags;
    float *sxyz, *sts, *ssbar, *values, *dxyz, *dvals;
    int32_t *counts, *offs, *dtotal, *coord_rays, *coord_hist, *dray;
    unsigned long long *evals;
    int64_t *nsel, *nact;
    void *cub_tmp;
    size_t cub_bytes;
    int64_t total;
};

static int64_t al256(int64_t x) { return (x + 255) & ~(int64_t)255; }

static RenderWs carve(void *base, int64_t npix, int k) {
    RenderWs w{};
    char *p = (char *)base;
    int64_t off = 0;
    auto take = [&](int64_t bytes) {
        char *r = p ? p + off : nullptr;
        off += al256(bytes);
        return r;
    };
    w.rays = (RayState *)take(npix * (int64_t)sizeof(RayState));
    w.ids[0] = (int32_t *)take(npix * 4);
    w.ids[1] = (int32_t *)take(npix * 4);
    w.flags = (uint8_t *)take(npix);
    w.sxyz = (float *)take(npix * k * 12);
    w.sts = (float *)take(npix * k * 4);
    w.ssbar = (float *)take(npix * k * 4);
    w.values = (float *)take(npix * k * 4);
    w.counts = (int32_t *)take(npix * 4);
    w.offs = (int32_t *)take(npix * 4);
    w.dxyz = (float *)take(npix * k * 12);
    w.dvals = (float *)take(npix * k * 4);
    w.dray = (int32_t *)take(npix * k * 4);
    w.dtotal = (int32_t *)take(8);
    w.coord_rays = (int32_t *)take(8);
    w.coord_hist = (int32_t *)take(4 * (int64_t)RM_HIST_CAP);
    w.evals = (unsigned long long *)take(8);
    w.nsel = (int64_t *)take(8);
    w.nact = (int64_t *)take(8);
    size_t cb = 0, cs = 0;
    cub::DeviceSelect::Flagged(nullptr, cb, (int32_t *)nullptr, (uint8_t *)nullptr, (int32_t *)nullptr,
                               (int64_t *)nullptr, (int64_t)npix);
    cub::DeviceScan::ExclusiveSum(nullptr, cs, (int32_t *)nullptr, (int32_t *)nullptr, (int)npix);
    cb = cb > cs ? cb : cs;
    w.cub_bytes = cb;
    w.cub_tmp = take((int64_t)cb);
    w.total = off;
    return w;
}

int field_exact_launch(const float *coords, int64_t b, const float *params, const GridTables &tab,
                       const float *weights, const int32_t *widths, int32_t n_layers, int32_t relu_out, int decode,
                       int64_t dx, int64_t dy, int64_t dz, int64_t z0, double lo, double scale, float *out,
                       cudaStream_t s);
int infer_tc_launch(const float *coords, int64_t b, const float *params, const GridTables &tab, const float *wflat,
                    uint8_t *wimg, int nn, int nh, int relu_out, int decode, int64_t dx, int64_t dy, int64_t dz,
                    int64_t z0, double lo, double scale, float *out, cudaStream_t s, bool pack,
                    const int32_t *b_dev = nullptr);
int pack_mlp_image(const float *wflat, int nin, int ninp, int nn, int nh, const uint32_t *o_w, uint32_t o_wout,
                   uint8_t *image, cudaStream_t s, const uint32_t *o_wlo);

// pt_coord staging has exactly one sample per alive ray: count it for the frame stats
__global__ void count_staged_kernel(const int32_t *__restrict__ counts, int64_t n,
                                    unsigned long long *__restrict__ evals) {
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    unsigned long long c = (r < n) ? (unsigned long long)counts[r] : 0ull;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(evals, c);
}

// render.py:355-368 (pt_reference) and 396-423 (pathtrace branch of render_wavefront)
static int render_pathtrace(const RmScene &S, const RenderWs &w, RayState *hits, int64_t n, const float *mu,
                            const FieldDesc &F, const GridTables &tab, const MlpShape &sh, int maxw,
                            const int32_t *widths, int32_t n_layers, int32_t relu_out, int32_t architecture,
                            int32_t eval_mode, void *mlp_image, float *img, int32_t *alive_hist, int32_t max_hist,
                            unsigned long long *violations, int &iters, cudaStream_t s) {
    iters = 0;
    if (n == 0) return NVOL_OK;
    PtState *pts[2] = {nullptr, nullptr};
    size_t sel_bytes = 0;
    cub::DeviceSelect::Flagged(nullptr, sel_bytes, (PtState *)nullptr, (uint8_t *)nullptr, (PtState *)nullptr,
                               (int64_t *)nullptr, n);
    void *sel_tmp = nullptr;
    if (cudaMallocAsync((void **)&pts[0], sizeof(PtState) * (size_t)n, s) != cudaSuccess ||
        cudaMallocAsync((void **)&pts[1], sizeof(PtState) * (size_t)n, s) != cudaSuccess ||
        cudaMallocAsync(&sel_tmp, sel_bytes, s) != cudaSuccess)
        return check_launch("pathtrace state alloc");
    pt_init_kernel<<<grid_for(n, 256), 256, 0, s>>>(hits, n, pts[0]);
    int st = check_launch("pt_init");
    int cur = 0;
    if (st == NVOL_OK && architecture == 1) {
        int wtot = 0;
        for (int i = 0; i < (F.use_grid ? 0 : n_layers); ++i) wtot += widths[i] * widths[i + 1];
        int nn = (!F.use_grid && n_layers >= 2) ? widths[1] : 0;
        bool uniform = !F.use_grid && n_layers >= 2;
        for (int i = 1; i < n_layers && uniform; ++i) uniform &= widths[i] == nn;
        const bool regpath = uniform && (nn == 16 || nn == 32 || nn == 64);  // one activation column
        size_t smem = sizeof(float) * (((wtot + 3) & ~3) +
                                       (regpath ? (size_t)max((int)widths[0], nn) : 2 * (size_t)maxw) * FE_THREADS);
        unsigned grid = grid_for(n, FE_THREADS);
#define LAUNCH_PT(NNV)                                                                                        \
    do {                                                                                                      \
        cudaFuncSetAttribute(pt_mega_kernel<NNV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);    \
        pt_mega_kernel<NNV><<<grid, FE_THREADS, smem, s>>>(pts[0], n, S, mu, F, tab, sh, maxw, img, w.evals,  \
                                                           violations);                                       \
    } while (0)
        if (uniform && nn == 16)
            LAUNCH_PT(16);
        else if (uniform && nn == 32)
            LAUNCH_PT(32);
        else if (uniform && nn == 64)
            LAUNCH_PT(64);
        else
            LAUNCH_PT(0);
#undef LAUNCH_PT
        st = check_launch("pt_mega_kernel");
        if (max_hist > 0) alive_hist[0] = (int32_t)n;
        iters = 1;
    } else {
        while (st == NVOL_OK && n > 0) {
            if (iters < max_hist) alive_hist[iters] = (int32_t)n;
            ++iters;
            PtState *ps = pts[cur];
            pt_coord_kernel<<<grid_for(n, 128), 128, 0, s>>>(ps, n, S, mu, w.sxyz, w.counts, w.flags, img);
            count_staged_kernel<<<grid_for(n, 256), 256, 0, s>>>(w.counts, n, w.evals);
            // dense evaluation of the staged collisions (rays that resolved stage none)
            size_t cb = w.cub_bytes;
            cub::DeviceScan::ExclusiveSum(w.cub_tmp, cb, w.counts, w.offs, (int)n, s);
            compact_staged_kernel<<<grid_for(n, 256), 256, 0, s>>>(w.sxyz, w.counts, w.offs, n, 1, w.dxyz, w.dtotal);
            int32_t ns32 = 0;
            cudaMemcpyAsync(&ns32, w.dtotal, 4, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (ns32 > 0) {
                if (F.use_grid) {
                    st = ::nvol_trilinear(F.norm, F.ndx, F.ndy, F.ndz, w.dxyz, ns32, w.dvals, s);
                } else if (eval_mode == 1) {
                    st = infer_tc_launch(w.dxyz, ns32, F.params, tab, F.weights, (uint8_t *)mlp_image, widths[1],
                                         n_layers - 1, relu_out, 0, 0, 0, 0, 0, 0.0, 1.0, w.dvals, s, iters == 1);
                } else {
                    st = field_exact_launch(w.dxyz, ns32, F.params, tab, F.weights, widths, n_layers, relu_out, 0,
                                            0, 0, 0, 0, 0.0, 1.0, w.dvals, s);
                }
                if (st) break;
                scatter_staged_kernel<<<grid_for(n, 256), 256, 0, s>>>(w.dvals, w.counts, w.offs, n, 1, w.values);
            }
            pt_shade_kernel<<<grid_for(n, 128), 128, 0, s>>>(ps, n, S, w.values, w.counts, w.flags, img, violations);
            st = check_launch("pt_shade");
            if (st) break;
            cub::DeviceSelect::Flagged(sel_tmp, sel_bytes, ps, w.flags, pts[cur ^ 1], w.nsel, n, s);
            cudaMemcpyAsync(&n, w.nsel, 8, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            cur ^= 1;
        }
    }
    cudaFreeAsync(pts[0], s);
    cudaFreeAsync(pts[1], s);
    cudaFreeAsync(sel_tmp, s);
    return st;
}

}  // namespace nvol

using namespace nvol;

extern "C" {

int64_t nvol_render_workspace_bytes(int64_t n_pixels, int32_t k_batch) {
    return carve(nullptr, n_pixels, k_batch < 1 ? 1 : k_batch).total;
}

// render.py:383-454 render_wavefront (architecture 0) or render.py:347-380
// render_reference (architecture 1, in-shader).  See nvol.h.
int nvol_render(const double *cam_params, const double *render_params, const float *tf_cv, const float *tf_crgb,
                int32_t ncv, const float *tf_ov, const float *tf_oa, int32_t nov, const float *mu, int64_t gx,
                int64_t gy, int64_t gz, int32_t use_grid, const float *norm, int64_t ndx, int64_t ndy, int64_t ndz,
                const float *params, const int64_t *level_off, const int64_t *level_res, const int64_t *level_entries,
                const uint8_t *level_dense, int32_t n_levels, int32_t n_feat, const float *weights,
                const int32_t *widths, int32_t n_layers, int32_t relu_out, int32_t architecture, int32_t eval_mode,
                void *mlp_image, float *img, void *workspace, int64_t workspace_bytes, int64_t *stats_out,
                int32_t *alive_hist, int32_t max_hist, void *stream) {
    cudaStream_t s = as_stream(stream);
    RmScene S;
    int st = fill_scene(S, render_params, tf_cv, tf_crgb, ncv, tf_ov, tf_oa, nov, gx, gy, gz);
    if (st) return st;
    NVOL_REQUIRE(mu && img && workspace && stats_out, "null pointer");
    CamParams C;
    fill_cam(C, cam_params);
    NVOL_REQUIRE(C.row0 >= 0 && C.nrows >= 1 && C.row0 + C.nrows <= C.height, "bad image tile rows");
    const int64_t npix = C.width * C.nrows;
    const int K = S.k_batch < 1 ? 1 : S.k_batch;
    RenderWs w = carve(workspace, npix, K);
    NVOL_REQUIRE(workspace_bytes >= w.total, "render workspace too small");
    GridTables tab{};
    MlpShape sh{};
    int maxw = 1;
    FieldDesc F{use_grid, norm, ndx, ndy, ndz, params, weights};
    if (!use_grid) {
        st = pack_tables(tab, level_off, level_res, level_entries, level_dense, n_levels, n_feat);
        if (st) return st;
        NVOL_REQUIRE(n_layers >= 1 && n_layers <= 11, "MLP depth out of range");
        sh.n_layers = n_layers;
        sh.relu_out = relu_out;
        for (int i = 0; i <= n_layers; ++i) {
            sh.widths[i] = widths[i];
            maxw = max(maxw, (int)widths[i]);
        }
    } else {
        NVOL_REQUIRE(norm, "grid field without data");
    }
    cudaMemsetAsync(w.evals, 0, 8, s);
    ray_hits_kernel<<<grid_for(npix, 256), 256, 0, s>>>(C, S, w.flags, img);
    iota_kernel<<<grid_for(npix, 256), 256, 0, s>>>(w.ids[0], npix);
    st = check_launch("ray_hits");
    if (st) return st;
    cub::DeviceSelect::Flagged(w.cub_tmp, w.cub_bytes, w.ids[0], w.flags, w.ids[1], w.nsel, npix, s);
    int64_t n = 0;
    cudaMemcpyAsync(&n, w.nsel, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    // ray records up front for the path tracer and the in-shader marcher; the wavefront
    // ray march generates each ray inside its first rm_step (no record write + read)
    // the in-shader marcher on the tensor cores (architecture 1, tcgen05 evaluator): rays are
    // generated inside rm_tc_kernel, so no ray records
    InferShape ish{};
    const bool tc_inshader = architecture == 1 && eval_mode == 1 && !use_grid && !S.pathtrace && n_layers >= 2 &&
                             widths[n_layers] == 1 && widths[0] == n_levels * n_feat &&
                             build_infer_shape(ish, n_levels, n_feat, widths[1], n_layers - 1, relu_out) &&
                             [&] {
                                 for (int i = 1; i < n_layers; ++i)
                                     if (widths[i] != widths[1]) return false;
                                 for (int l = 0; l < n_levels; ++l)
                                     if (level_entries[l] >= (1ll << 31)) return false;
                                 return true;
                             }();
    if (n > 0 && (S.pathtrace || (architecture == 1 && !tc_inshader))) {
        raygen_kernel<<<(unsigned)((n + RG_THREADS - 1) / RG_THREADS), RG_THREADS, 0, s>>>(C, S, w.ids[1], n, w.rays);
        st = check_launch("raygen");
        if (st) return st;
    }
    int iters = 0;
    if (S.pathtrace) {
        unsigned long long *viol = nullptr;
        if (cudaMallocAsync((void **)&viol, 8, s) != cudaSuccess) return check_launch("pathtrace alloc");
        cudaMemsetAsync(viol, 0, 8, s);
        st = render_pathtrace(S, w, w.rays, n, mu, F, tab, sh, maxw, widths, n_layers, relu_out, architecture,
                              eval_mode, mlp_image, img, alive_hist, max_hist, viol, iters, s);
        if (st) return st;
        unsigned long long ev = 0, vi = 0;
        cudaMemcpyAsync(&ev, w.evals, 8, cudaMemcpyDeviceToHost, s);
        cudaMemcpyAsync(&vi, viol, 8, cudaMemcpyDeviceToHost, s);
        cudaFreeAsync(viol, s);
        cudaStreamSynchronize(s);
        stats_out[0] = (int64_t)ev;
        stats_out[1] = iters;
        stats_out[2] = (int64_t)vi;
        return check_launch("render (pathtrace)");
    }
    if (tc_inshader) {
        if (n > 0) {
            NVOL_REQUIRE(mlp_image, "the tcgen05 evaluator needs an mlp_image scratch buffer (nvol_mlp_image_bytes)");
            st = pack_mlp_image(weights, ish.nin, ish.ninp, widths[1], n_layers - 1, ish.o_w, ish.o_wout,
                                (uint8_t *)mlp_image, s, ish.o_wlo);
            if (st) return st;
            cudaMemsetAsync(w.coord_rays, 0, 4, s);  // the ray queue
            int dev = 0, sms = 148;
            cudaGetDevice(&dev);
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
            const int64_t ctas = (n + IT_THREADS - 1) / IT_THREADS;
            const int grid = (int)(ctas < 2 * sms ? ctas : 2 * sms);
            auto go = [&](auto kern) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ish.smem_bytes);
                kern<<<grid, IT_THREADS, ish.smem_bytes, s>>>(w.ids[1], n, w.coord_rays, C, S, mu, params, tab, ish,
                                                              (const uint8_t *)mlp_image, img, w.evals);
            };
            switch (n_feat) {
                case 1: go(rm_tc_kernel<1>); break;
                case 2: go(rm_tc_kernel<2>); break;
                case 4: go(rm_tc_kernel<4>); break;
                default: go(rm_tc_kernel<8>); break;
            }
            st = check_launch("rm_tc_kernel");
            if (st) return st;
        }
        if (max_hist > 0) alive_hist[0] = (int32_t)n;
        iters = 1;
    } else if (architecture == 1) {
        // in-shader: one thread per ray to completion
        if (n > 0) {
            int wtot = 0;
            for (int i = 0; i < (use_grid ? 0 : n_layers); ++i) wtot += widths[i] * widths[i + 1];
            int nn = (!use_grid && n_layers >= 2) ? widths[1] : 0;
            bool uniform = !use_grid && n_layers >= 2;
            for (int i = 1; i < n_layers && uniform; ++i) uniform &= widths[i] == nn;
            const bool regpath = uniform && (nn == 16 || nn == 32 || nn == 64);  // one activation column
            size_t smem = sizeof(float) * (((wtot + 3) & ~3) +
                                           (regpath ? (size_t)max((int)widths[0], nn) : 2 * (size_t)maxw) * FE_THREADS);
            unsigned grid = grid_for(n, FE_THREADS);
#define LAUNCH_MK(NNV)                                                                                            \
    do {                                                                                                          \
        cudaFuncSetAttribute(rm_mega_kernel<NNV>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);        \
        rm_mega_kernel<NNV><<<grid, FE_THREADS, smem, s>>>(w.rays, n, S, mu, F, tab, sh, maxw, img, w.evals); \
    } while (0)
            if (uniform && nn == 16)
                LAUNCH_MK(16);
            else if (uniform && nn == 32)
                LAUNCH_MK(32);
            else if (uniform && nn == 64)
                LAUNCH_MK(64);
            else
                LAUNCH_MK(0);
#undef LAUNCH_MK
            st = check_launch("rm_mega_kernel");
            if (st) return st;
        }
        if (max_hist > 0) alive_hist[0] = (int32_t)n;
        iters = 1;
    } else {
        // alive rays: initially every hit ray (ids = 0..n-1)
        iota_kernel<<<grid_for(n, 256), 256, 0, s>>>(w.ids[0], n);
        static int force_sync = -1;  // NVOL_RENDER_SYNC=1: the synchronous loop below (A/B, tests)
        if (force_sync < 0) {
            const char *e = getenv("NVOL_RENDER_SYNC");
            force_sync = (e && atoi(e) != 0) ? 1 : 0;
        }
        if (eval_mode == 1 && !use_grid && n > 0 && !force_sync) {
            // Host-sync-free schedule (tcgen05 evaluator): every stage reads its live
            // count from the device (alive rays: nact, staged samples: dtotal) and is
            // launched on an upper bound, so iterations queue back to back; the host
            // only reads each iteration's alive count one iteration late, to tighten
            // the bound and to stop.  Per-iteration marcher counts land in coord_hist.
            // pinned read-back slots + events, per host thread and device (events belong to a device)
            struct CountSlots {
                int64_t *h = nullptr;
                cudaEvent_t ev[2];
            };
            static thread_local CountSlots slots[64];
            int dev = 0;
            cudaGetDevice(&dev);
            NVOL_REQUIRE(dev >= 0 && dev < 64, "device index out of range");
            CountSlots &cs = slots[dev];
            if (!cs.h) {
                if (cudaHostAlloc((void **)&cs.h, 2 * sizeof(int64_t), cudaHostAllocDefault) != cudaSuccess)
                    return check_launch("render pinned counters");
                cudaEventCreateWithFlags(&cs.ev[0], cudaEventDisableTiming);
                cudaEventCreateWithFlags(&cs.ev[1], cudaEventDisableTiming);
            }
            int64_t *h_cnt = cs.h;
            cudaEvent_t *ev_cnt = cs.ev;
            set_count_kernel<<<1, 1, 0, s>>>(w.nact, n);
            cudaMemsetAsync(w.coord_hist, 0, 4 * (size_t)RM_HIST_CAP, s);
            int64_t bound = n;
            int cur = 0, it = 0;
            for (;;) {
                const int slot = it < RM_HIST_CAP ? it : RM_HIST_CAP - 1;
                cudaMemsetAsync(w.dtotal, 0, 4, s);
                rm_step_kernel<<<grid_for(bound, 128), 128, 0, s>>>(w.ids[cur], bound, w.nact, w.rays, S, mu,
                                                                     it > 0 ? 1 : 0, w.values, w.sxyz, w.sts, w.ssbar,
                                                                     w.flags, img, w.evals,
                                                                     w.coord_hist + slot, C,
                                                                     it == 0 ? w.ids[1] : nullptr, w.dxyz, w.dray,
                                                                     w.dtotal);
                cub::DeviceSelect::Flagged(w.cub_tmp, w.cub_bytes, w.ids[cur], w.flags, w.ids[cur ^ 1], w.nact,
                                           bound, s);
                st = infer_tc_launch(w.dxyz, bound * K, params, tab, weights, (uint8_t *)mlp_image, widths[1],
                                     n_layers - 1, relu_out, 0, 0, 0, 0, 0, 0.0, 1.0, w.dvals, s, it == 0, w.dtotal);
                if (st) return st;
                scatter_dense_kernel<<<dense_grid(bound * K), 256, 0, s>>>(w.dvals, w.dray, w.dtotal, bound * K,
                                                                               w.values);
                st = check_launch("render iteration");
                if (st) return st;
                cudaMemcpyAsync(&h_cnt[it & 1], w.nact, 8, cudaMemcpyDeviceToHost, s);
                cudaEventRecord(ev_cnt[it & 1], s);
                if (it >= 1) {
                    cudaEventSynchronize(ev_cnt[(it - 1) & 1]);
                    const int64_t alive = h_cnt[(it - 1) & 1];  // rays entering iteration `it`
                    if (alive == 0) break;                      // iteration `it` had nothing to do
                    bound = alive;                              // bounds every later iteration
                }
                cur ^= 1;
                ++it;
            }
            const int nh = (it + 1) < RM_HIST_CAP ? it + 1 : RM_HIST_CAP;
            int32_t *hist = (int32_t *)malloc(4 * (size_t)nh);
            cudaMemcpyAsync(hist, w.coord_hist, 4 * (size_t)nh, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            for (int i = 0; i < nh && hist[i] > 0; ++i) {
                if (iters < max_hist) alive_hist[iters] = hist[i];
                ++iters;
            }
            free(hist);
            n = 0;
        }

        int cur = 0;
        bool shade = false;
        while (n > 0) {
            // shade the previous iteration's samples, stage this iteration's (one ray record pass)
            cudaMemsetAsync(w.coord_rays, 0, 4, s);
            cudaMemsetAsync(w.dtotal, 0, 4, s);
            rm_step_kernel<<<grid_for(n, 128), 128, 0, s>>>(w.ids[cur], n, nullptr, w.rays, S, mu, shade ? 1 : 0, w.values,
                                                             w.sxyz, w.sts, w.ssbar, w.flags, img, w.evals,
                                                             w.coord_rays, C, shade ? nullptr : w.ids[1], w.dxyz, w.dray,
                                                             w.dtotal);
            st = check_launch("rm_step");
            if (st) return st;
            shade = true;
            // dense evaluation of the staged samples + the next alive list, one host sync
            cub::DeviceSelect::Flagged(w.cub_tmp, w.cub_bytes, w.ids[cur], w.flags, w.ids[cur ^ 1], w.nsel, n, s);
            int32_t hv[2] = {0, 0};
            int64_t nn_next = 0;
            cudaMemcpyAsync(&hv[0], w.dtotal, 4, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(&hv[1], w.coord_rays, 4, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(&nn_next, w.nsel, 8, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            const int64_t ns = hv[0];
            if (hv[1] > 0) {
                if (iters < max_hist) alive_hist[iters] = hv[1];
                ++iters;
            }
            if (ns > 0) {
                if (use_grid) {
                    extern int nvol_trilinear(const float *, int64_t, int64_t, int64_t, const float *, int64_t, float *,
                                              void *);
                    st = nvol_trilinear(norm, ndx, ndy, ndz, w.dxyz, ns, w.dvals, stream);
                } else if (eval_mode == 1) {
                    int nnv = widths[1];
                    st = infer_tc_launch(w.dxyz, ns, params, tab, weights, (uint8_t *)mlp_image, nnv, n_layers - 1,
                                         relu_out, 0, 0, 0, 0, 0, 0.0, 1.0, w.dvals, s, /*pack=*/iters == 1);
                } else {
                    st = field_exact_launch(w.dxyz, ns, params, tab, weights, widths, n_layers, relu_out, 0, 0, 0, 0,
                                            0, 0.0, 1.0, w.dvals, s);
                }
                if (st) return st;
                scatter_dense_kernel<<<dense_grid(ns), 256, 0, s>>>(w.dvals, w.dray, w.dtotal, ns, w.values);
            }
            n = nn_next;
            cur ^= 1;
        }
    }
    unsigned long long ev = 0;
    cudaMemcpyAsync(&ev, w.evals, 8, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    stats_out[0] = (int64_t)ev;
    stats_out[1] = iters;
    stats_out[2] = 0;
    return check_launch("render");
}



int nvol_macrocell_ranges(const float *vals, int64_t dx, int64_t dy, int64_t dz, int64_t ng, int32_t clip,
                          float *lo, float *hi, void *stream) {
    NVOL_REQUIRE(vals && lo && hi && ng >= 1, "bad arguments");
    int64_t gx = (dx + ng - 1) / ng, gy = (dy + ng - 1) / ng, gz = (dz + ng - 1) / ng;
    mc_ranges_kernel<<<(unsigned)(gx * gy * gz), 256, 0, as_stream(stream)>>>(vals, dx, dy, dz, ng, gx, gy, gz, clip,
                                                                               lo, hi);
    return check_launch("macrocell_ranges");
}

int nvol_march_formula(int32_t which, const float *x, int64_t n, float a, float b, float c, float *out, void *stream) {
    NVOL_REQUIRE((which == 0 || which == 1) && n >= 0 && (n == 0 || (x && out)), "bad arguments");
    if (n == 0) return NVOL_OK;
    march_formula_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, as_stream(stream)>>>(which, x, n, a,
                                                                                                            b, c, out);
    return check_launch("march_formula");
}

int nvol_rng_u01(uint64_t seed, uint64_t frame, const int64_t *pixel, const int64_t *event, int64_t n, float *out,
                 void *stream) {
    NVOL_REQUIRE(n >= 0 && (n == 0 || (pixel && event && out)), "bad arguments");
    if (n == 0) return NVOL_OK;
    rng_u01_kernel<<<(unsigned)std::min<int64_t>((n + 255) / 256, 1024), 256, 0, as_stream(stream)>>>(seed, frame, pixel,
                                                                                                      event, n, out);
    return check_launch("rng_u01");
}

int nvol_dda_collect(const double *ray, double t0, double t1, double ng, int64_t gx, int64_t gy, int64_t gz,
                     int64_t cap, int64_t *cells, double *ts, int64_t *count, void *stream) {
    NVOL_REQUIRE(ray && cells && ts && count && cap >= 1 && ng > 0.0 && gx >= 1 && gy >= 1 && gz >= 1,
                 "bad arguments");
    dda_collect_kernel<<<1, 1, 0, as_stream(stream)>>>(ray[0], ray[1], ray[2], ray[3], ray[4], ray[5], t0, t1, ng, gx,
                                                       gy, gz, cap, cells, ts, count);
    return check_launch("dda_collect");
}

int nvol_macrocell_set_tf(const float *lo, const float *hi, int64_t ncell, const double *op_v, const double *op_a,
                          int32_t nop, double density_scale, float *mu, void *stream) {
    NVOL_REQUIRE(lo && hi && mu && nop >= 1 && nop <= MAX_TF, "bad arguments");
    OpacityPts P;
    P.n = nop;
    for (int i = 0; i < nop; ++i) {
        P.v[i] = op_v[i];
        P.a[i] = op_a[i];
    }
    if (ncell == 0) return NVOL_OK;
    mc_set_tf_kernel<<<grid_for(ncell, 256), 256, 0, as_stream(stream)>>>(lo, hi, ncell, P, density_scale, mu);
    return check_launch("macrocell_set_tf");
}

}  // extern "C"
