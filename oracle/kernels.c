/*
 * ORACLE — test infrastructure only.  CPU restatement of the reference's
 * numba kernels (arxiv 2207.11620 CPU reference, /root/reference/pkg/src/neuralvol)
 * for the hash-grid training / decode / render hot path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library, and only as the checker / CPU baseline; the product
 * path (paper_2207_11620_b200/) never links or calls it.
 *
 * Numerical contract: every function keeps the reference's float32 operation
 * order with no FMA contraction (compiled with -ffp-contract=off), so results
 * are bit-identical to the numba kernels they restate.  Parallel loops only
 * split work whose per-element arithmetic is independent (samples, levels,
 * parameters), so OpenMP does not change any value.
 *
 * Pinned against golden vectors produced by importing the reference in the
 * build container (oracle/gen_golden.py -> tests/golden/*.npz).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef unsigned __int128 u128;

/* encoding.py:22 HASH_PRIMES; _kernels.py:22-28 _vertex_slot.
 * Hashed levels always have entries == T = 2^k (encoding.py:160-164), so the
 * u32-wrapped XOR taken mod entries equals numba's u64-widened version. */
static inline int64_t vertex_slot(int64_t vx, int64_t vy, int64_t vz, int64_t res,
                                  int64_t entries, int dense) {
    if (dense) {
        int64_t r1 = res + 1;
        return (vz * r1 + vy) * r1 + vx;
    }
    uint32_t h = ((uint32_t)vx * 1u) ^ ((uint32_t)vy * 2654435761u) ^ ((uint32_t)vz * 805459861u);
    return (int64_t)(h % (uint32_t)entries);
}

static inline int64_t clampi(int64_t v, int64_t lo, int64_t hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}

int orc_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

/* _kernels.py:31-79 grid_encode_fwd.  idx_cache / w_cache may be NULL. */
void orc_grid_encode_fwd(const float *coords, int64_t b, const float *params,
                         const int64_t *level_off, const int64_t *level_res,
                         const int64_t *level_entries, const uint8_t *level_dense,
                         int m, int n_feat, int64_t *idx_cache, float *w_cache, float *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < b; ++i) {
        float *o = out + i * (int64_t)m * n_feat;
        for (int j = 0; j < m * n_feat; ++j) o[j] = 0.0f;
        for (int l = 0; l < m; ++l) {
            int64_t res = level_res[l];
            float sx = coords[3 * i + 0] * (float)res;
            float sy = coords[3 * i + 1] * (float)res;
            float sz = coords[3 * i + 2] * (float)res;
            int64_t cx = clampi((int64_t)floorf(sx), 0, res - 1);
            int64_t cy = clampi((int64_t)floorf(sy), 0, res - 1);
            int64_t cz = clampi((int64_t)floorf(sz), 0, res - 1);
            float fx = sx - (float)cx, fy = sy - (float)cy, fz = sz - (float)cz;
            int dense = level_dense[l] != 0;
            for (int c = 0; c < 8; ++c) {
                int ox = c & 1, oy = (c >> 1) & 1, oz = (c >> 2) & 1;
                int64_t slot = vertex_slot(cx + ox, cy + oy, cz + oz, res, level_entries[l], dense);
                float w = ox ? fx : 1.0f - fx;
                w *= oy ? fy : 1.0f - fy;
                w *= oz ? fz : 1.0f - fz;
                int64_t base = level_off[l] + slot * n_feat;
                int64_t ci = (i * m + l) * 8 + c;
                if (idx_cache) idx_cache[ci] = base;
                if (w_cache) w_cache[ci] = w;
                for (int f = 0; f < n_feat; ++f) o[l * n_feat + f] += w * params[base + f];
            }
        }
    }
}

/* _kernels.py:82-92 grid_encode_bwd.  The reference scatters serially in
 * i -> l -> c -> f order.  Levels own disjoint parameter ranges
 * (encoding.py:165), so one thread per level reproduces the serial per-entry
 * summation order exactly. */
void orc_grid_encode_bwd(const float *dl_dfeat, const int64_t *idx_cache, const float *w_cache,
                         int64_t b, int m, int n_feat, float *grad_out) {
    #pragma omp parallel for schedule(dynamic, 1)
    for (int l = 0; l < m; ++l) {
        for (int64_t i = 0; i < b; ++i) {
            for (int c = 0; c < 8; ++c) {
                int64_t ci = (i * m + l) * 8 + c;
                int64_t base = idx_cache[ci];
                float w = w_cache[ci];
                for (int f = 0; f < n_feat; ++f)
                    grad_out[base + f] += w * dl_dfeat[i * (int64_t)m * n_feat + l * n_feat + f];
            }
        }
    }
}

/* _kernels.py:95-117 _mlp_row + _kernels.py:120-151 _field_one +
 * _kernels.py:154-176 field_eval_model: fused per-sample encode + serial
 * float32 matvec chain, bias-free, ReLU on hidden layers (and output if
 * relu_out).  weights: concatenated row-major W_i (out x in); widths[0..nl]. */
float orc_field_one(float x, float y, float z, const float *params, const int64_t *level_off,
                       const int64_t *level_res, const int64_t *level_entries,
                       const uint8_t *level_dense, int m, int n_feat, const float *weights,
                       const int *widths, int nl, int relu_out, float *h0, float *h1) {
    int nin = m * n_feat;
    for (int j = 0; j < nin; ++j) h0[j] = 0.0f;
    for (int l = 0; l < m; ++l) {
        int64_t res = level_res[l];
        float sx = x * (float)res, sy = y * (float)res, sz = z * (float)res;
        int64_t cx = clampi((int64_t)floorf(sx), 0, res - 1);
        int64_t cy = clampi((int64_t)floorf(sy), 0, res - 1);
        int64_t cz = clampi((int64_t)floorf(sz), 0, res - 1);
        float fx = sx - (float)cx, fy = sy - (float)cy, fz = sz - (float)cz;
        int dense = level_dense[l] != 0;
        for (int c = 0; c < 8; ++c) {
            int ox = c & 1, oy = (c >> 1) & 1, oz = (c >> 2) & 1;
            int64_t slot = vertex_slot(cx + ox, cy + oy, cz + oz, res, level_entries[l], dense);
            float w = ox ? fx : 1.0f - fx;
            w *= oy ? fy : 1.0f - fy;
            w *= oz ? fz : 1.0f - fz;
            int64_t base = level_off[l] + slot * n_feat;
            for (int f = 0; f < n_feat; ++f) h0[l * n_feat + f] += w * params[base + f];
        }
    }
    float *cur = h0, *nxt = h1;
    const float *w = weights;
    for (int li = 0; li < nl; ++li) {
        int win = widths[li], wout = widths[li + 1];
        for (int j = 0; j < wout; ++j) {
            float acc = 0.0f;
            for (int k = 0; k < win; ++k) acc += w[j * win + k] * cur[k];
            if (li < nl - 1 || relu_out) acc = acc > 0.0f ? acc : 0.0f;
            nxt[j] = acc;
        }
        w += (int64_t)wout * win;
        float *t = cur; cur = nxt; nxt = t;
    }
    return cur[0];
}

void orc_field_eval_model(const float *coords, int64_t b, const float *params,
                          const int64_t *level_off, const int64_t *level_res,
                          const int64_t *level_entries, const uint8_t *level_dense, int m,
                          int n_feat, const float *weights, const int *widths, int nl,
                          int relu_out, float *out) {
    int maxw = m * n_feat;
    for (int i = 0; i <= nl; ++i) if (widths[i] > maxw) maxw = widths[i];
    #pragma omp parallel
    {
        float h0[1024], h1[1024];
        (void)maxw;
        #pragma omp for schedule(static)
        for (int64_t i = 0; i < b; ++i)
            out[i] = orc_field_one(coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], params,
                               level_off, level_res, level_entries, level_dense, m, n_feat,
                               weights, widths, nl, relu_out, h0, h1);
    }
}

/* network.py:160-183 adam_step for one float32 group, with the scalars cast
 * to float32 on the host exactly as `dt(...)` does (network.py:172-181). */
void orc_adam_f32(float *p, float *g, float *m, float *v, int64_t n, float lr, float beta1,
                  float one_minus_beta1, float beta2, float one_minus_beta2, float c1, float c2,
                  float eps, float l2) {
    #pragma omp parallel for schedule(static)
    for (int64_t j = 0; j < n; ++j) {
        float geff = g[j] + l2 * p[j];
        float mj = m[j] * beta1;
        mj = mj + one_minus_beta1 * geff;
        float vj = v[j] * beta2;
        vj = vj + one_minus_beta2 * (geff * geff);
        float mhat = mj / c1;
        float vhat = vj / c2;
        p[j] = p[j] - (lr * mhat) / (sqrtf(vhat) + eps);
        m[j] = mj;
        v[j] = vj;
        g[j] = 0.0f;
    }
}

/* numpy.random.PCG64 (numpy 2.3.5, third-party dependency of the reference,
 * used by sampler.py:54-55 `rng.random((b,3), dtype=float32)`): 128-bit LCG
 * stepped before each output, XSL-RR output, each u64 split low half first
 * into the u32 stream, float32 = (u32 >> 8) * 2^-24. */
static const u128 PCG_MULT = (((u128)0x2360ED051FC65DA4ULL) << 64) | (u128)0x4385DF649FCCF645ULL;

static u128 pcg_advance(u128 state, u128 inc, u128 delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = PCG_MULT, cur_plus = inc;
    while (delta) {
        if (delta & 1) {
            acc_mult *= cur_mult;
            acc_plus = acc_plus * cur_mult + cur_plus;
        }
        cur_plus = (cur_mult + 1) * cur_plus;
        cur_mult *= cur_mult;
        delta >>= 1;
    }
    return acc_mult * state + acc_plus;
}

static inline uint64_t pcg_out(u128 s) {
    uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
    unsigned rot = (unsigned)(s >> 122);
    uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64 - rot) & 63));
}

/* Fill out[0..count) with float32 draws number u32_offset .. u32_offset+count
 * of the generator whose initial (state, inc) is given. */
void orc_pcg64_random_f32(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                          uint64_t u32_offset, int64_t count, float *out) {
    u128 s0 = ((u128)state_hi << 64) | state_lo;
    u128 inc = ((u128)inc_hi << 64) | inc_lo;
    const int64_t chunk = 1 << 16;
    int64_t nchunks = (count + chunk - 1) / chunk;
    #pragma omp parallel for schedule(static)
    for (int64_t ch = 0; ch < nchunks; ++ch) {
        int64_t j0 = ch * chunk, j1 = j0 + chunk < count ? j0 + chunk : count;
        uint64_t g = u32_offset + (uint64_t)j0;           /* global u32 index */
        u128 s = pcg_advance(s0, inc, (u128)(g >> 1));     /* state before the u64 holding g */
        uint64_t word = 0;
        int have = 0;
        for (int64_t j = j0; j < j1; ++j, ++g) {
            if (!have || (g & 1) == 0) {
                s = s * PCG_MULT + inc;
                word = pcg_out(s);
                have = 1;
            }
            uint32_t u = (g & 1) ? (uint32_t)(word >> 32) : (uint32_t)word;
            out[j] = (float)(u >> 8) * (1.0f / 16777216.0f);
        }
    }
}

/* volume.py:148-164 _gather_corners (cell-centred, border-clamped trilinear,
 * float32 throughout) + sampler.py:73-74 clip to [0,1] when clip != 0.
 * norm is (dz, dy, dx) x-fastest. */
void orc_trilinear(const float *norm, int64_t dx, int64_t dy, int64_t dz, const float *pts,
                   int64_t n, int clip, float *out) {
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        float sx = pts[3 * i + 0] * (float)dx - 0.5f;
        float sy = pts[3 * i + 1] * (float)dy - 0.5f;
        float sz = pts[3 * i + 2] * (float)dz - 0.5f;
        int64_t x0 = (int64_t)floorf(sx), y0 = (int64_t)floorf(sy), z0 = (int64_t)floorf(sz);
        float fx = sx - (float)x0, fy = sy - (float)y0, fz = sz - (float)z0;
        float acc = 0.0f;
        for (int c = 0; c < 8; ++c) {
            int ox = c & 1, oy = (c >> 1) & 1, oz = (c >> 2) & 1;
            int64_t ix = clampi(x0 + ox, 0, dx - 1), iy = clampi(y0 + oy, 0, dy - 1),
                    iz = clampi(z0 + oz, 0, dz - 1);
            float w = 1.0f;
            w = w * (ox ? fx : 1.0f - fx);
            w = w * (oy ? fy : 1.0f - fy);
            w = w * (oz ? fz : 1.0f - fz);
            acc += w * norm[(iz * dy + iy) * dx + ix];
        }
        if (clip) acc = acc < 0.0f ? 0.0f : (acc > 1.0f ? 1.0f : acc);
        out[i] = acc;
    }
}
