/*
 * ORACLE — test infrastructure only (see kernels.c header).  C restatement of
 * the reference's ray-march renderer (_render_kernels.py:52-488): slab test,
 * macro-cell DDA (float64), adaptive step, the ray-march state machine with
 * phase-preserving empty-space skipping, transfer-function lookup, opacity
 * correction, front-to-back compositing and the shadow phase, run per ray to
 * completion (rm_reference, _render_kernels.py:455-488; the wavefront driver
 * is bitwise identical to it per the reference's own tests).  Float32 /
 * float64 operation order is kept, so with the same field values the result
 * is bit-identical (powf is glibc's, as numba's).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

float orc_field_one(float x, float y, float z, const float *params, const int64_t *level_off,
                    const int64_t *level_res, const int64_t *level_entries, const uint8_t *level_dense,
                    int m, int n_feat, const float *weights, const int *widths, int nl, int relu_out,
                    float *h0, float *h1);

static inline int64_t clampi64(int64_t v, int64_t lo, int64_t hi) { return v < lo ? lo : (v > hi ? hi : v); }

/* _kernels.py:179-203 _grid_one */
static float grid_one(float x, float y, float z, const float *norm, int64_t dx, int64_t dy, int64_t dz) {
    float sx = x * (float)dx - 0.5f, sy = y * (float)dy - 0.5f, sz = z * (float)dz - 0.5f;
    int64_t x0 = (int64_t)floorf(sx), y0 = (int64_t)floorf(sy), z0 = (int64_t)floorf(sz);
    float fx = sx - (float)x0, fy = sy - (float)y0, fz = sz - (float)z0;
    float acc = 0.0f;
    for (int c = 0; c < 8; ++c) {
        int ox = c & 1, oy = (c >> 1) & 1, oz = (c >> 2) & 1;
        int64_t ix = clampi64(x0 + ox, 0, dx - 1), iy = clampi64(y0 + oy, 0, dy - 1), iz = clampi64(z0 + oz, 0, dz - 1);
        float w = ox ? fx : 1.0f - fx;
        w *= oy ? fy : 1.0f - fy;
        w *= oz ? fz : 1.0f - fz;
        acc += w * norm[(iz * dy + iy) * dx + ix];
    }
    return acc;
}

typedef struct {
    /* field */
    int use_grid;
    const float *norm;
    int64_t ndx, ndy, ndz;
    const float *params;
    const int64_t *loff, *lres, *lent;
    const uint8_t *ldense;
    int m, nfeat;
    const float *weights;
    const int *widths;
    int nl, relu_out;
    /* transfer function */
    const float *cv, *crgb, *ov, *oa;
    int ncv, nov;
    float ds;
    /* macro-cells */
    const float *mu;
    int64_t gx, gy, gz;
    double ng;
    int use_mc, skip_empty;
    /* march */
    float s1, s2, pexp, term, ka;
    int mode_shadow;
    float sdx, sdy, sdz, bgr, bgg, bgb;
    double hx, hy, hz;
} Scene;

/* _render_kernels.py:54-89 _isect */
static int isect(double ox, double oy, double oz, double dx, double dy, double dz, double hx, double hy,
                 double hz, double *t0o, double *t1o) {
    double t0 = -INFINITY, t1 = INFINITY;
    double o[3] = {ox, oy, oz}, d[3] = {dx, dy, dz}, h[3] = {hx, hy, hz};
    for (int a = 0; a < 3; ++a) {
        if (d[a] != 0.0) {
            double ta = (0.0 - o[a]) / d[a], tb = (h[a] - o[a]) / d[a];
            if (ta > tb) { double t = ta; ta = tb; tb = t; }
            t0 = t0 > ta ? t0 : ta;
            t1 = t1 < tb ? t1 : tb;
        } else if (o[a] < 0.0 || o[a] > h[a]) {
            return 0;
        }
    }
    t0 = t0 > 0.0 ? t0 : 0.0;
    if (t1 <= t0) return 0;
    *t0o = t0;
    *t1o = t1;
    return 1;
}

typedef struct {
    float T, r, g, b, clock, sbar, best_w, best_t, Tsh, o[3], d[3], muc;  /* RMF */
    double cell_exit, march_end, tm[3], td[3];                            /* RMD */
    int64_t pixel, phase, in_cell, c[3], st[3];                           /* RMI */
} Ray;

/* _render_kernels.py:244-253 */
static float adaptive(float muc, float s1, float s2, float pexp) {
    float mm = muc > 1.0f ? 1.0f : muc;
    float gap = 1.0f - mm;
    float s = s1 + (s2 - s1) * powf(gap, pexp);
    return s < s1 ? s1 : s;
}

static float mu_read(const Scene *S, int64_t cx, int64_t cy, int64_t cz) {
    int64_t ix = clampi64(cx, 0, S->gx - 1), iy = clampi64(cy, 0, S->gy - 1), iz = clampi64(cz, 0, S->gz - 1);
    return S->mu[(iz * S->gy + iy) * S->gx + ix];
}

/* _render_kernels.py:92-138 _dda_enter + 268-305 _rm_cell_entry */
static void cell_entry(const Scene *S, Ray *R) {
    double t1 = R->march_end;
    if (!S->use_mc) {
        R->cell_exit = t1;
        R->sbar = S->s1;
        R->muc = 1.0f;
        R->in_cell = 1;
        return;
    }
    double o[3] = {R->o[0], R->o[1], R->o[2]}, d[3] = {R->d[0], R->d[1], R->d[2]};
    double t0 = (double)R->clock, ng = S->ng;
    int64_t gdim[3] = {S->gx, S->gy, S->gz};
    for (int a = 0; a < 3; ++a) {
        double p = o[a] + t0 * d[a];
        int64_t c = clampi64((int64_t)floor(p / ng), 0, gdim[a] - 1);
        R->c[a] = c;
        if (d[a] > 0.0) {
            R->st[a] = 1;
            R->tm[a] = t0 + ((double)(c + 1) * ng - p) / d[a];
            R->td[a] = ng / d[a];
        } else if (d[a] < 0.0) {
            R->st[a] = -1;
            R->tm[a] = t0 + ((double)c * ng - p) / d[a];
            R->td[a] = -ng / d[a];
        } else {
            R->st[a] = 0;
            R->tm[a] = INFINITY;
            R->td[a] = INFINITY;
        }
    }
    double se = R->tm[0];
    if (R->tm[1] < se) se = R->tm[1];
    if (R->tm[2] < se) se = R->tm[2];
    if (se > t1) se = t1;
    R->cell_exit = se;
    R->muc = mu_read(S, R->c[0], R->c[1], R->c[2]);
    R->sbar = adaptive(R->muc, S->s1, S->s2, S->pexp);
    R->in_cell = 1;
}

/* _render_kernels.py:308-333 _rm_cell_advance */
static void cell_advance(const Scene *S, Ray *R) {
    double t1 = R->march_end;
    if (R->tm[0] <= R->tm[1] && R->tm[0] <= R->tm[2]) {
        R->c[0] += R->st[0];
        R->tm[0] = R->tm[0] + R->td[0];
    } else if (R->tm[1] <= R->tm[2]) {
        R->c[1] += R->st[1];
        R->tm[1] = R->tm[1] + R->td[1];
    } else {
        R->c[2] += R->st[2];
        R->tm[2] = R->tm[2] + R->td[2];
    }
    double se = R->tm[0];
    if (R->tm[1] < se) se = R->tm[1];
    if (R->tm[2] < se) se = R->tm[2];
    if (se > t1) se = t1;
    R->cell_exit = se;
    R->muc = mu_read(S, R->c[0], R->c[1], R->c[2]);
    R->sbar = adaptive(R->muc, S->s1, S->s2, S->pexp);
}

/* _render_kernels.py:336-361 _rm_next: returns ts or -1 */
static float rm_next(const Scene *S, Ray *R) {
    double t1 = R->march_end;
    if (R->in_cell == 0) cell_entry(S, R);
    for (;;) {
        float sbar = R->sbar;
        double se = R->cell_exit;
        if (S->use_mc && S->skip_empty && R->muc <= 0.0f) {
            float t = R->clock;
            while ((double)(t + 0.5f * sbar) < se) t = t + sbar;
            R->clock = t;
        } else {
            float ts = R->clock + 0.5f * sbar;
            if ((double)ts < se) {
                R->clock = R->clock + sbar;
                return ts;
            }
        }
        if (se >= t1) return -1.0f;
        cell_advance(S, R);
    }
}

/* _render_kernels.py:203-241 */
static float tf_alpha(const Scene *S, float v) {
    float x = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
    int n = S->nov;
    if (x <= S->ov[0]) return S->oa[0];
    if (x >= S->ov[n - 1]) return S->oa[n - 1];
    int i = 1;
    while (S->ov[i] < x) ++i;
    float w = (x - S->ov[i - 1]) / (S->ov[i] - S->ov[i - 1]);
    return S->oa[i - 1] + w * (S->oa[i] - S->oa[i - 1]);
}

static void tf_rgb(const Scene *S, float v, float *r, float *g, float *b) {
    float x = v < 0.0f ? 0.0f : (v > 1.0f ? 1.0f : v);
    int n = S->ncv;
    const float *c = S->crgb;
    if (x <= S->cv[0]) { *r = c[0]; *g = c[1]; *b = c[2]; return; }
    if (x >= S->cv[n - 1]) { *r = c[3 * (n - 1)]; *g = c[3 * (n - 1) + 1]; *b = c[3 * (n - 1) + 2]; return; }
    int i = 1;
    while (S->cv[i] < x) ++i;
    float w = (x - S->cv[i - 1]) / (S->cv[i] - S->cv[i - 1]);
    *r = c[3 * (i - 1)] + w * (c[3 * i] - c[3 * (i - 1)]);
    *g = c[3 * (i - 1) + 1] + w * (c[3 * i + 1] - c[3 * (i - 1) + 1]);
    *b = c[3 * (i - 1) + 2] + w * (c[3 * i + 2] - c[3 * (i - 1) + 2]);
}

/* _render_kernels.py:364-392 _rm_consume: 1 when the march just ended */
static int rm_consume(const Scene *S, Ray *R, float v, float ts, float sbar) {
    float a = tf_alpha(S, v) * S->ds;
    if (a < 0.0f) a = 0.0f;
    if (a > 1.0f) a = 1.0f;
    float abar = 1.0f - powf(1.0f - a, sbar / S->s1);
    if (R->phase == 0) {
        float T = R->T;
        float w = T * abar;
        if (S->mode_shadow && w > R->best_w) {
            R->best_w = w;
            R->best_t = ts;
        }
        float cr, cg, cb;
        tf_rgb(S, v, &cr, &cg, &cb);
        R->r += w * cr;
        R->g += w * cg;
        R->b += w * cb;
        T = T * (1.0f - abar);
        R->T = T;
        return T < S->term;
    }
    float Tsh = R->Tsh * (1.0f - abar);
    R->Tsh = Tsh;
    return Tsh < S->term;
}

/* _render_kernels.py:395-420 _rm_phase_end: 1 = ray done */
static int rm_phase_end(const Scene *S, Ray *R) {
    if (!S->mode_shadow || R->phase != 0) return 1;
    R->phase = 1;
    if (R->r == 0.0f && R->g == 0.0f && R->b == 0.0f) return 1;
    double bt = (double)R->best_t;
    double bx = (double)R->o[0] + bt * (double)R->d[0];
    double by = (double)R->o[1] + bt * (double)R->d[1];
    double bz = (double)R->o[2] + bt * (double)R->d[2];
    double t0s, t1s;
    if (!isect(bx, by, bz, (double)S->sdx, (double)S->sdy, (double)S->sdz, S->hx, S->hy, S->hz, &t0s, &t1s)) return 1;
    R->o[0] = (float)bx;
    R->o[1] = (float)by;
    R->o[2] = (float)bz;
    R->d[0] = S->sdx;
    R->d[1] = S->sdy;
    R->d[2] = S->sdz;
    R->clock = (float)t0s;
    R->march_end = t1s;
    R->in_cell = 0;
    return 0;
}

/* _render_kernels.py:423-432 _rm_final */
static void rm_final(const Scene *S, const Ray *R, float *img) {
    float scale = 1.0f;
    if (S->mode_shadow) scale = S->ka + (1.0f - S->ka) * R->Tsh;
    float T = R->T;
    int64_t p = R->pixel;
    img[3 * p] = R->r * scale + T * S->bgr;
    img[3 * p + 1] = R->g * scale + T * S->bgg;
    img[3 * p + 2] = R->b * scale + T * S->bgb;
}

/* _render_kernels.py:435-452 _coord_at */
static void coord_at(const Scene *S, const Ray *R, float ts, float *x, float *y, float *z) {
    const float one_below = 0.99999994f;
    float c[3];
    double h[3] = {S->hx, S->hy, S->hz};
    for (int a = 0; a < 3; ++a) {
        float v = (float)(((double)R->o[a] + (double)ts * (double)R->d[a]) / h[a]);
        if (v < 0.0f) v = 0.0f;
        if (v >= 1.0f) v = one_below;
        c[a] = v;
    }
    *x = c[0];
    *y = c[1];
    *z = c[2];
}

static float phi(const Scene *S, float x, float y, float z, float *h0, float *h1) {
    if (S->use_grid) return grid_one(x, y, z, S->norm, S->ndx, S->ndy, S->ndz);
    return orc_field_one(x, y, z, S->params, S->loff, S->lres, S->lent, S->ldense, S->m, S->nfeat, S->weights,
                         S->widths, S->nl, S->relu_out, h0, h1);
}

/* _render_kernels.py:455-488 rm_reference over rays [0, n); rays given as
 * origins/dirs (f32), t0/t1 (f64, from the batched slab test) and pixel ids.
 * Returns the number of field evaluations. */
int64_t orc_render_rm(const float *origins, const float *dirs, const double *t0, const double *t1,
                      const int64_t *pixels, int64_t n, int mode_shadow, int use_mc, int skip_empty, float s1,
                      float s2, float pexp, float term, float ka, const float *mu, int64_t gx, int64_t gy,
                      int64_t gz, double ng, float sdx, float sdy, float sdz, float bgr, float bgg, float bgb,
                      double hx, double hy, double hz, int use_grid, const float *norm, int64_t ndx, int64_t ndy,
                      int64_t ndz, const float *params, const int64_t *loff, const int64_t *lres,
                      const int64_t *lent, const uint8_t *ldense, int m, int nfeat, const float *weights,
                      const int *widths, int nl, int relu_out, const float *cv, const float *crgb, int ncv,
                      const float *ov, const float *oa, int nov, float ds, int64_t k_batch, float *img) {
    Scene S = {use_grid, norm, ndx, ndy, ndz, params, loff, lres, lent, ldense, m, nfeat, weights, widths, nl,
               relu_out, cv, crgb, ov, oa, ncv, nov, ds, mu, gx, gy, gz, ng, use_mc, skip_empty, s1, s2, pexp,
               term, ka, mode_shadow, sdx, sdy, sdz, bgr, bgg, bgb, hx, hy, hz};
    int64_t evals = 0;
    #pragma omp parallel for schedule(dynamic, 64) reduction(+ : evals)
    for (int64_t r = 0; r < n; ++r) {
        float h0[1024], h1[1024];
        Ray R;
        memset(&R, 0, sizeof(R));
        R.T = 1.0f;
        R.clock = (float)t0[r];
        R.Tsh = 1.0f;
        for (int a = 0; a < 3; ++a) {
            R.o[a] = origins[3 * r + a];
            R.d[a] = dirs[3 * r + a];
        }
        R.march_end = t1[r];
        R.pixel = pixels[r];
        int64_t in_batch = 0;  /* samples staged in the current wavefront batch */
        for (;;) {
            float ts = rm_next(&S, &R);
            if (ts < 0.0f) {
                in_batch = 0;
                if (rm_phase_end(&S, &R)) {
                    rm_final(&S, &R, img);
                    break;
                }
                continue;
            }
            float x, y, z;
            coord_at(&S, &R, ts, &x, &y, &z);
            float v = phi(&S, x, y, z, h0, h1);
            evals += 1;
            if (k_batch > 0 && ++in_batch == k_batch) in_batch = 0;
            if (rm_consume(&S, &R, v, ts, R.sbar)) {
                /* wavefront accounting (render.py:424-450): the rest of this
                 * K-batch was already staged and evaluated */
                if (k_batch > 0 && in_batch > 0) {
                    Ray C = R;
                    while (in_batch < k_batch && rm_next(&S, &C) >= 0.0f) {
                        ++in_batch;
                        ++evals;
                    }
                }
                in_batch = 0;
                if (rm_phase_end(&S, &R)) {
                    rm_final(&S, &R, img);
                    break;
                }
            }
        }
    }
    return evals;
}

int orc_render_version(void) { return 2; }
