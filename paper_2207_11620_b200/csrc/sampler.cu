// Training-sample generation, analytic field rasterisation and metrics.
//
// Reference: sampler.py:54-74 (sample_incore: numpy PCG64 float32 coords +
// volume.py:148-164 trilinear GT, clamped), fields.py:15-88 (rasterize),
// volume.py:197-207 (mse / psnr).
#include "common.cuh"

namespace nvol {

// PCG64 jump table: entry i advances the LCG by 2^i steps (state -> mult[i] *
// state + plus[i]).  Built on the host once per stream increment and passed
// by value, so every thread jumps straight to its own draws with popcount(
// delta) 128-bit multiply-adds (no serial per-block jump, no per-step state).
struct PcgJump {
    U128 mult[64], plus[64];
};

static PcgJump make_jump(U128 inc) {
    typedef unsigned __int128 u128;
    u128 cm = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
    u128 cp = ((u128)inc.hi << 64) | (u128)inc.lo;
    PcgJump j;
    for (int i = 0; i < 64; ++i) {
        j.mult[i] = U128{(uint64_t)(cm >> 64), (uint64_t)cm};
        j.plus[i] = U128{(uint64_t)(cp >> 64), (uint64_t)cp};
        cp = (cm + 1) * cp;
        cm = cm * cm;
    }
    return j;
}

// macrocell.py:101-133 macrocell_update_online for one sample: widen the
// value range of every cell whose bordered scan window contains the sample's
// trilinear stencil (the containing cell, plus a neighbour where the stencil
// straddles a cell boundary).  Stencil arithmetic is the float32 lookup path
// (s = p*D - 0.5, two roundings).  Targets are in [0, 1], so IEEE order equals
// signed-int order of the bit patterns (lo starts at +inf, hi at -inf): int
// atomicMin / atomicMax are exact and order-independent (bit-exact with the
// reference's np.minimum.at / np.maximum.at).
struct McGrid {
    float *lo, *hi;
    int64_t gx, gy, gz, n_g;
};

__device__ __forceinline__ void mc_widen(const McGrid &g, int64_t dx, int64_t dy, int64_t dz, float px, float py,
                                         float pz, float t) {
    const float ps[3] = {px, py, pz};
    const int64_t dims[3] = {dx, dy, dz}, gd[3] = {g.gx, g.gy, g.gz};
    int64_t clo[3], chi[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float sa = xsub(xmul(ps[a], (float)dims[a]), 0.5f);
        const int64_t i0 = (int64_t)floorf(sa);
        const int64_t vmax = dims[a] - 1;
        const int64_t vlo = min(max(i0, (int64_t)0), vmax);
        const int64_t vhi = min(max(i0 + (sa > (float)i0 ? 1 : 0), (int64_t)0), vmax);
        const int64_t bound = gd[a] - 1;
        // floor division of non-negative values
        clo[a] = min(max((vhi + g.n_g - 1) / g.n_g - 1, (int64_t)0), bound);
        chi[a] = min(max((vlo + 1) / g.n_g, (int64_t)0), bound);
    }
    const int ti = __float_as_int(t);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const int64_t ix = (k & 1) ? chi[0] : clo[0], iy = (k & 2) ? chi[1] : clo[1], iz = (k & 4) ? chi[2] : clo[2];
        const int64_t c = (iz * g.gy + iy) * g.gx + ix;
        atomicMin(reinterpret_cast<int *>(g.lo) + c, ti);
        atomicMax(reinterpret_cast<int *>(g.hi) + c, ti);
    }
}

__global__ void mc_update_kernel(const float *__restrict__ coords, const float *__restrict__ targets, int64_t n,
                                 int64_t dx, int64_t dy, int64_t dz, const McGrid g) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) mc_widen(g, dx, dy, dz, coords[3 * i], coords[3 * i + 1], coords[3 * i + 2], targets[i]);
}

// One thread per row: the row's three u32 draws are u32 indices g0..g0+2 of
// the stream (sample i, axis a -> 3i+a); they live in u64 outputs g0>>1 and
// (g0+2)>>1.  The GT read is the bit-exact trilinear of volume.py:148-164,
// clamped to [0,1] as sampler.py:74.
__global__ void __launch_bounds__(256) sample_incore_kernel(U128 s0, U128 inc, const PcgJump jump, uint64_t u32_base,
                                                            const int64_t *__restrict__ step_counter,
                                                            int64_t counter0, int64_t b_global, int64_t row0,
                                                            int64_t b,
                                                            const float *__restrict__ vol, int64_t dx,
                                                            int64_t dy, int64_t dz, float *__restrict__ coords,
                                                            float *__restrict__ targets, const McGrid mc) {
    __shared__ U128 sm_mult[64], sm_plus[64];
    if (threadIdx.x < 64) {
        sm_mult[threadIdx.x] = jump.mult[threadIdx.x];
        sm_plus[threadIdx.x] = jump.plus[threadIdx.x];
    }
    __syncthreads();
    const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= b) return;
    uint64_t base = u32_base;
    if (step_counter)
        base += (uint64_t)(*step_counter - counter0) * 3ull * (uint64_t)b_global + 3ull * (uint64_t)row0;
    const uint64_t g0 = base + 3ull * (uint64_t)r;
    // state after (g0 >> 1) steps
    U128 st = s0;
    for (uint64_t d = g0 >> 1; d; d &= d - 1) {
        const int i = __ffsll((long long)d) - 1;
        st = u128_add(u128_mul(sm_mult[i], st), sm_plus[i]);
    }
    const U128 m = pcg_mult();
    st = u128_add(u128_mul(st, m), inc);
    const uint64_t w0 = pcg_output(st);
    st = u128_add(u128_mul(st, m), inc);
    const uint64_t w1 = pcg_output(st);
    uint32_t u[3];
    if ((g0 & 1) == 0) {
        u[0] = (uint32_t)w0;
        u[1] = (uint32_t)(w0 >> 32);
        u[2] = (uint32_t)w1;
    } else {
        u[0] = (uint32_t)(w0 >> 32);
        u[1] = (uint32_t)w1;
        u[2] = (uint32_t)(w1 >> 32);
    }
    const float x = u32_to_f32(u[0]), y = u32_to_f32(u[1]), z = u32_to_f32(u[2]);
    coords[3 * r] = x;
    coords[3 * r + 1] = y;
    coords[3 * r + 2] = z;
    const float t = fminf(fmaxf(trilinear_at<true>(vol, dx, dy, dz, x, y, z), 0.0f), 1.0f);
    targets[r] = t;
    if (mc.lo) mc_widen(mc, dx, dy, dz, x, y, z, t);  // online macro-cells fused into the sampler
}

static const PcgJump &jump_for(U128 inc) {
    static PcgJump cached;
    static U128 cached_inc{0, 0};
    static bool have = false;
    if (!have || cached_inc.hi != inc.hi || cached_inc.lo != inc.lo) {
        cached = make_jump(inc);
        cached_inc = inc;
        have = true;
    }
    return cached;
}

// sampler.py:224-253 BlockBuffer.sample on the device: the batch's slot /
// voxel / jitter draws come from the caller's numpy generator (so the stream is
// the reference's), the coordinate arithmetic and the payload-local trilinear
// (or nearest) gather run here, float32 in the reference's operation order.
// Payloads [R][pz][py][px] carry a one-voxel ghost border (index 0 = origin-1).
__global__ void sample_outofcore_kernel(const int32_t *__restrict__ slots, const float *__restrict__ u,
                                        const float *__restrict__ jit, int64_t b, const int64_t *__restrict__ origins,
                                        const int64_t *__restrict__ interiors, const float *__restrict__ payloads,
                                        int64_t px, int64_t py, int64_t pz, int64_t dx, int64_t dy, int64_t dz,
                                        int nearest, float *__restrict__ coords, float *__restrict__ targets) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= b) return;
    const int64_t sl = slots[i];
    const float *pl = payloads + sl * pz * py * px;
    const int64_t dims[3] = {dx, dy, dz};
    const float one_below_1 = __int_as_float(0x3f7fffff);
    int64_t vox[3], org[3];
    float c[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        org[a] = origins[3 * sl + a];
        const int64_t in = interiors[3 * sl + a];
        vox[a] = min((int64_t)xmul(u[3 * i + a], (float)in), in - 1);          // (u * interior).astype(int64)
        const float center = xadd(xadd((float)org[a], (float)vox[a]), 0.5f);   // origin + voxel + 0.5
        const float j = xsub(jit[3 * i + a], 0.5f);                             // rng.random - 0.5
        c[a] = fminf(fmaxf(xdiv(xadd(center, j), (float)dims[a]), 0.0f), one_below_1);
        coords[3 * i + a] = c[a];
    }
    float t;
    if (nearest) {
        t = pl[((vox[2] + 1) * py + (vox[1] + 1)) * px + (vox[0] + 1)];
    } else {
        int64_t i0[3];
        float fr[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float sa = xsub(xmul(c[a], (float)dims[a]), 0.5f);
            i0[a] = (int64_t)floorf(sa);
            fr[a] = xsub(sa, (float)i0[a]);
        }
        t = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            int64_t l[3];
            float w = 1.0f;
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const int off = (k >> a) & 1;
                const int64_t g = min(max(i0[a] + off, (int64_t)0), dims[a] - 1);
                l[a] = g - (org[a] - 1);
                w = xmul(w, off ? fr[a] : xsub(1.0f, fr[a]));
            }
            t = xadd(t, xmul(w, pl[(l[2] * py + l[1]) * px + l[0]]));
        }
    }
    targets[i] = fminf(fmaxf(t, 0.0f), 1.0f);
}

__global__ void trilinear_kernel(const float *__restrict__ vol, int64_t dx, int64_t dy, int64_t dz,
                                 const float *__restrict__ pts, int64_t n, float *__restrict__ out) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = trilinear_at(vol, dx, dy, dz, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
}

// fields.py:15-57 in float64 (device libm: <= 2 ulp from glibc, so the
// float32-cast result can differ from the host rasteriser by 1 ulp in rare
// voxels; tests that need bit-identical inputs upload the host volume).
__device__ __forceinline__ double gauss3(double x, double y, double z, double cx, double cy, double cz,
                                         double sigma) {
    double ax = x - cx, ay = y - cy, az = z - cz;
    double d2 = ax * ax + ay * ay + az * az;
    return exp(-d2 / (2.0 * sigma * sigma));
}

__device__ double field_value(int field, double x, double y, double z) {
    const double pi = 3.141592653589793;
    switch (field) {
        case 0: return gauss3(x, y, z, 0.5, 0.5, 0.5, 0.18);
        case 1: {
            double a = gauss3(x, y, z, 0.30, 0.32, 0.28, 0.09);
            double b = gauss3(x, y, z, 0.68, 0.60, 0.55, 0.07);
            double c = gauss3(x, y, z, 0.45, 0.75, 0.72, 0.06);
            return fmax(fmax(a, b), c);
        }
        case 2: {
            double tp = 2.0 * pi;
            double v = sin(tp * 3 * x) * sin(tp * 2 * y) * sin(tp * 4 * z);
            return 0.5 + 0.5 * v;
        }
        default: {
            const double fm = 6.0, alpha = 0.25;
            double qx = 2.0 * x - 1.0, qy = 2.0 * y - 1.0, qz = 2.0 * z - 1.0;
            double r = sqrt(qx * qx + qy * qy);
            double rho = cos(2.0 * pi * fm * 0.5 * cos(pi * r / 2.0));
            double v = (1.0 - sin(pi * qz / 2.0) + alpha * (1.0 + rho)) / (2.0 * (1.0 + alpha));
            return fmin(fmax(v, 0.0), 1.0);
        }
    }
}

__global__ void rasterize_kernel(int field, int64_t dx, int64_t dy, int64_t dz, int64_t z0, int64_t nz,
                                 void *__restrict__ out, int out_u8) {
    int64_t n = dx * dy * nz;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        int64_t ix = k % dx, iy = (k / dx) % dy, iz = z0 + k / (dx * dy);
        double x = ((double)ix + 0.5) / (double)dx;
        double y = ((double)iy + 0.5) / (double)dy;
        double z = ((double)iz + 0.5) / (double)dz;
        double v = fmin(fmax(field_value(field, x, y, z), 0.0), 1.0);
        if (out_u8)
            reinterpret_cast<uint8_t *>(out)[k] = (uint8_t)rint(v * 255.0);
        else
            reinterpret_cast<float *>(out)[k] = (float)v;
    }
}

__global__ void sq_err_kernel(const float *__restrict__ a, const float *__restrict__ b, int64_t n,
                              double *__restrict__ sum) {
    __shared__ double red[32];
    double s = 0.0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        double d = (double)a[i] - (double)b[i];
        s += d * d;
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x < 32) {
        s = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (threadIdx.x == 0) atomicAdd(sum, s);
    }
}

}  // namespace nvol

using namespace nvol;

extern "C" {

int nvol_sample_incore(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                       uint64_t u32_offset, int64_t b, const float *volume, int64_t dx, int64_t dy, int64_t dz,
                       float *coords, float *targets, void *stream) {
    NVOL_REQUIRE(b >= 1, "batch size must be >= 1");
    NVOL_REQUIRE(volume && coords && targets, "null pointer");
    NVOL_REQUIRE(dx >= 1 && dy >= 1 && dz >= 1, "bad volume dims");
    const U128 inc{inc_hi, inc_lo};
    sample_incore_kernel<<<grid_for(b, 256), 256, 0, as_stream(stream)>>>(
        U128{state_hi, state_lo}, inc, jump_for(inc), u32_offset, nullptr, 0, 0, 0, b, volume, dx, dy, dz,
        coords, targets, McGrid{nullptr, nullptr, 0, 0, 0, 1});
    return check_launch("sample_incore");
}

int nvol_sample_incore_dev_mc(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                              uint64_t u32_base, const int64_t *step_counter, int64_t counter0, int64_t b_global,
                              int64_t row0, int64_t b, const float *volume, int64_t dx, int64_t dy, int64_t dz,
                              float *coords, float *targets, float *mc_lo, float *mc_hi, int64_t gx, int64_t gy,
                              int64_t gz, int64_t n_g, void *stream) {
    NVOL_REQUIRE(b >= 1 && step_counter, "bad arguments");
    NVOL_REQUIRE(volume && coords && targets, "null pointer");
    NVOL_REQUIRE(!mc_lo || (mc_hi && n_g >= 1 && gx >= 1 && gy >= 1 && gz >= 1), "bad macro-cell grid");
    const U128 inc{inc_hi, inc_lo};
    sample_incore_kernel<<<grid_for(b, 256), 256, 0, as_stream(stream)>>>(
        U128{state_hi, state_lo}, inc, jump_for(inc), u32_base, step_counter, counter0, b_global, row0, b, volume,
        dx, dy, dz, coords, targets, McGrid{mc_lo, mc_hi, gx, gy, gz, n_g});
    return check_launch("sample_incore_dev");
}

int nvol_sample_incore_dev(uint64_t state_hi, uint64_t state_lo, uint64_t inc_hi, uint64_t inc_lo,
                           uint64_t u32_base, const int64_t *step_counter, int64_t counter0, int64_t b_global,
                           int64_t row0, int64_t b,
                           const float *volume, int64_t dx, int64_t dy, int64_t dz, float *coords, float *targets,
                           void *stream) {
    return nvol_sample_incore_dev_mc(state_hi, state_lo, inc_hi, inc_lo, u32_base, step_counter, counter0, b_global,
                                     row0, b, volume, dx, dy, dz, coords, targets, nullptr, nullptr, 0, 0, 0, 1,
                                     stream);
}

int nvol_macrocell_update_online(const float *coords, const float *targets, int64_t n, int64_t dx, int64_t dy,
                                 int64_t dz, float *lo, float *hi, int64_t gx, int64_t gy, int64_t gz, int64_t n_g,
                                 void *stream) {
    if (n == 0) return NVOL_OK;
    NVOL_REQUIRE(coords && targets && lo && hi, "null pointer");
    NVOL_REQUIRE(n_g >= 1 && gx >= 1 && gy >= 1 && gz >= 1 && dx >= 1 && dy >= 1 && dz >= 1, "bad grid");
    mc_update_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(coords, targets, n, dx, dy, dz,
                                                                      McGrid{lo, hi, gx, gy, gz, n_g});
    return check_launch("macrocell_update_online");
}

int nvol_sample_outofcore(const int32_t *slots, const float *u, const float *jitter, int64_t b,
                          const int64_t *origins, const int64_t *interiors, const float *payloads, int64_t px,
                          int64_t py, int64_t pz, int64_t dx, int64_t dy, int64_t dz, int32_t nearest, float *coords,
                          float *targets, void *stream) {
    if (b == 0) return NVOL_OK;
    NVOL_REQUIRE(slots && u && jitter && origins && interiors && payloads && coords && targets, "null pointer");
    NVOL_REQUIRE(px >= 1 && py >= 1 && pz >= 1 && dx >= 1 && dy >= 1 && dz >= 1, "bad dims");
    sample_outofcore_kernel<<<grid_for(b, 256), 256, 0, as_stream(stream)>>>(
        slots, u, jitter, b, origins, interiors, payloads, px, py, pz, dx, dy, dz, nearest, coords, targets);
    return check_launch("sample_outofcore");
}

int nvol_trilinear(const float *volume, int64_t dx, int64_t dy, int64_t dz, const float *pts, int64_t n, float *out,
                   void *stream) {
    if (n == 0) return NVOL_OK;
    NVOL_REQUIRE(volume && pts && out, "null pointer");
    trilinear_kernel<<<grid_for(n, 256), 256, 0, as_stream(stream)>>>(volume, dx, dy, dz, pts, n, out);
    return check_launch("trilinear");
}

int nvol_rasterize(int32_t field, int64_t dx, int64_t dy, int64_t dz, int64_t z0, int64_t nz, void *out,
                   int32_t out_u8, void *stream) {
    NVOL_REQUIRE(field >= 0 && field <= 3, "unknown synthetic field");
    NVOL_REQUIRE(out && dx >= 1 && dy >= 1 && dz >= 1 && z0 >= 0 && nz >= 0 && z0 + nz <= dz, "bad arguments");
    if (nz == 0) return NVOL_OK;
    int64_t n = dx * dy * nz;
    unsigned grid = (unsigned)min((int64_t)148 * 16, (n + 255) / 256);
    rasterize_kernel<<<grid, 256, 0, as_stream(stream)>>>(field, dx, dy, dz, z0, nz, out, out_u8);
    return check_launch("rasterize");
}

int nvol_sq_err_sum(const float *a, const float *b, int64_t n, double *sum, void *stream) {
    NVOL_REQUIRE(a && b && sum, "null pointer");
    if (n == 0) return NVOL_OK;
    unsigned grid = (unsigned)min((int64_t)148 * 8, (n + 255) / 256);
    sq_err_kernel<<<grid, 256, 0, as_stream(stream)>>>(a, b, n, sum);
    return check_launch("sq_err_sum");
}

}  // extern "C"
