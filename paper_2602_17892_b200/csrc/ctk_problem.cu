// ctk_problem.cu -- on-device problem generation.
//
// * ctk_phantom: ellipse phantoms sampled at pixel centres -- the reference's
//   modified Shepp-Logan (ctkrylov/ct.py:115-134) and the harness's seeded
//   random-ellipse recipe (paper_2602_17892_b200/problems.py).  One thread per
//   pixel, every ellipse in the reference's order, the reference's fp64
//   expression sequence with explicit round-to-nearest intrinsics (no FMA
//   contraction), so the image is bitwise numpy's.  At c5 (64 slices of
//   2048^2) this replaces ~1 s of numpy per slice with a few microseconds.
// * ctk_add_noise: add_noise (ctkrylov/ct.py:267-283) on a device sinogram:
//   noise_norm = level * ||b_clean||, b = b_clean + (noise_norm * g) / ||g||.
//   The Gaussian draw g is numpy's default_rng(seed).standard_normal(m),
//   made on the host (the PCG64/ziggurat stream is what fixes the data) and
//   copied in; both norms are fp64 fixed-order reductions.
#include "ctk_common.cuh"

namespace ctk {

constexpr int PH_MAX_ELL = 128;

struct PhantomArgs {
    int nx, ny, n_ell;
    double xmin, ymax, h, scale;
    // per ellipse: value, a, b, x0, y0, cos(phi), sin(phi)  (host numpy trig)
    double e[PH_MAX_ELL][7];
};

__global__ void __launch_bounds__(256) k_phantom(const __grid_constant__ PhantomArgs P,
                                                 double* __restrict__ img64,
                                                 float* __restrict__ img32) {
    const int ix = blockIdx.x * 32 + (threadIdx.x & 31);
    const int iy = blockIdx.y * 8 + (threadIdx.x >> 5);
    if (ix >= P.nx || iy >= P.ny) return;
    // pixel centres, ImageGrid.pixel_centers (ct.py:60-66):
    //   xc = xmin + (ix + 0.5) * h,  yc = ymax - (iy + 0.5) * h;  then / scale
    const double X = __ddiv_rn(__dadd_rn(P.xmin, __dmul_rn((double)ix + 0.5, P.h)), P.scale);
    const double Y = __ddiv_rn(__dsub_rn(P.ymax, __dmul_rn((double)iy + 0.5, P.h)), P.scale);
    double acc = 0.0;
    for (int k = 0; k < P.n_ell; ++k) {
        const double* e = P.e[k];
        const double dx = __dsub_rn(X, e[3]), dy = __dsub_rn(Y, e[4]);
        // u = ((X - x0) c + (Y - y0) s) / a ;  v = (-(X - x0) s + (Y - y0) c) / b
        const double u = __ddiv_rn(__dadd_rn(__dmul_rn(dx, e[5]), __dmul_rn(dy, e[6])), e[1]);
        const double v = __ddiv_rn(__dadd_rn(__dmul_rn(-dx, e[6]), __dmul_rn(dy, e[5])), e[2]);
        if (__dadd_rn(__dmul_rn(u, u), __dmul_rn(v, v)) <= 1.0) acc = __dadd_rn(acc, e[0]);
    }
    const size_t o = (size_t)iy * P.nx + ix;
    if (img64) img64[o] = acc;
    if (img32) img32[o] = __double2float_rn(acc);
}

constexpr int NOISE_BLOCKS = 296;   // 2 per SM
constexpr int NOISE_THREADS = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// clean data in fp32 (a device A x) or fp64 (a host array copied in)
__device__ __forceinline__ double clean_at(const float* b32, const double* b64, int64_t i) {
    return b64 ? b64[i] : (double)b32[i];
}

// Block partials of ||b_clean||^2 and ||g||^2 (fixed per-thread strides and
// a fixed tree: deterministic for a given m).

__global__ void __launch_bounds__(NOISE_THREADS) k_noise_norms(const float* __restrict__ b,
                                                               const double* __restrict__ bd,
                                                               const double* __restrict__ g,
                                                               int64_t m, double* part) {
    double sb = 0.0, sg = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)NOISE_THREADS + threadIdx.x; i < m;
         i += (int64_t)NOISE_BLOCKS * NOISE_THREADS) {
        const double bv = clean_at(b, bd, i), gv = g[i];
        sb = fma(bv, bv, sb);
        sg = fma(gv, gv, sg);
    }
    __shared__ double s[2][NOISE_THREADS / 32];
    sb = warp_sum(sb);
    sg = warp_sum(sg);
    if ((threadIdx.x & 31) == 0) {
        s[0][threadIdx.x >> 5] = sb;
        s[1][threadIdx.x >> 5] = sg;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tb = 0.0, tg = 0.0;
        for (int w = 0; w < NOISE_THREADS / 32; ++w) {
            tb += s[0][w];
            tg += s[1][w];
        }
        part[2 * blockIdx.x] = tb;
        part[2 * blockIdx.x + 1] = tg;
    }
}

// Every block reduces the NOISE_BLOCKS partials in the same order (bitwise
// identical norms everywhere), then b = b_clean + (noise_norm * g) / ||g||.
__global__ void __launch_bounds__(NOISE_THREADS) k_noise_apply(const float* __restrict__ b,
                                                               const double* __restrict__ bd,
                                                               const double* __restrict__ g,
                                                               int64_t m, double level,
                                                               const double* part,
                                                               double* __restrict__ b64,
                                                               float* __restrict__ b32,
                                                               double* noise_norm_out) {
    __shared__ double s_nn, s_ng;
    if (threadIdx.x == 0) {
        double tb = 0.0, tg = 0.0;
        for (int k = 0; k < NOISE_BLOCKS; ++k) {
            tb += part[2 * k];
            tg += part[2 * k + 1];
        }
        s_nn = level * sqrt(tb);
        s_ng = sqrt(tg);
        if (blockIdx.x == 0 && noise_norm_out) noise_norm_out[0] = s_nn;
    }
    __syncthreads();
    const double nn = s_nn, ng = s_ng;
    for (int64_t i = blockIdx.x * (int64_t)NOISE_THREADS + threadIdx.x; i < m;
         i += (int64_t)gridDim.x * NOISE_THREADS) {
        const double v = __dadd_rn(clean_at(b, bd, i), __ddiv_rn(__dmul_rn(nn, g[i]), ng));
        if (b64) b64[i] = v;
        if (b32) b32[i] = __double2float_rn(v);
    }
}

}  // namespace ctk

using namespace ctk;

extern "C" int ctk_phantom(int nx, int ny, double xmin, double ymax, double pixel_size,
                           double scale, const double* ellipses, int n_ellipses, double* img64,
                           float* img32, void* stream) {
    if (nx <= 0 || ny <= 0 || !(pixel_size > 0.0) || !(scale != 0.0))
        return ctk_fail(CTK_ERR_GEOMETRY, "phantom: invalid grid %dx%d, h=%g, scale=%g", nx, ny,
                        pixel_size, scale);
    if (n_ellipses < 0 || n_ellipses > PH_MAX_ELL || (n_ellipses > 0 && !ellipses))
        return ctk_fail(CTK_ERR_ARG, "phantom: %d ellipses (at most %d)", n_ellipses, PH_MAX_ELL);
    if (!img64 && !img32) return ctk_fail(CTK_ERR_ARG, "phantom: no output");
    PhantomArgs P;
    P.nx = nx;
    P.ny = ny;
    P.n_ell = n_ellipses;
    P.xmin = xmin;
    P.ymax = ymax;
    P.h = pixel_size;
    P.scale = scale;
    for (int k = 0; k < n_ellipses; ++k)
        for (int c = 0; c < 7; ++c) P.e[k][c] = ellipses[7 * k + c];
    dim3 grid((nx + 31) / 32, (ny + 7) / 8);
    k_phantom<<<grid, 256, 0, ctk_stream(stream)>>>(P, img64, img32);
    CTK_LAUNCH_CHECK("k_phantom");
    return CTK_OK;
}

extern "C" size_t ctk_noise_scratch_bytes(void) { return sizeof(double) * 2 * NOISE_BLOCKS; }

extern "C" int ctk_add_noise(const float* b_clean, const double* b_clean64, const double* g,
                             int64_t m, double level, double* b64, float* b32,
                             double* noise_norm_dev, void* scratch, void* stream) {
    if (!(level >= 0.0)) return ctk_fail(CTK_ERR_ARG, "noise level must be nonnegative, got %g", level);
    if (m <= 0 || (!b_clean == !b_clean64) || !g || !scratch)
        return ctk_fail(CTK_ERR_ARG, "add_noise: need exactly one of b_clean / b_clean64, g, scratch");
    if (!b64 && !b32) return ctk_fail(CTK_ERR_ARG, "add_noise: no output");
    cudaStream_t st = ctk_stream(stream);
    double* part = static_cast<double*>(scratch);
    k_noise_norms<<<NOISE_BLOCKS, NOISE_THREADS, 0, st>>>(b_clean, b_clean64, g, m, part);
    CTK_LAUNCH_CHECK("k_noise_norms");
    k_noise_apply<<<NOISE_BLOCKS, NOISE_THREADS, 0, st>>>(b_clean, b_clean64, g, m, level, part,
                                                          b64, b32, noise_norm_dev);
    CTK_LAUNCH_CHECK("k_noise_apply");
    return CTK_OK;
}
