// ctk_metrics.cu -- device-side per-iteration reconstruction metrics (SURVEY
// row f1): RRE and SSIM of x_k against x_true, so solves that report them
// (ctkrylov/gmres.py:254-257 -> metrics.py:13-62) need no host round trip.
//
// RRE  = ||x - x_true|| / ||x_true||                       (metrics.py:13-22)
// SSIM = mean over "valid" 8x8 windows of the SSIM map with a Gaussian window
//        (sigma 1.5, normalised), C1 = (0.01 L)^2, C2 = (0.03 L)^2, L the
//        dynamic range of x_true                            (metrics.py:25-62)
// The reference filters with fftconvolve; here each window is summed
// directly in fp64 (same quantity, rounding-level differences).  Reductions
// are deterministic (fixed-order partials, last-CTA pass with an integer
// ticket).
#include <math.h>

#include "ctk_common.cuh"

namespace ctk {

constexpr int MT = 256;

__device__ __forceinline__ double mwarp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// CTA sum of v -> partial[blockIdx.x]; the last CTA sums the partials in
// index order into *out.
__device__ void cta_reduce_to(double v, double* partial, unsigned* ticket, double* out) {
    __shared__ double red[MT / 32];
    __shared__ unsigned s_last;
    v = mwarp_sum(v);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < MT / 32; ++w) t += red[w];
        partial[blockIdx.x] = t;
        __threadfence();
        s_last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    if (threadIdx.x < 32) {
        double t = 0.0;
        for (unsigned b = threadIdx.x; b < gridDim.x; b += 32) t += __ldcg(partial + b);
        t = mwarp_sum(t);
        if (threadIdx.x == 0) {
            *out = t;
            *ticket = 0u;
        }
    }
}

__global__ void __launch_bounds__(MT) k_diff_norm2(const float* __restrict__ a,
                                                   const float* __restrict__ b, int64_t n,
                                                   double* partial, unsigned* ticket, double* out) {
    double s = 0.0;
    for (int64_t i = blockIdx.x * (int64_t)MT + threadIdx.x; i < n; i += (int64_t)gridDim.x * MT) {
        const double d = (double)a[i] - (double)b[i];
        s = fma(d, d, s);
    }
    cta_reduce_to(s, partial, ticket, out);
}

// Sum of the SSIM map over valid windows (top-left corner (i, j), i < ny-7,
// j < nx-7); the host divides by the window count.
__global__ void __launch_bounds__(MT) k_ssim_sum(const float* __restrict__ x,
                                                 const float* __restrict__ t, int nx, int ny,
                                                 double c1, double c2, double* partial,
                                                 unsigned* ticket, double* out) {
    __shared__ double w8[8];
    if (threadIdx.x < 8) {            // normalised 1-D Gaussian, sigma 1.5 (outer product = window)
        double tot = 0.0, gi = 0.0;
        for (int q = 0; q < 8; ++q) {
            const double r = q - 3.5;
            const double e = exp(-(r * r) / (2.0 * 1.5 * 1.5));
            tot += e;
            if (q == (int)threadIdx.x) gi = e;
        }
        w8[threadIdx.x] = gi / tot;
    }
    __syncthreads();
    const int ox = nx - 7, oy = ny - 7;
    const int64_t nout = (int64_t)ox * oy;
    double s = 0.0;
    for (int64_t o = blockIdx.x * (int64_t)MT + threadIdx.x; o < nout;
         o += (int64_t)gridDim.x * MT) {
        const int i = (int)(o / ox), j = (int)(o % ox);
        double ma = 0, mb = 0, maa = 0, mbb = 0, mab = 0;
        for (int u = 0; u < 8; ++u) {
            const float* ra = x + (size_t)(i + u) * nx + j;
            const float* rb = t + (size_t)(i + u) * nx + j;
            double la = 0, lb = 0, laa = 0, lbb = 0, lab = 0;
#pragma unroll
            for (int v = 0; v < 8; ++v) {
                const double av = (double)__ldg(ra + v), bv = (double)__ldg(rb + v);
                const double wv = w8[v];
                la = fma(wv, av, la);
                lb = fma(wv, bv, lb);
                laa = fma(wv, av * av, laa);
                lbb = fma(wv, bv * bv, lbb);
                lab = fma(wv, av * bv, lab);
            }
            const double wu = w8[u];
            ma = fma(wu, la, ma);
            mb = fma(wu, lb, mb);
            maa = fma(wu, laa, maa);
            mbb = fma(wu, lbb, mbb);
            mab = fma(wu, lab, mab);
        }
        const double va = maa - ma * ma, vb = mbb - mb * mb, cv = mab - ma * mb;
        s += ((2.0 * ma * mb + c1) * (2.0 * cv + c2)) / ((ma * ma + mb * mb + c1) * (va + vb + c2));
    }
    cta_reduce_to(s, partial, ticket, out);
}

}  // namespace ctk

using namespace ctk;

extern "C" size_t ctk_metrics_scratch_bytes(void) { return 256 + 8 * 2048; }

extern "C" int ctk_metrics(const float* x, const float* x_true, int nx, int ny, double dyn_range,
                           double* out, void* scratch, void* stream) {
    if (!x || !x_true || !out || !scratch || nx <= 0 || ny <= 0)
        return ctk_fail(CTK_ERR_ARG, "bad metrics arguments");
    cudaStream_t st = ctk_stream(stream);
    unsigned* ticket = reinterpret_cast<unsigned*>(scratch);
    double* partial = reinterpret_cast<double*>((char*)scratch + 256);
    const int64_t n = (int64_t)nx * ny;
    int G = (int)((n + MT - 1) / MT);
    if (G > 2 * 148) G = 2 * 148;
    k_diff_norm2<<<G, MT, 0, st>>>(x, x_true, n, partial, ticket, out);
    CTK_LAUNCH_CHECK("k_diff_norm2");
    if (nx >= 8 && ny >= 8 && dyn_range > 0) {
        const int64_t nout = (int64_t)(nx - 7) * (ny - 7);
        int G2 = (int)((nout + MT - 1) / MT);
        if (G2 > 4 * 148) G2 = 4 * 148;
        const double c1 = (0.01 * dyn_range) * (0.01 * dyn_range);
        const double c2 = (0.03 * dyn_range) * (0.03 * dyn_range);
        k_ssim_sum<<<G2, MT, 0, st>>>(x, x_true, nx, ny, c1, c2, partial + 1024, ticket + 1,
                                      out + 1);
        CTK_LAUNCH_CHECK("k_ssim_sum");
    }
    return CTK_OK;
}
