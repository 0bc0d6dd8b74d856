// ctk_back.cu -- K2: the reference's unmatched pixel-driven backprojector B.
//
// Reference semantics (ctkrylov/ct.py:204-245), per pixel p and angle a:
//   g   = (X_p cos + Y_p sin) / s + (D-1)/2,   i0 = floor(g),   w = g - i0
//   out += h * ((1-w) * u[a, i0] [0<=i0<D] + w * u[a, idx1] [0<=i0+1<D])
// with idx1 = clip(clip(i0, 0, D-1) + 1, 0, D-1): the reference indexes the
// second tap from the CLIPPED first tap, so i0 == -1 reads u[a, 1] (u[a, 0]
// when D == 1).  That quirk is reproduced.
//
// B200 mapping: one CTA = a 32 x 16 pixel tile, 256 threads, 2 pixels per
// thread.  Angles are processed in chunks of 32: for each chunk the CTA
// stages, per angle, the short detector window its tile projects onto (zero
// filled outside [0, D), which is exactly the reference's masks) into shared
// memory with coalesced loads; the interpolation taps then come from smem.
// g is evaluated in fp64 (no hardware texture lerp: its 8-bit fraction would
// break the 1e-5 bar); taps and the lerp are fp32, each 32-angle partial sum
// is folded into an fp64 accumulator.  Small images split the angle range
// over blockIdx.z into partial images reduced in a fixed order (no atomics).
#include <math.h>

#include "ctk_common.cuh"

namespace ctk {

constexpr int BTX = 32, BTY = 16, BROWS = 8, BCA = 32;
constexpr int BTHREADS = BTX * BROWS;

struct BackArgs {
    const BackParams* bp;
    const float* u;       // row a at u + (a - a0) * D
    const float* x0;      // optional
    float* out;           // final image (S == 1) or partials [S][n]
    float* x;             // final image (S > 1)
    unsigned* cnt;        // S > 1: per-tile arrival tickets (zeroed once)
    int nx, ny, D, a0, a1, per_split, wmax, split;
    double h, xmin, ymax, center;
};

__global__ void __launch_bounds__(BTHREADS) k_back(BackArgs A) {
    extern __shared__ float win[];                 // [BCA][wmax]
    __shared__ double s_cg[BCA], s_sg[BCA];
    __shared__ int s_w0[BCA];

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BTX + tx;
    const int ix0 = blockIdx.x * BTX, iy0 = blockIdx.y * BTY;
    const int ix = ix0 + tx, iyA = iy0 + ty, iyB = iy0 + ty + BROWS;
    const double X = A.xmin + ((double)ix + 0.5) * A.h;
    const double YA = A.ymax - ((double)iyA + 0.5) * A.h;
    const double YB = A.ymax - ((double)iyB + 0.5) * A.h;
    // tile corner pixel centres
    const double Xlo = A.xmin + ((double)ix0 + 0.5) * A.h;
    const double Xhi = A.xmin + ((double)(ix0 + BTX - 1) + 0.5) * A.h;
    const double Yhi = A.ymax - ((double)iy0 + 0.5) * A.h;
    const double Ylo = A.ymax - ((double)(iy0 + BTY - 1) + 0.5) * A.h;

    const int aS = A.a0 + blockIdx.z * A.per_split;
    const int aE = min(A.a1, aS + A.per_split);
    const int D = A.D, wmax = A.wmax;
    const int q1 = D > 1 ? 1 : 0;                  // reference quirk tap for i0 == -1

    double accA = 0.0, accB = 0.0;
    for (int ac = aS; ac < aE; ac += BCA) {
        const int na = min(BCA, aE - ac);
        if (tid < na) {
            const BackParams p = A.bp[ac + tid];
            const double g00 = fma(Xlo, p.cg, fma(Ylo, p.sg, A.center));
            const double g01 = fma(Xlo, p.cg, fma(Yhi, p.sg, A.center));
            const double g10 = fma(Xhi, p.cg, fma(Ylo, p.sg, A.center));
            const double g11 = fma(Xhi, p.cg, fma(Yhi, p.sg, A.center));
            const double gmin = fmin(fmin(g00, g01), fmin(g10, g11));
            s_cg[tid] = p.cg;
            s_sg[tid] = p.sg;
            s_w0[tid] = (int)floor(gmin) - 1;
        }
        __syncthreads();
        // stage the detector windows, zero outside [0, D)
        for (int ai = ty; ai < na; ai += BROWS) {
            const float* row = A.u + (size_t)(ac + ai - A.a0) * D;
            const int w0 = s_w0[ai];
            float* dst = win + ai * wmax;
            for (int i = tx; i < wmax; i += BTX) {
                const int bin = w0 + i;
                dst[i] = (bin >= 0 && bin < D) ? __ldg(row + bin) : 0.f;
            }
        }
        __syncthreads();
        float sA = 0.f, sB = 0.f;
#pragma unroll 4
        for (int ai = 0; ai < na; ++ai) {
            const double cg = s_cg[ai], sg = s_sg[ai];
            const int w0 = s_w0[ai];
            const float* wrow = win + ai * wmax;
            const int iq = min(max(q1 - w0, 0), wmax - 1);
            {
                const double g = fma(X, cg, fma(YA, sg, A.center));
                const double fl = floor(g);
                const int i0 = (int)fl;
                const float w = (float)(g - fl);
                const int li = min(max(i0 - w0, 0), wmax - 2);
                const float v0 = wrow[li];
                const float v1 = (i0 == -1) ? wrow[iq] : wrow[li + 1];
                sA += fmaf(w, v1 - v0, v0);
            }
            {
                const double g = fma(X, cg, fma(YB, sg, A.center));
                const double fl = floor(g);
                const int i0 = (int)fl;
                const float w = (float)(g - fl);
                const int li = min(max(i0 - w0, 0), wmax - 2);
                const float v0 = wrow[li];
                const float v1 = (i0 == -1) ? wrow[iq] : wrow[li + 1];
                sB += fmaf(w, v1 - v0, v0);
            }
        }
        accA += (double)sA;
        accB += (double)sB;
        __syncthreads();
    }
    const size_t n = (size_t)A.nx * A.ny;
    if (A.split) {
        // angle split: the last of the gridDim.z CTAs of this tile sums the
        // partial images in split order (deterministic) and adds x0.
        float* part = A.out;
        const bool inx = ix < A.nx;
        if (inx && iyA < A.ny) part[(size_t)blockIdx.z * n + (size_t)iyA * A.nx + ix] = (float)accA;
        if (inx && iyB < A.ny) part[(size_t)blockIdx.z * n + (size_t)iyB * A.nx + ix] = (float)accB;
        __threadfence();
        __syncthreads();
        __shared__ unsigned s_last;
        unsigned* ticket = A.cnt + (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (tid == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.z - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (inx) {
            for (int r = 0; r < 2; ++r) {
                const int iy = r ? iyB : iyA;
                if (iy >= A.ny) continue;
                const size_t o = (size_t)iy * A.nx + ix;
                double t = 0.0;
                for (unsigned z = 0; z < gridDim.z; ++z) t += (double)__ldcg(part + z * n + o);
                A.x[o] = (float)((A.x0 ? (double)A.x0[o] : 0.0) + A.h * t);
            }
        }
        if (tid == 0) *ticket = 0u;
    } else {
        if (ix >= A.nx) return;
        if (iyA < A.ny) {
            const size_t o = (size_t)iyA * A.nx + ix;
            A.out[o] = (float)((A.x0 ? (double)A.x0[o] : 0.0) + A.h * accA);
        }
        if (iyB < A.ny) {
            const size_t o = (size_t)iyB * A.nx + ix;
            A.out[o] = (float)((A.x0 ? (double)A.x0[o] : 0.0) + A.h * accB);
        }
    }
}

static int back_splits(const ctk_geom* g, int a0, int a1) {
    const int tiles = ((g->nx + BTX - 1) / BTX) * ((g->ny + BTY - 1) / BTY);
    const int target = 148 * 4;
    int S = (target + tiles - 1) / tiles;
    const int max_s = (a1 - a0 + BCA - 1) / BCA;
    if (S > max_s) S = max_s;
    if (S < 1) S = 1;
    return S;
}

}  // namespace ctk

using namespace ctk;

static int64_t back_tiles(const ctk_geom* g) {
    return (int64_t)((g->nx + BTX - 1) / BTX) * ((g->ny + BTY - 1) / BTY);
}

extern "C" int64_t ctk_back_work_floats(const ctk_geom_t* g, int a0, int a1) {
    if (!g || a0 < 0 || a1 > g->n_angles || a0 >= a1) return 0;
    const int S = back_splits(g, a0, a1);
    return S > 1 ? (int64_t)S * g->nx * g->ny + back_tiles(g) : 0;
}

extern "C" int ctk_back(const ctk_geom_t* g, const float* u, float* x, int a0, int a1,
                        const float* x0, float* work, void* stream) {
    if (!g) return ctk_fail(CTK_ERR_ARG, "null geometry");
    if (a0 < 0 || a1 > g->n_angles || a0 > a1)
        return ctk_fail(CTK_ERR_SHAPE, "angle range [%d, %d) outside [0, %d)", a0, a1, g->n_angles);
    if (!u || !x) return ctk_fail(CTK_ERR_ARG, "null vector");
    CTK_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = ctk_stream(stream);
    const size_t n = (size_t)g->nx * g->ny;
    if (a1 == a0) {
        if (x0) CTK_CUDA(cudaMemcpyAsync(x, x0, n * sizeof(float), cudaMemcpyDeviceToDevice, st));
        else CTK_CUDA(cudaMemsetAsync(x, 0, n * sizeof(float), st));
        return CTK_OK;
    }
    const int S = back_splits(g, a0, a1);
    if (S > 1 && !work) return ctk_fail(CTK_ERR_ARG, "ctk_back needs %lld work floats",
                                        (long long)S * (long long)n);
    BackArgs A;
    A.bp = g->d_bp;
    A.u = u;
    A.x0 = x0;
    A.out = S > 1 ? work : x;
    A.x = x;
    A.cnt = S > 1 ? reinterpret_cast<unsigned*>(work + (size_t)S * n) : nullptr;
    A.nx = g->nx;
    A.ny = g->ny;
    A.D = g->det_count;
    A.a0 = a0;
    A.a1 = a1;
    A.per_split = (a1 - a0 + S - 1) / S;
    A.wmax = g->back_wmax;
    A.split = S > 1;
    A.h = g->h;
    A.xmin = g->xmin;
    A.ymax = g->ymax;
    A.center = g->center;
    dim3 grid((g->nx + BTX - 1) / BTX, (g->ny + BTY - 1) / BTY, S), block(BTX, BROWS);
    const size_t smem = (size_t)BCA * g->back_wmax * sizeof(float);
    if (smem > 48 * 1024)
        CTK_CUDA(cudaFuncSetAttribute(k_back, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      (int)smem));
    const int ph = ctk_prof_open(1, st);
    k_back<<<grid, block, smem, st>>>(A);
    CTK_LAUNCH_CHECK("k_back");
    ctk_prof_close(ph, st);
    return CTK_OK;
}
