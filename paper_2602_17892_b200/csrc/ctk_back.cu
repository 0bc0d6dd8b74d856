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
// stages, per angle, the short detector window its tile projects onto into
// shared memory with coalesced loads, as (p, d) pairs per bin b:
//   v0 = u[b] (0 outside [0, D)),  v1 = the reference's second tap for i0 = b
//   (u[b+1], 0 outside, u[1] for b == -1: the quirk is baked into the window),
//   d = v1 - v0,  p = v0 - d,   so  (1 - w) v0 + w v1 = p + (1 + w) d.
// g is evaluated in fixed point: the tile origin's g (fp64, the reference's
// geometry) becomes T0 = (g - w0) * 2^F and the per-pixel steps h cg, -h sg
// become 32-bit integers C, S with F = 32 - ceil(log2(wmax + 1)) fraction bits
// (26 for the BASELINE configs), so every pixel's T = T0 + dx C + dy S is one
// integer multiply-add with |error| <= 47 * 2^-(F+1) bin (~3.5e-7 at F = 26).
// No hardware texture lerp (its 8-bit fraction would break the 1e-5 bar) and
// no fp64 / conversion-pipe work per pixel-angle (FRND/F2I/F2F.F64 bounded the
// previous version): T >> F indexes the pair, the top 23 fraction bits OR'ed
// into 1.0f give 1 + w, and the tap is one FFMA.  Each 32-angle partial sum
// is folded into an fp64 accumulator.  Small images split the angle range
// over blockIdx.z into partial images reduced in a fixed order.
#include <math.h>
#include <stdlib.h>

#include "ctk_common.cuh"

namespace ctk {

constexpr int BTX = 32, BROWS = 8, BCA = 32;      // tile: BTX x (BROWS * PPT) pixels
constexpr int BTHREADS = BTX * BROWS;

struct BackArgs {
    const BackParams* bp;
    const float* u;       // row a at u + (a - a0) * D
    const float* x0;      // optional
    float* out;           // final image (S == 1) or partials [S][n]
    float* x;             // final image (S > 1)
    unsigned* cnt;        // S > 1: per-tile arrival tickets (zeroed once)
    int nx, ny, D, a0, a1, per_split, wmax, split, fbits;
    float* stP;           // optional: also write the K1 staged copies of the result
    float* stPT;
    int pad;
    double h, xmin, ymax, center;
};

// K1's zero-padded copies of the output pixel (ix, iy) (see ctk_forward.cu).
__device__ __forceinline__ void stage_out(const BackArgs& A, int ix, int iy, float v) {
    A.stP[(size_t)iy * (A.nx + 2 * A.pad) + ix + A.pad] = v;
    A.stPT[(size_t)ix * (A.ny + 2 * A.pad) + iy + A.pad] = v;
}

template <int PPT>                                 // pixels (rows) per thread
__global__ void __launch_bounds__(BTHREADS) k_back(BackArgs A) {
    constexpr int BTY = BROWS * PPT;
    extern __shared__ float2 win[];                // [BCA][wmax] (p, d)
    __shared__ int4 s_par[BCA];                    // T0, C, S, smem base of the window
    __shared__ int s_w0[BCA];

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * BTX + tx;
    const int ix0 = blockIdx.x * BTX, iy0 = blockIdx.y * BTY;
    const int ix = ix0 + tx;
    // tile corner pixel centres
    const double Xlo = A.xmin + ((double)ix0 + 0.5) * A.h;
    const double Xhi = A.xmin + ((double)(ix0 + BTX - 1) + 0.5) * A.h;
    const double Yhi = A.ymax - ((double)iy0 + 0.5) * A.h;
    const double Ylo = A.ymax - ((double)(iy0 + BTY - 1) + 0.5) * A.h;
    const int F = A.fbits, I = 32 - A.fbits;
    const double scale = ldexp(1.0, F);

    const int aS = A.a0 + blockIdx.z * A.per_split;
    const int aE = min(A.a1, aS + A.per_split);
    const int D = A.D, wmax = A.wmax;
    const int q1 = D > 1 ? 1 : 0;                  // reference quirk tap for i0 == -1
    ctk_pdl_trigger();

    double acc[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) acc[r] = 0.0;
    for (int ac = aS; ac < aE; ac += BCA) {
        const int na = min(BCA, aE - ac);
        if (tid < na) {
            const BackParams p = A.bp[ac + tid];
            const double g00 = fma(Xlo, p.cg, fma(Ylo, p.sg, A.center));
            const double g01 = fma(Xlo, p.cg, fma(Yhi, p.sg, A.center));
            const double g10 = fma(Xhi, p.cg, fma(Ylo, p.sg, A.center));
            const double g11 = fma(Xhi, p.cg, fma(Yhi, p.sg, A.center));
            const double gmin = fmin(fmin(g00, g01), fmin(g10, g11));
            const int w0 = (int)floor(gmin) - 1;
            s_w0[tid] = w0;
            // origin = pixel (ix0, iy0), i.e. g01 at (Xlo, Yhi)
            const unsigned T0 = (unsigned)llrint((g01 - (double)w0) * scale);
            const int C = (int)llrint(p.cg * A.h * scale);
            const int S = (int)llrint(-p.sg * A.h * scale);
            s_par[tid] = make_int4((int)T0, C, S,
                                   (int)(unsigned)__cvta_generic_to_shared(win + tid * wmax));
        }
        __syncthreads();
        ctk_pdl_wait();                            // u comes from the previous kernel
        // stage the (p, d) windows; zero taps outside [0, D), quirk at b == -1
        for (int ai = ty; ai < na; ai += BROWS) {
            const float* row = A.u + (size_t)(ac + ai - A.a0) * D;
            const int w0 = s_w0[ai];
            float2* dst = win + ai * wmax;
            for (int i = tx; i < wmax; i += BTX) {
                const int b = w0 + i;
                const float v0 = (b >= 0 && b < D) ? __ldg(row + b) : 0.f;
                const int b1 = b == -1 ? q1 : b + 1;
                const float v1 = (b >= -1 && b + 1 < D) ? __ldg(row + b1) : 0.f;
                const float d = v1 - v0;
                dst[i] = make_float2(v0 - d, d);
            }
        }
        __syncthreads();
        float sp[PPT];
#pragma unroll
        for (int r = 0; r < PPT; ++r) sp[r] = 0.f;
#pragma unroll 4
        for (int ai = 0; ai < na; ++ai) {
            const int4 P = s_par[ai];
            const unsigned T0 = (unsigned)P.x + (unsigned)tx * (unsigned)P.y + (unsigned)ty * (unsigned)P.z;
            const unsigned dT = (unsigned)BROWS * (unsigned)P.z;
#pragma unroll
            for (int r = 0; r < PPT; ++r) {
                const unsigned T = T0 + (unsigned)r * dT;
                const float f1 = __uint_as_float(0x3f800000u | ((T << I) >> 9));   // 1 + w
                float2 pd;
                asm("ld.shared.v2.f32 {%0, %1}, [%2];"
                    : "=f"(pd.x), "=f"(pd.y) : "r"((T >> F) * 8u + (unsigned)P.w));
                sp[r] += fmaf(f1, pd.y, pd.x);
            }
        }
#pragma unroll
        for (int r = 0; r < PPT; ++r) acc[r] += (double)sp[r];
        __syncthreads();
    }
    const size_t n = (size_t)A.nx * A.ny;
    if (A.split) {
        // angle split: the last of the gridDim.z CTAs of this tile sums the
        // partial images in split order (deterministic) and adds x0.
        float* part = A.out;
        const bool inx = ix < A.nx;
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
            const int iy = iy0 + ty + r * BROWS;
            if (inx && iy < A.ny) part[(size_t)blockIdx.z * n + (size_t)iy * A.nx + ix] = (float)acc[r];
        }
        __threadfence();
        __syncthreads();
        __shared__ unsigned s_last;
        unsigned* ticket = A.cnt + (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (tid == 0) s_last = (atomicAdd(ticket, 1u) == gridDim.z - 1);
        __syncthreads();
        if (!s_last) return;
        __threadfence();
        if (inx) {
            for (int r = 0; r < PPT; ++r) {
                const int iy = iy0 + ty + r * BROWS;
                if (iy >= A.ny) continue;
                const size_t o = (size_t)iy * A.nx + ix;
                double t = 0.0;
                for (unsigned z = 0; z < gridDim.z; ++z) t += (double)__ldcg(part + z * n + o);
                const float v = (float)((A.x0 ? (double)A.x0[o] : 0.0) + A.h * t);
                A.x[o] = v;
                if (A.stP) stage_out(A, ix, iy, v);
            }
        }
        if (tid == 0) *ticket = 0u;
    } else {
        if (ix >= A.nx) return;
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
            const int iy = iy0 + ty + r * BROWS;
            if (iy >= A.ny) continue;
            const size_t o = (size_t)iy * A.nx + ix;
            const float v = (float)((A.x0 ? (double)A.x0[o] : 0.0) + A.h * acc[r]);
            A.out[o] = v;
            if (A.stP) stage_out(A, ix, iy, v);
        }
    }
}

static int back_tiles_y(const ctk_geom* g) {
    const int bty = BROWS * g->back_ppt;
    return (g->ny + bty - 1) / bty;
}

static int back_splits(const ctk_geom* g, int a0, int a1) {
    const int tiles = ((g->nx + BTX - 1) / BTX) * back_tiles_y(g);
    static int target = -1;
    if (target < 0) {
        const char* e = getenv("CTK_BACK_TARGET");       // tuning override (CTAs)
        target = e && atoi(e) > 0 ? atoi(e) : 148 * 12;   // ~1.5 waves of 256-thread CTAs
    }
    int S = (target + tiles - 1) / tiles;
    const int max_s = (a1 - a0 + BCA - 1) / BCA;      // >= one 32-angle chunk per CTA
    if (S > max_s) S = max_s;
    if (S < 1) S = 1;
    return S;
}

}  // namespace ctk

using namespace ctk;

static int64_t back_tiles(const ctk_geom* g) {
    return (int64_t)((g->nx + BTX - 1) / BTX) * back_tiles_y(g);
}

extern "C" int64_t ctk_back_work_floats(const ctk_geom_t* g, int a0, int a1) {
    if (!g || a0 < 0 || a1 > g->n_angles || a0 >= a1) return 0;
    const int S = back_splits(g, a0, a1);
    return S > 1 ? (int64_t)S * g->nx * g->ny + back_tiles(g) : 0;
}

extern "C" int ctk_back(const ctk_geom_t* g, const float* u, float* x, int a0, int a1,
                        const float* x0, float* work, void* stream) {
    return ctk_back_ex(g, u, x, a0, a1, x0, work, nullptr, stream);
}

// stage != NULL: also write K1's zero-padded P / PT copies of x into the
// forward workspace `stage` (interior only: its zero padding is written by
// any plain ctk_forward on that workspace).
int ctk_back_ex(const ctk_geom_t* g, const float* u, float* x, int a0, int a1, const float* x0,
                float* work, float* stage, void* stream) {
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
    A.pad = g->fwd_pad;
    A.stP = stage;
    A.stPT = stage ? stage + (size_t)g->ny * (g->nx + 2 * g->fwd_pad) : nullptr;
    {   // fixed-point fraction bits: window coordinates [0, wmax] need I bits
        int I = 1;
        while ((1 << I) <= g->back_wmax + 1) ++I;
        A.fbits = 32 - I;
    }
    A.split = S > 1;
    A.h = g->h;
    A.xmin = g->xmin;
    A.ymax = g->ymax;
    A.center = g->center;
    dim3 grid((g->nx + BTX - 1) / BTX, back_tiles_y(g), S), block(BTX, BROWS);
    const size_t smem = (size_t)BCA * g->back_wmax * sizeof(float2);
    const bool p4 = g->back_ppt == 4;
    if (smem > 48 * 1024)
        CTK_CUDA(cudaFuncSetAttribute(p4 ? k_back<4> : k_back<2>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int ph = ctk_prof_open(1, st);
    CTK_CUDA(ctk_launch_pdl(p4 ? k_back<4> : k_back<2>, grid, block, smem, st, dim3(1, 1, 1), A));
    ctk_count_launch();
    ctk_prof_close(ph, st);
    return CTK_OK;
}
