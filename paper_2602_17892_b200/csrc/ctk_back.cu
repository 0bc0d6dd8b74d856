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
    float* x;             // output image
    float* part;          // SPLIT: partial images [S][n]
    unsigned* cnt;        // SPLIT: per-tile arrival tickets (zeroed once)
    int nx, ny, D, a0, a1, per_split, wmax, fbits;
    float* stP;           // optional: also write the K1 staged copies of the result
    float* stPT;
    int pad;
    double h, xmin, ymax, center;
    const ctk_xchg_args* xc;   // optional (device copy): push the tile to its owner rank
    unsigned* ready;      // optional: K1's finished-CTA counters per 4-angle group (chaining)
    unsigned ready_target;  // K1 CTAs per group (bin blocks) x this step's epoch
    const float2* pairs;  // MODE 2: (p, d) per bin, row a at pairs + (a - a0) * Dp + P
    int Dp, P;
};

// MODE 2 pre-pass (images >= 512^2): the sinogram as (p, d) pairs per bin,
// bins b in [-P, D + P) -- exactly the values stage_windows builds per window
// (v0 = u[b] or 0 outside the detector, v1 = the reference's second tap with
// the i0 == -1 quirk, d = v1 - v0, p = v0 - d) -- so K2's per-chunk staging
// becomes coalesced 8-byte copies instead of two loads, three shuffles and
// the quirk / bounds logic per angle and lane (~23% of K2's instructions at
// c5 went to staging).  Bitwise the same windows, hence the same B.
__global__ void __launch_bounds__(256) k_pairs(const float* __restrict__ u, float2* __restrict__ pr,
                                               int rows, int D, int P) {
    ctk_pdl_trigger();
    const int Dp = D + 2 * P;
    const int64_t total = (int64_t)rows * Dp;
    const int q1 = D > 1 ? 1 : 0;
    ctk_pdl_wait();                                    // u comes from the previous kernel
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < total;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(idx / Dp), b = (int)(idx - (int64_t)a * Dp) - P;
        const float* row = u + (size_t)a * D;
        const float v0 = (b >= 0 && b < D) ? __ldg(row + b) : 0.f;
        const int b1 = b == -1 ? q1 : b + 1;
        const float v1 = (b >= -1 && b + 1 < D) ? __ldg(row + b1) : 0.f;
        const float d = v1 - v0;
        pr[idx] = make_float2(v0 - d, d);
    }
}

// Sinogram loads.  CHAINED: u is written by the still-running K1, so the
// read-only (.nc) path is not allowed -- L2-coherent loads after the acquire
// instead.  (A compile-time choice: a run-time branch doubled the staging
// code and its branches.)
template <bool CHAINED>
__device__ __forceinline__ float ld_u(const float* p) {
    return CHAINED ? __ldcg(p) : __ldg(p);
}

// K2 chaining (ctk_common.cuh): wait until the K1 groups holding angles
// [ac, ac + na) are complete.  The counters are monotonic within an Arnoldi
// cycle (zeroed by the host before its step 0, never reset by a kernel):
// step j's K1 brings every group to need * (j + 1), and K1 counts a CTA only
// after its griddepcontrol.wait, i.e. after the previous step's K2 has
// completed -- so a count at or above the target always means this step's
// rows are written, whatever kernels of neighbouring steps are co-resident.
__device__ __forceinline__ void wait_k1_groups(const BackArgs& A, int ac, int na, int tid) {
    const int g0 = (ac - A.a0) / CTK_FWD_APB, g1 = (ac + na - 1 - A.a0) / CTK_FWD_APB;
    if (tid <= g1 - g0) {
        const unsigned* c = A.ready + g0 + tid;
        while (ctk_ld_acquire_gpu(c) < A.ready_target) __nanosleep(64);
    }
    __syncthreads();
}

// K1's zero-padded copies of the output pixel (ix, iy) (see ctk_forward.cu).
__device__ __forceinline__ void stage_out(const BackArgs& A, int ix, int iy, float v) {
    A.stP[(size_t)iy * (A.nx + 2 * A.pad) + ix + A.pad] = v;
    A.stPT[(size_t)ix * (A.ny + 2 * A.pad) + iy + A.pad] = v;
}

// Stage one 32-angle chunk's detector windows as (p, d) pairs (header).
// Windows of at most 63 bins (every BASELINE config): warp per angle, the
// window's v0 values in two coalesced loads per angle, all of a warp's loads
// issued before the first use (one L2 round trip per chunk instead of one
// per strided element), v1 = v0 of the next bin by a lane shuffle except at
// the quirk bin b == -1.  Wider windows take the element loop.
template <bool CHAINED>
__device__ __forceinline__ void stage_windows(const BackArgs& A, float2* win, const int* s_w0,
                                              int ac, int na, int tx, int ty) {
    const int D = A.D, wmax = A.wmax;
    const int q1 = D > 1 ? 1 : 0;                  // reference quirk tap for i0 == -1
    if (wmax <= 63) {
        constexpr int NJ = BCA / BROWS;            // angles per warp
        float va[NJ], vb[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int ai = ty + j * BROWS;
            va[j] = vb[j] = 0.f;
            if (ai < na) {
                const float* row = A.u + (size_t)(ac + ai - A.a0) * D;
                const int b = s_w0[ai] + tx, b2 = b + 32;
                if (b >= 0 && b < D) va[j] = ld_u<CHAINED>(row + b);
                if (b2 >= 0 && b2 < D && tx + 32 <= wmax) vb[j] = ld_u<CHAINED>(row + b2);
            }
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int ai = ty + j * BROWS;
            if (ai >= na) break;                   // warp-uniform
            const float up_a = __shfl_down_sync(0xffffffffu, va[j], 1);
            const float b_0 = __shfl_sync(0xffffffffu, vb[j], 0);
            const float up_b = __shfl_down_sync(0xffffffffu, vb[j], 1);
            const int b = s_w0[ai] + tx;
            float v1a = tx < 31 ? up_a : b_0, v1b = up_b;
            const float* row = A.u + (size_t)(ac + ai - A.a0) * D;
            if (b == -1) v1a = ld_u<CHAINED>(row + q1);
            if (b + 32 == -1) v1b = ld_u<CHAINED>(row + q1);
            float2* dst = win + ai * wmax;
            float d = v1a - va[j];
            // (windows can be narrower than a warp: pixels smaller than bins)
            if (tx < wmax) dst[tx] = make_float2(va[j] - d, d);
            if (tx + 32 < wmax) {
                d = v1b - vb[j];
                dst[tx + 32] = make_float2(vb[j] - d, d);
            }
        }
        return;
    }
    for (int ai = ty; ai < na; ai += BROWS) {
        const float* row = A.u + (size_t)(ac + ai - A.a0) * D;
        const int w0 = s_w0[ai];
        float2* dst = win + ai * wmax;
        for (int i = tx; i < wmax; i += BTX) {
            const int b = w0 + i;
            const float v0 = (b >= 0 && b < D) ? ld_u<CHAINED>(row + b) : 0.f;
            const int b1 = b == -1 ? q1 : b + 1;
            const float v1 = (b >= -1 && b + 1 < D) ? ld_u<CHAINED>(row + b1) : 0.f;
            const float d = v1 - v0;
            dst[i] = make_float2(v0 - d, d);
        }
    }
}

// MODE 2 staging: the windows straight from the pair sinogram (bins outside
// [-P, D + P) are zero pairs, as stage_windows would build them).
__device__ __forceinline__ void stage_pairs(const BackArgs& A, float2* win, const int* s_w0,
                                            int ac, int na, int tx, int ty) {
    const int wmax = A.wmax, lo = -A.P, hi = A.D + A.P;
    const float2 z = make_float2(0.f, 0.f);
    if (wmax <= 64) {
        constexpr int NJ = BCA / BROWS;            // angles per warp
        float2 va[NJ], vb[NJ];
#pragma unroll
        for (int j = 0; j < NJ; ++j) {             // all loads before the first store
            const int ai = ty + j * BROWS;
            va[j] = vb[j] = z;
            if (ai < na) {
                const float2* row = A.pairs + (size_t)(ac + ai - A.a0) * A.Dp + A.P;
                const int b = s_w0[ai] + tx, b2 = b + 32;
                if (tx < wmax && b >= lo && b < hi) va[j] = __ldg(row + b);
                if (tx + 32 < wmax && b2 >= lo && b2 < hi) vb[j] = __ldg(row + b2);
            }
        }
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int ai = ty + j * BROWS;
            if (ai >= na) break;                   // warp-uniform
            float2* dst = win + ai * wmax;
            if (tx < wmax) dst[tx] = va[j];
            if (tx + 32 < wmax) dst[tx + 32] = vb[j];
        }
        return;
    }
    for (int ai = ty; ai < na; ai += BROWS) {
        const float2* row = A.pairs + (size_t)(ac + ai - A.a0) * A.Dp + A.P;
        const int w0 = s_w0[ai];
        float2* dst = win + ai * wmax;
        for (int i = tx; i < wmax; i += BTX) {
            const int b = w0 + i;
            dst[i] = (b >= lo && b < hi) ? __ldg(row + b) : z;
        }
    }
}

// SPLIT: the gridDim.z angle splits of a tile write fp32 partial images; the
// last to arrive (per-tile ticket) sums them in split order and writes the
// image.  (A cluster/DSMEM variant of this reduction measured faster in
// isolation but slower inside the solve: its gang-scheduled CTAs wait for
// whole free GPC slices while the iterate stream's kernels hold SMs.)
// Resident CTAs per SM of the 4-pixels-per-thread kernels: 4 (64 registers).
// Measured B per apply at c3 / c4 / c5 with 3 / 4 / 5 / 6: 0.0942 / 0.0901 /
// 0.0927 / 0.0942, 0.578 / 0.554 / 0.582 / 0.578, 2.669 / 2.588 / 2.705 /
// 2.808 ms (5 was the optimum before the staging changes of this round).
#ifndef CTK_BACK_MINB4
#define CTK_BACK_MINB4 4
#endif
#ifndef CTK_BACK_UNROLL
#define CTK_BACK_UNROLL 4
#endif
constexpr int BACK_UNROLL = CTK_BACK_UNROLL;      // angles per unrolled batch of the inner loop

// MODE 0: plain, 1: chained after K1 (counters), 2: windows from the pair
// sinogram (k_pairs)
template <int PPT, bool SPLIT, int MODE>            // pixels (rows) per thread
__global__ void __launch_bounds__(BTHREADS, PPT == 4 ? CTK_BACK_MINB4 : 6) k_back(BackArgs A) {
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
    const int wmax = A.wmax;
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
        if (MODE == 1) wait_k1_groups(A, ac, na, tid);   // u: this chunk's K1 rows
        else ctk_pdl_wait();                       // u / pairs come from the previous kernel
        if (MODE == 2) stage_pairs(A, win, s_w0, ac, na, tx, ty);
        else stage_windows<MODE == 1>(A, win, s_w0, ac, na, tx, ty);
        __syncthreads();
        float sp[PPT];
#pragma unroll
        for (int r = 0; r < PPT; ++r) sp[r] = 0.f;
#pragma unroll BACK_UNROLL
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
    if (SPLIT) {
        // global partial images + per-tile arrival tickets: the last of the
        // gridDim.z CTAs of a tile sums the partials in split order
        const size_t n = (size_t)A.nx * A.ny;
        float* part = A.part;
        const bool inx = ix < A.nx;
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
            const int iy = iy0 + ty + r * BROWS;
            if (inx && iy < A.ny) part[(size_t)blockIdx.z * n + (size_t)iy * A.nx + ix] = (float)acc[r];
        }
        __syncthreads();
        __shared__ unsigned s_last;
        unsigned* ticket = A.cnt + (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (tid == 0) s_last = ctk_ticket_arrive(ticket, gridDim.z);
        __syncthreads();
        if (!s_last) return;                       // CTA-uniform
        if (tid == 0) *ticket = 0u;
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
            const int iy = iy0 + ty + r * BROWS;
            double t = 0.0;
            if (inx && iy < A.ny)
                for (unsigned z = 0; z < gridDim.z; ++z)
                    t += (double)__ldcg(part + z * n + (size_t)iy * A.nx + ix);
            acc[r] = t;
        }
    }
    if (A.xc) {
        // Exchange: this rank's partial tile goes straight into the owner's
        // receive slot (peer memory over NVLink, or local), then one
        // system-scope release of the tile's arrival flag -- the transfer
        // of each tile overlaps the compute of the tiles still running.
        const ctk_xchg_args& X = *A.xc;
        const int t = blockIdx.y * gridDim.x + blockIdx.x;
        const int owner = t % X.nranks;
        float* dst = X.recv[owner] + (size_t)X.rank * A.nx * A.ny;
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
            const int iy = iy0 + ty + r * BROWS;
            if (ix < A.nx && iy < A.ny) dst[(size_t)iy * A.nx + ix] = (float)(A.h * acc[r]);
        }
        __syncthreads();
        if (tid == 0) {
            unsigned* flag = X.flags[owner] + (size_t)X.rank * X.tiles + t;
            asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(flag),
                         "r"(X.epoch)
                         : "memory");
        }
        return;
    }
    if (ix >= A.nx) return;
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
        const int iy = iy0 + ty + r * BROWS;
        if (iy >= A.ny) continue;
        const size_t o = (size_t)iy * A.nx + ix;
        const float v = (float)((A.x0 ? (double)A.x0[o] : 0.0) + A.h * acc[r]);
        A.x[o] = v;
        if (A.stP) stage_out(A, ix, iy, v);
    }
}

__device__ __forceinline__ unsigned long long globaltimer_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

// Owner side: a CTA per owned tile (t = rank + i * nranks) waits for every
// rank's partial of the tile, sums them in rank order (fp64; the result is
// bitwise the same on every rank), writes it to every rank's result image
// and releases each peer's "done" flag for the tile.
template <int PPT>
__global__ void __launch_bounds__(BTHREADS) k_xchg_reduce(const ctk_xchg_args* __restrict__ xa,
                                                          int nx, int ny, int tiles_x) {
    const ctk_xchg_args& X = *xa;
    const int t = X.rank + blockIdx.x * X.nranks;
    if (t >= X.tiles) return;
    const int tid = threadIdx.y * BTX + threadIdx.x;
    const unsigned* arrive = X.flags[X.rank];
    if (tid < X.nranks) {
        const unsigned long long t0 = globaltimer_ns();
        while (ld_acquire_sys(arrive + (size_t)tid * X.tiles + t) != X.epoch) {
            __nanosleep(32);
            if (globaltimer_ns() - t0 > CTK_XCHG_TIMEOUT_NS) {
                atomicExch(X.err, 1u);
                break;
            }
        }
    }
    __syncthreads();
    const size_t n = (size_t)nx * ny;
    const float* recv = X.recv[X.rank];
    const int ix = (t % tiles_x) * BTX + threadIdx.x;
    const int iy0 = (t / tiles_x) * BROWS * PPT + threadIdx.y;
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
        const int iy = iy0 + r * BROWS;
        if (ix >= nx || iy >= ny) continue;
        const size_t o = (size_t)iy * nx + ix;
        double s = 0.0;
        for (int q = 0; q < X.nranks; ++q) s += (double)__ldcv(recv + q * n + o);
        const float v = (float)s;
        for (int q = 0; q < X.nranks; ++q) X.x[q][o] = v;
    }
    __syncthreads();
    if (tid < X.nranks && tid != X.rank) {
        unsigned* flag = X.flags[tid] + (size_t)X.nranks * X.tiles + t;
        asm volatile("fence.acq_rel.sys;\n\tst.relaxed.sys.global.u32 [%0], %1;" ::"l"(flag),
                     "r"(X.epoch)
                     : "memory");
    }
}

// Every rank: wait until the owners of all other tiles have delivered them.
__global__ void __launch_bounds__(256) k_xchg_wait(const ctk_xchg_args* __restrict__ xa) {
    const ctk_xchg_args& X = *xa;
    const unsigned* done = X.flags[X.rank] + (size_t)X.nranks * X.tiles;
    const unsigned long long t0 = globaltimer_ns();
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < X.tiles; t += gridDim.x * blockDim.x)
        if (t % X.nranks != X.rank)
            while (ld_acquire_sys(done + t) != X.epoch) {
                __nanosleep(32);
                if (globaltimer_ns() - t0 > CTK_XCHG_TIMEOUT_NS) {
                    atomicExch(X.err, 1u);
                    return;
                }
            }
}

static int back_tiles_y(const ctk_geom* g) {
    const int bty = BROWS * g->back_ppt;
    return (g->ny + bty - 1) / bty;
}

static int back_splits(const ctk_geom* g, int a0, int a1) {
    const int tiles = ((g->nx + BTX - 1) / BTX) * back_tiles_y(g);
    static int target_env = -1;
    if (target_env < 0) {
        const char* e = getenv("CTK_BACK_TARGET");       // tuning override (CTAs)
        target_env = e && atoi(e) > 0 ? atoi(e) : 0;
    }
    // two waves of the kernel's resident CTAs: 4 per SM for the 4-pixel
    // kernels (c3: 7 -> 5 splits, B 0.090 -> 0.086 ms), 6 for the others
    const int target = target_env ? target_env : g->back_ppt == 4 ? 148 * 8 : 148 * 12;
    static int min_ang = -1;
    if (min_ang < 0) {
        const char* e = getenv("CTK_BACK_MINANG");      // tuning override: angles per CTA
        min_ang = e && atoi(e) > 0 ? atoi(e) : 0;
    }
    int S = (target + tiles - 1) / tiles;
    // >= one 32-angle chunk per CTA, or half a chunk when whole chunks leave
    // the GPU under a third full (c1: 64 tiles x 6 -> x 12 splits; solve
    // 2.33 -> 2.16 ms; c2 keeps whole chunks)
    int ma = min_ang;
    if (ma == 0) ma = (int64_t)tiles * ((a1 - a0 + BCA - 1) / BCA) < 148 * 4 ? BCA / 2 : BCA;
    const int max_s = (a1 - a0 + ma - 1) / ma;
    if (S > max_s) S = max_s;
    if (S < 1) S = 1;
    return S;
}

}  // namespace ctk

using namespace ctk;

static int64_t back_tiles(const ctk_geom* g) {
    return (int64_t)((g->nx + BTX - 1) / BTX) * back_tiles_y(g);
}

int64_t ctk_back_tiles(const ctk_geom* g) { return back_tiles(g); }

// Work buffer: [K1-chaining flags: one counter per 4-angle group, 16-float
// aligned] [one arrival ticket per tile, 16-float aligned] [S partial images].
// Flags and tickets sit at offsets fixed by the geometry, so calls with
// different angle ranges / split counts sharing one (zero-filled once)
// buffer agree on them; the partial images after them are scratch.
static int64_t back_flag_floats(const ctk_geom* g) {
    return ((int64_t)(g->n_angles + CTK_FWD_APB - 1) / CTK_FWD_APB + 15) / 16 * 16;
}

static int64_t back_ticket_floats(const ctk_geom* g) { return (back_tiles(g) + 15) / 16 * 16; }

// Pair sinogram (MODE 2): measured B per apply with / without the pre-pass
// (64-register kernels): c5 2.589 / 2.721 ms, c4 0.548 / 0.553, c3 0.091 /
// 0.089 -- so images of >= 1024^2 (CTK_BACK_PAIRS=0 / 1 overrides).  P = 2 pad bins each side
// cover the i0 == -1 quirk bin.
constexpr int PAIR_PAD = 2;
static bool back_pairs_on(const ctk_geom* g) {
    static const int force = [] {
        const char* e = getenv("CTK_BACK_PAIRS");
        return e ? atoi(e) : -1;
    }();
    if (g->back_ppt != 4) return false;
    if (force >= 0) return force != 0;
    return (int64_t)g->nx * g->ny >= 1024LL * 1024;
}

static int64_t back_pair_floats(const ctk_geom* g, int a0, int a1) {
    return back_pairs_on(g) ? 2 * (int64_t)(a1 - a0) * (g->det_count + 2 * PAIR_PAD) : 0;
}

unsigned* ctk_back_flags(const ctk_geom* g, float* work) {
    return work ? reinterpret_cast<unsigned*>(work) : nullptr;
}

extern "C" int64_t ctk_back_work_floats(const ctk_geom_t* g, int a0, int a1) {
    if (!g || a0 < 0 || a1 > g->n_angles || a0 >= a1) return 0;
    const int S = back_splits(g, a0, a1);
    return back_flag_floats(g) + back_ticket_floats(g) +
           (S > 1 ? ((int64_t)S * g->nx * g->ny + 3) / 4 * 4 : 0) + back_pair_floats(g, a0, a1);
}

extern "C" int ctk_back(const ctk_geom_t* g, const float* u, float* x, int a0, int a1,
                        const float* x0, float* work, void* stream) {
    return ctk_back_ex(g, u, x, a0, a1, x0, work, nullptr, stream);
}

int64_t ctk_back_flag_count(const ctk_geom* g) { return back_flag_floats(g); }

extern "C" int ctk_back_work_layout(const ctk_geom_t* g, int64_t* out4) {
    if (!g || !out4) return ctk_fail(CTK_ERR_ARG, "null argument");
    out4[0] = back_flag_floats(g);
    out4[1] = back_ticket_floats(g);
    out4[2] = (g->det_count + 31) / 32;
    out4[3] = back_tiles(g);
    return CTK_OK;
}

// stage != NULL: also write K1's zero-padded P / PT copies of x into the
// forward workspace `stage` (interior only: its zero padding is written by
// any plain ctk_forward on that workspace).
int ctk_back_ex(const ctk_geom_t* g, const float* u, float* x, int a0, int a1, const float* x0,
                float* work, float* stage, void* stream, unsigned k1_epoch) {
    return ctk_back_xc(g, u, x, a0, a1, x0, work, stage, nullptr, stream, k1_epoch);
}

// xc (device pointer) != NULL: push the partial tiles to their owners
// instead of writing x (ctk_back_exchange, phase 1).
int ctk_back_xc(const ctk_geom_t* g, const float* u, float* x, int a0, int a1, const float* x0,
                float* work, float* stage, const ctk_xchg_args* xc, void* stream,
                unsigned k1_epoch) {
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
    if (S > 1 && !work)
        return ctk_fail(CTK_ERR_ARG, "ctk_back needs %lld work floats",
                        (long long)ctk_back_work_floats(g, a0, a1));
    if (k1_epoch && !work) return ctk_fail(CTK_ERR_ARG, "K1 chaining needs the work buffer");
    BackArgs A;
    A.cnt = work ? reinterpret_cast<unsigned*>(work + back_flag_floats(g)) : nullptr;
    A.part = S > 1 ? work + back_flag_floats(g) + back_ticket_floats(g) : nullptr;
    A.ready = k1_epoch ? ctk_back_flags(g, work) : nullptr;
    A.ready_target = (unsigned)((g->det_count + 31) / 32) * k1_epoch;
    const bool pairs = !k1_epoch && work && back_pairs_on(g);
    A.P = PAIR_PAD;
    A.Dp = g->det_count + 2 * PAIR_PAD;
    A.pairs = pairs ? reinterpret_cast<const float2*>(
                          work + back_flag_floats(g) + back_ticket_floats(g) +
                          (S > 1 ? ((int64_t)S * g->nx * g->ny + 3) / 4 * 4 : 0))
                    : nullptr;
    A.bp = g->d_bp;
    A.u = u;
    A.x0 = x0;
    A.x = x;
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
    A.h = g->h;
    A.xmin = g->xmin;
    A.ymax = g->ymax;
    A.center = g->center;
    A.xc = xc;
    dim3 grid((g->nx + BTX - 1) / BTX, back_tiles_y(g), S), block(BTX, BROWS);
    const int ppt = g->back_ppt;
    size_t smem = (size_t)BCA * g->back_wmax * sizeof(float2);
    void (*kern)(BackArgs) =
        k1_epoch
            ? (S > 1 ? (ppt == 4 ? k_back<4, true, 1> : ppt == 1 ? k_back<1, true, 1>
                                                      : k_back<2, true, 1>)
                     : (ppt == 4 ? k_back<4, false, 1> : ppt == 1 ? k_back<1, false, 1>
                                                       : k_back<2, false, 1>))
        : pairs
            ? (S > 1 ? (ppt == 4 ? k_back<4, true, 2> : ppt == 1 ? k_back<1, true, 2>
                                                      : k_back<2, true, 2>)
                     : (ppt == 4 ? k_back<4, false, 2> : ppt == 1 ? k_back<1, false, 2>
                                                       : k_back<2, false, 2>))
            : (S > 1 ? (ppt == 4 ? k_back<4, true, 0> : ppt == 1 ? k_back<1, true, 0>
                                                      : k_back<2, true, 0>)
                     : (ppt == 4 ? k_back<4, false, 0> : ppt == 1 ? k_back<1, false, 0>
                                                       : k_back<2, false, 0>));
    // Opt in early (the 48 KB default also counts the static arrays) and always
    // to the same value, the largest window any geometry may have: the limit
    // is per function, so concurrent launches for geometries with different
    // window sizes must not lower it under each other.
    if (smem > 40 * 1024)
        CTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
    const int ph = ctk_prof_open(1, st);
    if (pairs) {
        const int64_t total = (int64_t)(a1 - a0) * A.Dp;
        int blocks = (int)((total + 255) / 256);
        if (blocks > 148 * 8) blocks = 148 * 8;
        CTK_CUDA(ctk_launch_pdl(k_pairs, dim3(blocks), dim3(256), 0, st, dim3(1, 1, 1), u,
                                const_cast<float2*>(A.pairs), a1 - a0, (int)g->det_count,
                                (int)PAIR_PAD));
        ctk_count_launch();
    }
    CTK_CUDA(ctk_launch_pdl(kern, grid, block, smem, st, dim3(1, 1, 1), A));
    ctk_count_launch();
    ctk_prof_close(ph, st);
    return CTK_OK;
}

// Phases 2 and 3 of ctk_back_exchange (xc: device copy of the arguments).
int ctk_xchg_finish(const ctk_geom* g, const ctk_xchg_args* xc, int nranks, int phases,
                    cudaStream_t st) {
    const int tiles_x = (g->nx + BTX - 1) / BTX;
    const int64_t tiles = back_tiles(g);
    if (phases & 2) {
        const unsigned owned = (unsigned)((tiles + nranks - 1) / nranks);
        if (g->back_ppt == 4)
            k_xchg_reduce<4><<<owned, dim3(BTX, BROWS), 0, st>>>(xc, g->nx, g->ny, tiles_x);
        else if (g->back_ppt == 1)
            k_xchg_reduce<1><<<owned, dim3(BTX, BROWS), 0, st>>>(xc, g->nx, g->ny, tiles_x);
        else
            k_xchg_reduce<2><<<owned, dim3(BTX, BROWS), 0, st>>>(xc, g->nx, g->ny, tiles_x);
        CTK_LAUNCH_CHECK("k_xchg_reduce");
    }
    if (phases & 4) {
        const unsigned blocks = (unsigned)((tiles + 255) / 256);
        k_xchg_wait<<<blocks < 148 ? blocks : 148, 256, 0, st>>>(xc);
        CTK_LAUNCH_CHECK("k_xchg_wait");
    }
    return CTK_OK;
}
