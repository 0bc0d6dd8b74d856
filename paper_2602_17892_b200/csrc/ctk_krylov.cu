// ctk_krylov.cu -- K3 (fused CGS2 orthogonalisation), K4 (basis combination)
// and the fp64 norm/dot epilogues (K5) for the Arnoldi process.
//
// Reference: ctkrylov/arnoldi.py:56-82 (MGS + full reorthogonalisation in
// fp64 numpy) and ctkrylov/gmres.py:205-211 (W @ y, x0 + ..., norms).
//
// The basis lives on the device as fp32 rows W[j][0..L) (row pitch ld, 16-B
// aligned) -- HBM-resident for the whole solve, never copied.  Every kernel
// streams rows with 128-bit loads and accumulates in fp64.
//
// Dots use a 2-D grid (L-chunk x group of 8 rows) so that even the small
// Krylov vectors of c1/c2 (33k-65k floats) spread over hundreds of CTAs with 8
// independent 16-B loads in flight per thread.  Reductions are a fixed tree:
// warp shuffles, a per-CTA smem pass, one fp64 partial per (chunk, row), and a
// last-CTA-done pass (integer ticket, no float atomics) that sums the chunk
// partials in a fixed order -- bitwise reproducible run to run.
#include <cooperative_groups.h>
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <unordered_map>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ctk_common.cuh"

namespace ctk {

constexpr int KT = 256;            // dots: threads per CTA
constexpr int KWARPS = KT / 32;
constexpr int JG = 8;              // rows per dots CTA
constexpr int MAXCH = 1024;        // max L-chunks (= partial rows)
constexpr int CT = 256;            // combine: threads per CTA
constexpr int KMAX_VEC = 4096;     // rows per call (smem bound of k_combine)

// Gram matrix E = W^T W - I of the stored basis rows (fp32, symmetric,
// [GRAM_LD][GRAM_LD]), kept by the single-launch Gram-Schmidt paths across the
// steps of one Arnoldi cycle (see gram_coefs).
constexpr int GRAM_LD = 128;
constexpr size_t GRAM_BYTES = sizeof(float) * GRAM_LD * GRAM_LD;

struct Scratch {                   // carved from the caller's zero-filled scratch
    unsigned int* ticket;          // [1]
    float* gram;                   // [GRAM_LD][GRAM_LD]
    double* partial;               // [MAXCH][nvec_cap]
    double* tmp;                   // [3][nvec_cap]
    int nvec_cap;
};

static inline Scratch carve(void* scratch, int nvec_cap) {
    char* p = (char*)scratch;
    Scratch s;
    s.ticket = (unsigned int*)p;
    s.gram = (float*)(p + 256);
    s.partial = (double*)(p + 256 + GRAM_BYTES);
    s.tmp = s.partial + (size_t)MAXCH * nvec_cap;
    s.nvec_cap = nvec_cap;
    return s;
}

// float4 per chunk: at least one per thread, at most MAXCH chunks.
static inline int64_t chunk_len(int64_t L4) {
    int64_t ch = (L4 + MAXCH - 1) / MAXCH;
    ch = (ch + KT - 1) / KT * KT;
    return ch < KT ? KT : ch;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double dot4(float4 a, float4 b, double acc) {
    acc = fma((double)a.x, (double)b.x, acc);
    acc = fma((double)a.y, (double)b.y, acc);
    acc = fma((double)a.z, (double)b.z, acc);
    acc = fma((double)a.w, (double)b.w, acc);
    return acc;
}

// Last CTA of the grid sums partial[c * nv + j] over chunks c in a fixed
// order (lane-strided, then a fixed shuffle tree) and writes out[j].
__device__ void last_cta_reduce(const double* partial, int nchunks, int nv, unsigned int* ticket,
                                double* out, unsigned arrivals = 0) {
    __shared__ unsigned int s_last;
    __syncthreads();
    if (arrivals == 0) arrivals = gridDim.x * gridDim.y;
    if (threadIdx.x == 0)
        s_last = ctk_ticket_arrive(ticket, arrivals);
    __syncthreads();
    if (!s_last) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = warp; j < nv; j += nw) {
        double s = 0.0;
        for (int c = lane; c < nchunks; c += 32) s += __ldcg(partial + (size_t)c * nv + j);
        s = warp_sum(s);
        if (lane == 0) out[j] = s;
    }
    if (threadIdx.x == 0) *ticket = 0u;   // ready for the next stream-ordered call
}

// out[j] = <W_j, v> (j < nvec); out[nvec] = <v, v> if want_norm.
// grid = (nchunks, ceil(nv / JG)).
// 3 resident CTAs per SM (79 registers) instead of the 2 that 96 allow: the
// multi-kernel CGS2 of the angle-sharded AB solve, c4 at world size 1,
// 0.585 -> 0.539 ms per step (solve 178.9 -> 173.2 ms)
#ifndef CTK_DOTS_MINB
#define CTK_DOTS_MINB 3
#endif
__global__ void __launch_bounds__(KT, CTK_DOTS_MINB) k_dots(const float* __restrict__ W, int64_t ld, int nvec,
                                             const float* __restrict__ v, int64_t L, int want_norm,
                                             int64_t ch, double* out, double* partial,
                                             unsigned int* ticket) {
    __shared__ double red[JG][KWARPS];
    const int nv = nvec + (want_norm ? 1 : 0);
    const int j0 = blockIdx.y * JG;
    const int nj = min(JG, nv - j0);
    const int64_t L4 = L >> 2;
    const int64_t i0 = (int64_t)blockIdx.x * ch, i1 = min(L4, i0 + ch);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const float4* rows[JG];
#pragma unroll
    for (int q = 0; q < JG; ++q) {
        const int j = j0 + (q < nj ? q : 0);
        rows[q] = reinterpret_cast<const float4*>(j < nvec ? W + (size_t)j * ld : v);
    }
    double acc[JG];
#pragma unroll
    for (int q = 0; q < JG; ++q) acc[q] = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += KT) {
        const float4 vv = __ldg(v4 + i);
        float4 w[JG];
#pragma unroll
        for (int q = 0; q < JG; ++q)
            if (q < nj) w[q] = __ldg(rows[q] + i);
#pragma unroll
        for (int q = 0; q < JG; ++q)
            if (q < nj) acc[q] = dot4(w[q], vv, acc[q]);
    }
    if (blockIdx.x == gridDim.x - 1) {     // scalar tail L % 4
        for (int64_t i = (L4 << 2) + threadIdx.x; i < L; i += KT) {
            const double vv = (double)v[i];
#pragma unroll
            for (int q = 0; q < JG; ++q)
                if (q < nj) acc[q] = fma((double)reinterpret_cast<const float*>(rows[q])[i], vv, acc[q]);
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < JG; ++q) {
        const double s = warp_sum(acc[q]);
        if (lane == 0) red[q][warp] = s;
    }
    __syncthreads();
    if (threadIdx.x < nj) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < KWARPS; ++w) s += red[threadIdx.x][w];
        partial[(size_t)blockIdx.x * nv + j0 + threadIdx.x] = s;
    }
    last_cta_reduce(partial, gridDim.x, nv, ticket, out);
}

// dst = (base ? base : 0) + sgn * sum_j coef[j] W_j ; optional ||dst||^2.
// A CTA owns a tile of 32 float4 columns; its 8 warps split the rows
// (row j -> warp j % 8, each lane one float4 column, 4 rows unrolled), so
// even 33k-65k-float vectors with ~40 rows keep every SM busy with many
// independent 16-B loads; the 8 fp64 partial float4s of a column meet in
// SMEM and are added in warp order (deterministic).
constexpr int CW = CT / 32;                 // row groups (warps) per CTA

struct CombineJob {
    const float* W;
    int64_t ld;
    double sgn;
    const float* base;
    float* dst;
    int64_t L;
    double* norm_out;
    double* partial;
    unsigned int* ticket;
    int G;                  // CTAs of this job
};

// One or two combinations sharing the coefficients (ctk_iterate's x_k and
// residual): CTAs [0, j0.G) run job 0, the rest job 1.
constexpr int COEF_BYVAL = 160;          // y passed in the kernel parameters up to this k

struct CoefPack {
    double c[COEF_BYVAL];
};

__global__ void __launch_bounds__(CT) k_combine(CombineJob j0, CombineJob j1, int nvec,
                                                const double* __restrict__ coef,
                                                const __grid_constant__ CoefPack cp) {
    extern __shared__ double c[];                                 // [nvec]
    __shared__ double4 red[CW][32];
    __shared__ double nred[CW];
    const bool second = (int)blockIdx.x >= j0.G;
    const CombineJob& J = second ? j1 : j0;
    const int bid = second ? (int)blockIdx.x - j0.G : (int)blockIdx.x;
    const float* __restrict__ W = J.W;
    const int64_t ld = J.ld, L = J.L;
    const float* base = J.base;
    float* dst = J.dst;
    for (int j = threadIdx.x; j < nvec; j += CT) c[j] = J.sgn * (coef ? coef[j] : cp.c[j]);
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t L4 = L >> 2;
    const int64_t ntiles = (L4 + 31) >> 5;
    double nrm = 0.0;
    for (int64_t t = bid; t < ntiles; t += J.G) {
        const int64_t i = (t << 5) + lane;
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
        if (i < L4) {
            const float4* col = reinterpret_cast<const float4*>(W) + i;
            const int64_t ld4 = ld >> 2;
            int j = warp;
            for (; j + 3 * CW < nvec; j += 4 * CW) {
                float4 w[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) w[q] = __ldg(col + (size_t)(j + q * CW) * ld4);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const double cj = c[j + q * CW];
                    a0 = fma(cj, (double)w[q].x, a0); a1 = fma(cj, (double)w[q].y, a1);
                    a2 = fma(cj, (double)w[q].z, a2); a3 = fma(cj, (double)w[q].w, a3);
                }
            }
            for (; j < nvec; j += CW) {
                const float4 w = __ldg(col + (size_t)j * ld4);
                const double cj = c[j];
                a0 = fma(cj, (double)w.x, a0); a1 = fma(cj, (double)w.y, a1);
                a2 = fma(cj, (double)w.z, a2); a3 = fma(cj, (double)w.w, a3);
            }
        }
        red[warp][lane] = make_double4(a0, a1, a2, a3);
        __syncthreads();
        if (warp == 0 && i < L4) {
            if (base) {
                const float4 b = reinterpret_cast<const float4*>(base)[i];
                a0 = b.x; a1 = b.y; a2 = b.z; a3 = b.w;
            } else {
                a0 = a1 = a2 = a3 = 0.0;
            }
#pragma unroll
            for (int w = 0; w < CW; ++w) {
                const double4 p = red[w][lane];
                a0 += p.x; a1 += p.y; a2 += p.z; a3 += p.w;
            }
            const float4 o = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
            reinterpret_cast<float4*>(dst)[i] = o;
            nrm = fma((double)o.x, (double)o.x, nrm); nrm = fma((double)o.y, (double)o.y, nrm);
            nrm = fma((double)o.z, (double)o.z, nrm); nrm = fma((double)o.w, (double)o.w, nrm);
        }
        __syncthreads();
    }
    if (bid == J.G - 1 && warp == 0) {                            // scalar tail L % 4
        for (int64_t i = (L4 << 2) + lane; i < L; i += 32) {
            double a = base ? (double)base[i] : 0.0;
            for (int j = 0; j < nvec; ++j) a = fma(c[j], (double)W[(size_t)j * ld + i], a);
            const float o = (float)a;
            dst[i] = o;
            nrm = fma((double)o, (double)o, nrm);
        }
    }
    if (!J.norm_out) return;
    const double s = warp_sum(nrm);
    if (lane == 0) nred[warp] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < CW; ++w) t += nred[w];
        J.partial[bid] = t;
    }
    last_cta_reduce(J.partial, J.G, 1, J.ticket, J.norm_out, (unsigned)J.G);
}

// ---------------------------------------------------------------------------
// Batched iterate norms (ctk_iterate_batch): for up to IB_NB consecutive
// iterations k_b = k0 + b of one cycle, ||x0 + X y_b||^2 and ||d0 - AX y_b||^2
// in ONE pass over the basis (each X / AX element is read and widened once and
// used for every iterate of the batch, instead of once per iterate), and the
// last iterate of the batch (x and r) stored.  Job 0 (CTAs [0, G0)) is the
// image-space combination, job 1 the residual.  Per element the rows are
// summed in order j = 0, 1, ... from the base (x0 / d0); every CTA's norm
// partials meet in a fixed-order reduction by the job's last CTA.
// ---------------------------------------------------------------------------
constexpr int IB_NB = 8;                 // iterates per batch
constexpr int IB_T = 128;                // threads per CTA
constexpr int IB_MAXK = 512;             // SMEM coefficient table rows

struct IterBatchJob {
    const float* X;
    int64_t ld;
    const float* base;
    float* dst;              // last iterate of the batch (may be null)
    int64_t L;
    double* out;             // out[2 b]: ||.||^2 of iterate b
    double* partial;         // [IB_NB][G]
    unsigned int* ticket;
    int G;
};

template <int V>
struct IbVec;
template <>
struct IbVec<4> {
    __device__ static void load(const float* p, float* v) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
    }
    __device__ static void store(float* p, const float* v) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct IbVec<2> {
    __device__ static void load(const float* p, float* v) {
        const float2 t = __ldg(reinterpret_cast<const float2*>(p));
        v[0] = t.x; v[1] = t.y;
    }
    __device__ static void store(float* p, const float* v) {
        *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
    }
};

// V floats per thread and row, IB_RB rows loaded per batch.
#ifndef CTK_IB_RB
#define CTK_IB_RB 12
#endif
constexpr int IB_RB = CTK_IB_RB;
template <int V>
// Resident CTAs per SM: 4 (128 registers, a few spilled) rather than the 2
// that 174 registers allow -- the pass is bound by bytes in flight.  Measured
// at c4 / c5, k_max = 17 / 37 / 57, % of the HBM peak: 32 / 40 / 46 and
// 38 / 45 / 50 before, 40 / 50 / 54 and 48 / 57 / 59 with 4 CTAs and 12 rows
// of loads in flight per thread (3 CTAs: 37 / 46 / 53 and 45 / 54 / 60).
#ifndef CTK_IB_MINB
#define CTK_IB_MINB 4
#endif
#ifndef CTK_IB_GCAP
#define CTK_IB_GCAP 4
#endif
__global__ void __launch_bounds__(IB_T, CTK_IB_MINB) k_iter_batch(IterBatchJob j0, IterBatchJob j1,
                                                     const double* __restrict__ y, int ystride,
                                                     int k0, int nb) {
    __shared__ __align__(16) double cy[IB_MAXK][IB_NB];   // cy[j][b] = sgn * y_b[j] (0: j >= k_b)
    __shared__ double nred[IB_T / 32][IB_NB];
    __shared__ unsigned int s_last;
    const bool second = (int)blockIdx.x >= j0.G;
    const IterBatchJob& J = second ? j1 : j0;
    const int bid = second ? (int)blockIdx.x - j0.G : (int)blockIdx.x;
    const double sgn = second ? -1.0 : 1.0;
    const int kmax = k0 + nb - 1;
    for (int t = threadIdx.x; t < kmax * IB_NB; t += IB_T) {
        const int j = t / IB_NB, b = t - j * IB_NB;
        cy[j][b] = (b < nb && j < k0 + b) ? sgn * y[(size_t)b * ystride + j] : 0.0;
    }
    __syncthreads();
    const int64_t LV = J.L / V;
    double nrm[IB_NB];
#pragma unroll
    for (int b = 0; b < IB_NB; ++b) nrm[b] = 0.0;
    for (int64_t i = (int64_t)bid * IB_T + threadIdx.x; i < LV; i += (int64_t)J.G * IB_T) {
        double a[IB_NB][V];
        {
            float bv[V];
#pragma unroll
            for (int e = 0; e < V; ++e) bv[e] = 0.f;
            if (J.base) IbVec<V>::load(J.base + i * V, bv);
#pragma unroll
            for (int b = 0; b < IB_NB; ++b)
#pragma unroll
                for (int e = 0; e < V; ++e) a[b][e] = bv[e];
        }
        const float* col = J.X + i * V;
        int j = 0;
        // IB_RB rows' loads in flight per thread: the pass is latency-bound
        // (bytes in flight per SM), not fp64- or conversion-bound
        for (; j + IB_RB <= kmax; j += IB_RB) {
            float w[IB_RB][V];
#pragma unroll
            for (int q = 0; q < IB_RB; ++q) IbVec<V>::load(col + (size_t)(j + q) * J.ld, w[q]);
#pragma unroll
            for (int q = 0; q < IB_RB; ++q) {
                double wd[V];
#pragma unroll
                for (int e = 0; e < V; ++e) wd[e] = w[q][e];
#pragma unroll
                for (int b = 0; b < IB_NB; ++b) {
                    const double c = cy[j + q][b];
#pragma unroll
                    for (int e = 0; e < V; ++e) a[b][e] = fma(c, wd[e], a[b][e]);
                }
            }
        }
        for (; j < kmax; ++j) {
            float w[V];
            IbVec<V>::load(col + (size_t)j * J.ld, w);
            double wd[V];
#pragma unroll
            for (int e = 0; e < V; ++e) wd[e] = w[e];
#pragma unroll
            for (int b = 0; b < IB_NB; ++b) {
                const double c = cy[j][b];
#pragma unroll
                for (int e = 0; e < V; ++e) a[b][e] = fma(c, wd[e], a[b][e]);
            }
        }
#pragma unroll
        for (int b = 0; b < IB_NB; ++b) {
            float o[V];
#pragma unroll
            for (int e = 0; e < V; ++e) o[e] = (float)a[b][e];
            if (b == nb - 1 && J.dst) IbVec<V>::store(J.dst + i * V, o);
#pragma unroll
            for (int e = 0; e < V; ++e) nrm[b] = fma((double)o[e], (double)o[e], nrm[b]);
        }
    }
    if (bid == J.G - 1 && threadIdx.x < 32) {                  // scalar tail L % V
        for (int64_t i = LV * V + threadIdx.x; i < J.L; i += 32) {
            double a[IB_NB];
            const double b0 = J.base ? (double)J.base[i] : 0.0;
#pragma unroll
            for (int b = 0; b < IB_NB; ++b) a[b] = b0;
            for (int j = 0; j < kmax; ++j) {
                const double w = J.X[(size_t)j * J.ld + i];
#pragma unroll
                for (int b = 0; b < IB_NB; ++b) a[b] = fma(cy[j][b], w, a[b]);
            }
#pragma unroll
            for (int b = 0; b < IB_NB; ++b) {
                const float o = (float)a[b];
                if (b == nb - 1 && J.dst) J.dst[i] = o;
                nrm[b] = fma((double)o, (double)o, nrm[b]);
            }
        }
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int b = 0; b < IB_NB; ++b) {
        const double t = warp_sum(nrm[b]);
        if (lane == 0) nred[warp][b] = t;
    }
    __syncthreads();
    if (threadIdx.x < IB_NB) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < IB_T / 32; ++w) t += nred[w][threadIdx.x];
        J.partial[(size_t)threadIdx.x * J.G + bid] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) s_last = ctk_ticket_arrive(J.ticket, (unsigned)J.G);
    __syncthreads();
    if (!s_last) return;
    for (int b = warp; b < nb; b += IB_T / 32) {
        double t = 0.0;
        for (int c = lane; c < J.G; c += 32) t += __ldcg(J.partial + (size_t)b * J.G + c);
        t = warp_sum(t);
        if (lane == 0) J.out[2 * b] = t;
    }
    if (threadIdx.x == 0) *J.ticket = 0u;
}

__global__ void k_scale(const float* __restrict__ v, float* __restrict__ dst, int64_t L,
                        const double* __restrict__ scale) {
    const float sc = (float)(*scale);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < L;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = v[i] * sc;
}

// h = h1 + h2; h[k+1] = sqrt(n2); stat = {||q||, breakdown, 1/h[k+1] or 0, h[k+1]}
__global__ void k_cgs2_finalize(const double* h1, const double* h2, const double* n2, int k,
                                double* h, double* stat) {
    for (int i = threadIdx.x; i <= k; i += blockDim.x) h[i] = h2 ? h1[i] + h2[i] : h1[i];
    if (threadIdx.x == 0) {
        const double hk = sqrt(n2[0]);
        const double qn = sqrt(h1[k + 1]);
        h[k + 1] = hk;
        const bool broke = hk <= 1e-14 * qn;    // BREAKDOWN_RTOL, arnoldi.py:17,80
        stat[0] = qn;
        stat[1] = broke ? 1.0 : 0.0;
        stat[2] = broke ? 0.0 : 1.0 / hk;
        stat[3] = hk;
    }
}

// ---------------------------------------------------------------------------
// Fused CGS2 step for small Krylov vectors (c1/c2: L <= 1M): one cooperative
// launch, one CTA per SM, five grid-wide barriers instead of six launches.
// Each CTA owns a contiguous chunk of L; each warp owns basis rows j = warp
// (mod 8) and reduces them over the chunk, so no CTA-wide barrier is needed
// for the dots.  Block partials are reduced warp-per-row in a fixed order.
// ---------------------------------------------------------------------------
namespace cg = cooperative_groups;

constexpr int FT = 256;                 // fused kernel threads per CTA
constexpr int FW = FT / 32;

__device__ __forceinline__ void chunk_of(int64_t L4, int64_t* i0, int64_t* i1) {
    const int64_t ch = (L4 + gridDim.x - 1) / gridDim.x;
    *i0 = (int64_t)blockIdx.x * ch;
    *i1 = min(L4, *i0 + ch);
}

constexpr int FR = 16;                  // rows per batch: 16 independent 16-B loads

// partial[blk * nv + j] = <row_j, v> over this CTA's chunk (+ scalar tail on
// the last CTA); row nvec is v itself (norm).  Each thread owns float4
// elements of the chunk and streams FR rows at a time (memory-level
// parallelism), then rows are reduced warp -> CTA through smem red[j][warp].
__device__ __forceinline__ void chunk_dots(const float* W, int64_t ld, int nvec, const float* v,
                                           int64_t L, bool norm, double* partial, double* red) {
    const int nv = nvec + (norm ? 1 : 0);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int64_t i0, i1;
    const int64_t L4 = L >> 2;
    chunk_of(L4, &i0, &i1);
    const float4* v4 = reinterpret_cast<const float4*>(v);
    const bool tail = blockIdx.x == gridDim.x - 1;
    for (int j0 = 0; j0 < nv; j0 += FR) {
        double acc[FR];
#pragma unroll
        for (int q = 0; q < FR; ++q) acc[q] = 0.0;
        for (int64_t i = i0 + threadIdx.x; i < i1; i += FT) {
            const float4 vv = v4[i];
            float4 w[FR];
#pragma unroll
            for (int q = 0; q < FR; ++q) {
                const int j = j0 + q;
                if (j < nv) w[q] = __ldg(reinterpret_cast<const float4*>(j < nvec ? W + (size_t)j * ld : v) + i);
            }
#pragma unroll
            for (int q = 0; q < FR; ++q)
                if (j0 + q < nv) acc[q] = dot4(w[q], vv, acc[q]);
        }
        if (tail) {
            for (int64_t i = (L4 << 2) + threadIdx.x; i < L; i += FT) {
                const double vv = (double)v[i];
#pragma unroll
                for (int q = 0; q < FR; ++q) {
                    const int j = j0 + q;
                    if (j < nv) acc[q] = fma((double)(j < nvec ? W[(size_t)j * ld + i] : v[i]), vv, acc[q]);
                }
            }
        }
#pragma unroll
        for (int q = 0; q < FR; ++q) {
            const double t = warp_sum(acc[q]);
            if (lane == 0 && j0 + q < nv) red[(j0 + q) * FW + warp] = t;
        }
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nv; j += FT) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < FW; ++w) t += red[j * FW + w];
        partial[(size_t)blockIdx.x * nv + j] = t;
    }
    __syncthreads();
}

// out[j] = sum over CTAs of partial[b * nv + j], one warp per row (grid-wide).
__device__ __forceinline__ void grid_reduce(const double* partial, int nv, double* out) {
    const int lane = threadIdx.x & 31;
    const int gw = blockIdx.x * FW + (threadIdx.x >> 5);
    for (int j = gw; j < nv; j += gridDim.x * FW) {
        double s = 0.0;
        for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(partial + (size_t)b * nv + j);
        s = warp_sum(s);
        if (lane == 0) out[j] = s;
    }
}

// dst = v - sum_j c[j] W_j over this CTA's chunk; returns this thread's ||dst||^2 part.
__device__ __forceinline__ double chunk_update(const float* W, int64_t ld, int nvec,
                                               const double* c, const float* v, float* dst,
                                               int64_t L) {
    int64_t i0, i1;
    const int64_t L4 = L >> 2;
    chunk_of(L4, &i0, &i1);
    double nrm = 0.0;
    for (int64_t i = i0 + threadIdx.x; i < i1; i += FT) {
        const float4 b = reinterpret_cast<const float4*>(v)[i];
        double a0 = b.x, a1 = b.y, a2 = b.z, a3 = b.w;
        int j = 0;
        for (; j + FR <= nvec; j += FR) {
            float4 w[FR];
#pragma unroll
            for (int q = 0; q < FR; ++q)
                w[q] = __ldg(reinterpret_cast<const float4*>(W + (size_t)(j + q) * ld) + i);
#pragma unroll
            for (int q = 0; q < FR; ++q) {
                const double cj = c[j + q];
                a0 = fma(-cj, (double)w[q].x, a0); a1 = fma(-cj, (double)w[q].y, a1);
                a2 = fma(-cj, (double)w[q].z, a2); a3 = fma(-cj, (double)w[q].w, a3);
            }
        }
        for (; j < nvec; ++j) {
            const float4 w = __ldg(reinterpret_cast<const float4*>(W + (size_t)j * ld) + i);
            const double cj = c[j];
            a0 = fma(-cj, (double)w.x, a0); a1 = fma(-cj, (double)w.y, a1);
            a2 = fma(-cj, (double)w.z, a2); a3 = fma(-cj, (double)w.w, a3);
        }
        const float4 o = make_float4((float)a0, (float)a1, (float)a2, (float)a3);
        reinterpret_cast<float4*>(dst)[i] = o;
        nrm = fma((double)o.x, (double)o.x, nrm); nrm = fma((double)o.y, (double)o.y, nrm);
        nrm = fma((double)o.z, (double)o.z, nrm); nrm = fma((double)o.w, (double)o.w, nrm);
    }
    if (blockIdx.x == gridDim.x - 1) {
        for (int64_t i = (L4 << 2) + threadIdx.x; i < L; i += FT) {
            double a = (double)v[i];
            for (int j = 0; j < nvec; ++j) a = fma(-c[j], (double)W[(size_t)j * ld + i], a);
            const float o = (float)a;
            dst[i] = o;
            nrm = fma((double)o, (double)o, nrm);
        }
    }
    return nrm;
}

__global__ void __launch_bounds__(FT) k_cgs2_fused(float* W, int64_t ld, int k, int64_t L,
                                                   float* q, double* h, double* stat,
                                                   double* partial, double* red) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sh_c[];                 // [k+1] coefficients, then red
    double* red_s = sh_c + (k + 1);                  // [(k+2) * FW] per-warp row sums
    __shared__ double s_red[FW];
    const int nb = k + 1;
    double* h1 = red;                                // [nb + 1]: h1, ||q||^2
    double* h2 = red + (nb + 1);                     // [nb]
    double* n2 = red + (2 * nb + 1);                 // [1]
    float* wnext = W + (size_t)(k + 1) * ld;

    chunk_dots(W, ld, nb, q, L, true, partial, red_s);   // h1 = W^T q, ||q||^2
    grid.sync();
    grid_reduce(partial, nb + 1, h1);
    grid.sync();
    for (int j = threadIdx.x; j < nb; j += FT) sh_c[j] = h1[j];
    __syncthreads();
    chunk_update(W, ld, nb, sh_c, q, q, L);          // q1 = q - W h1 (in place, own chunk)
    __syncthreads();
    chunk_dots(W, ld, nb, q, L, false, partial, red_s);  // h2 = W^T q1
    grid.sync();
    grid_reduce(partial, nb, h2);
    grid.sync();
    for (int j = threadIdx.x; j < nb; j += FT) sh_c[j] = h2[j];
    __syncthreads();
    double nrm = chunk_update(W, ld, nb, sh_c, q, wnext, L);   // q2 -> row k+1
    nrm = warp_sum(nrm);
    if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = nrm;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < FW; ++w) t += s_red[w];
        partial[blockIdx.x] = t;
    }
    grid.sync();
    if (blockIdx.x == 0) {
        grid_reduce(partial, 1, n2);                 // one warp: fixed order over CTAs
        __syncthreads();
        for (int i = threadIdx.x; i <= k; i += FT) h[i] = h1[i] + h2[i];
        if (threadIdx.x == 0) {
            const double hk = sqrt(n2[0]);
            const double qn = sqrt(h1[nb]);
            h[k + 1] = hk;
            const bool broke = hk <= 1e-14 * qn;    // BREAKDOWN_RTOL, arnoldi.py:17,80
            stat[0] = qn;
            stat[1] = broke ? 1.0 : 0.0;
            stat[2] = broke ? 0.0 : 1.0 / hk;
            stat[3] = hk;
        }
    }
    grid.sync();
    const float sc = (float)__ldcg(stat + 2);
    int64_t i0, i1;
    chunk_of(L >> 2, &i0, &i1);
    for (int64_t i = i0 + threadIdx.x; i < i1; i += FT) {
        float4 v = reinterpret_cast<float4*>(wnext)[i];
        v.x *= sc; v.y *= sc; v.z *= sc; v.w *= sc;
        reinterpret_cast<float4*>(wnext)[i] = v;
    }
    if (blockIdx.x == gridDim.x - 1)
        for (int64_t i = ((L >> 2) << 2) + threadIdx.x; i < L; i += FT) wnext[i] *= sc;
}

constexpr int64_t FUSED_MAX_L = 1 << 21;

// ---------------------------------------------------------------------------
// SMEM-resident Gram-Schmidt step (c1/c2 sizes: the whole basis fits in the
// aggregate shared memory of the 148 SMs, e.g. 81 x 65536 fp32 = 21 MB).
// One cooperative launch, one CTA per SM.  Each CTA pulls its L-chunk of all
// k+1 basis rows into shared memory with bulk async copies (TMA engine, one
// mbarrier, no register staging), so both Gram-Schmidt passes, the norm and
// the scale run out of SMEM: the basis is read from L2/HBM once per step
// instead of four times, and there are 3 grid barriers instead of 5.  Chunk
// partials are stored row-major [row][cta]; after each barrier EVERY CTA
// reduces all rows in the same fixed order (lane-strided over CTAs, then a
// fixed shuffle tree), so the coefficients are bitwise identical across CTAs
// and run to run without a second barrier.
// ---------------------------------------------------------------------------
constexpr int ST = 512;                 // threads per CTA
constexpr int SW = ST / 32;
constexpr size_t SMEM_LIMIT = 224 * 1024;       // + static smem (<= 3 KB) <= 227 KB opt-in

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
        "r"(phase)
        : "memory");
}

// partial[j * G + b] = <Ws[j], v> over this CTA's chunk (row vrow is v
// itself: pass vrow = nrows - 1 to fold ||v||^2 in).  vd is v widened to fp64
// once (SMEM), so only the basis elements go through the conversion pipe.
// Up to four rows per warp are in flight at once (independent fp64
// accumulators); the warp's row count is exact (no clamped duplicate rows).
constexpr int GS_DR = 4;

template <int NR>
__device__ __forceinline__ void smem_dots_rows(const float* Ws, int cpad, int j0, int vrow,
                                               const float* v, const double* vd, int cn,
                                               double* partial) {
    const int lane = threadIdx.x & 31;
    const int cn4 = cn >> 2;
    const double2* vd2 = reinterpret_cast<const double2*>(vd);
    const float* row[NR];
    double s[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int j = j0 + r * SW;
        row[r] = j == vrow ? v : Ws + (size_t)j * cpad;
        s[r] = 0.0;
    }
    for (int i = lane; i < cn4; i += 32) {
        const double2 a = vd2[2 * i], b = vd2[2 * i + 1];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const float4 w = reinterpret_cast<const float4*>(row[r])[i];
            s[r] = fma((double)w.x, a.x, s[r]);
            s[r] = fma((double)w.y, a.y, s[r]);
            s[r] = fma((double)w.z, b.x, s[r]);
            s[r] = fma((double)w.w, b.y, s[r]);
        }
    }
    for (int i = (cn4 << 2) + lane; i < cn; i += 32)
#pragma unroll
        for (int r = 0; r < NR; ++r) s[r] = fma((double)row[r][i], vd[i], s[r]);
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const double t = warp_sum(s[r]);
        if (lane == 0) partial[(size_t)(j0 + r * SW) * gridDim.x + blockIdx.x] = t;
    }
}

__device__ __forceinline__ void smem_dots(const float* Ws, int cpad, int nrows, int vrow,
                                          const float* v, const double* vd, int cn,
                                          double* partial) {
    const int warp = threadIdx.x >> 5;
    for (int j0 = warp; j0 < nrows; j0 += SW * GS_DR) {
        const int nr = (nrows - j0 + SW - 1) / SW;      // rows j0, j0 + SW, ... below nrows
        if (nr >= 4) smem_dots_rows<4>(Ws, cpad, j0, vrow, v, vd, cn, partial);
        else if (nr == 3) smem_dots_rows<3>(Ws, cpad, j0, vrow, v, vd, cn, partial);
        else if (nr == 2) smem_dots_rows<2>(Ws, cpad, j0, vrow, v, vd, cn, partial);
        else smem_dots_rows<1>(Ws, cpad, j0, vrow, v, vd, cn, partial);
    }
}

// Gram variant (one pass over the chunk): partial rows 0..nb-1 = <W_j, q>,
// row nb = ||q||^2, rows nb+1+j = <W_j, w_k> (k = nb - 1, the newest row,
// widened once into wd).
template <int NR>
__device__ __forceinline__ void smem_dots2_rows(const float* Ws, int cpad, int j0, int nb,
                                                const float* v, const double* vd,
                                                const double* wd, int cn, double* partial) {
    const int lane = threadIdx.x & 31;
    const int cn4 = cn >> 2;
    const double2* vd2 = reinterpret_cast<const double2*>(vd);
    const double2* wd2 = reinterpret_cast<const double2*>(wd);
    const float* row[NR];
    double s[NR], g[NR];
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int j = j0 + r * SW;
        row[r] = j == nb ? v : Ws + (size_t)j * cpad;
        s[r] = 0.0;
        g[r] = 0.0;
    }
    for (int i = lane; i < cn4; i += 32) {
        const double2 a = vd2[2 * i], b = vd2[2 * i + 1];
        const double2 c = wd2[2 * i], d = wd2[2 * i + 1];
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const float4 w = reinterpret_cast<const float4*>(row[r])[i];
            const double x0 = w.x, x1 = w.y, x2 = w.z, x3 = w.w;
            s[r] = fma(x0, a.x, s[r]);
            s[r] = fma(x1, a.y, s[r]);
            s[r] = fma(x2, b.x, s[r]);
            s[r] = fma(x3, b.y, s[r]);
            g[r] = fma(x0, c.x, g[r]);
            g[r] = fma(x1, c.y, g[r]);
            g[r] = fma(x2, d.x, g[r]);
            g[r] = fma(x3, d.y, g[r]);
        }
    }
    for (int i = (cn4 << 2) + lane; i < cn; i += 32)
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const double x = (double)row[r][i];
            s[r] = fma(x, vd[i], s[r]);
            g[r] = fma(x, wd[i], g[r]);
        }
#pragma unroll
    for (int r = 0; r < NR; ++r) {
        const int j = j0 + r * SW;
        const double t = warp_sum(s[r]);
        const double u = warp_sum(g[r]);
        if (lane == 0) {
            partial[(size_t)j * gridDim.x + blockIdx.x] = t;
            if (j < nb) partial[(size_t)(nb + 1 + j) * gridDim.x + blockIdx.x] = u;
        }
    }
}

__device__ __forceinline__ void smem_dots2(const float* Ws, int cpad, int nb, const float* v,
                                           const double* vd, const double* wd, int cn,
                                           double* partial) {
    const int warp = threadIdx.x >> 5;
    const int nrows = nb + 1;
    for (int j0 = warp; j0 < nrows; j0 += SW * GS_DR) {
        const int nr = (nrows - j0 + SW - 1) / SW;
        if (nr >= 4) smem_dots2_rows<4>(Ws, cpad, j0, nb, v, vd, wd, cn, partial);
        else if (nr == 3) smem_dots2_rows<3>(Ws, cpad, j0, nb, v, vd, wd, cn, partial);
        else if (nr == 2) smem_dots2_rows<2>(Ws, cpad, j0, nb, v, vd, wd, cn, partial);
        else smem_dots2_rows<1>(Ws, cpad, j0, nb, v, vd, wd, cn, partial);
    }
}

// coef[j] = sum over CTAs of partial[j * G + b], identical in every CTA.
// All loads of a warp's rows are issued before any add (one L2 round trip
// instead of one per row x CTA group); per-lane order then a fixed shuffle
// tree, so the result does not depend on which CTA computes it.
constexpr int GS_MAXG = 160;            // <= 5 partials per lane
constexpr int GS_RU = 6;                // rows per warp in flight

__device__ __forceinline__ void all_reduce_rows(const double* partial, int nrows, double* coef) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int G = gridDim.x;
    for (int j0 = warp; j0 < nrows; j0 += SW * GS_RU) {
        double v[GS_RU][GS_MAXG / 32];
#pragma unroll
        for (int r = 0; r < GS_RU; ++r) {
            const int j = j0 + r * SW;
#pragma unroll
            for (int t = 0; t < GS_MAXG / 32; ++t) {
                const int b = lane + 32 * t;
                v[r][t] = (j < nrows && b < G) ? __ldcg(partial + (size_t)j * G + b) : 0.0;
            }
        }
#pragma unroll
        for (int r = 0; r < GS_RU; ++r) {
            double s = v[r][0];
#pragma unroll
            for (int t = 1; t < GS_MAXG / 32; ++t) s += v[r][t];
            s = warp_sum(s);
            const int j = j0 + r * SW;
            if (lane == 0 && j < nrows) coef[j] = s;
        }
    }
}

// Gram-corrected CGS2 (one reduction per step instead of two or three).
// CGS2's second pass computes h2 = W^T (q - W h1) = h1 - (W^T W) h1 = -E h1,
// E = W^T W - I, so with E at hand the reorthogonalisation needs no second
// sweep over the basis: c = h1 + h2 = h1 - E h1 and q2 = q - W c in one
// update, with one rounding to fp32 instead of two (q1 is never stored).  E
// is the Gram matrix of the STORED fp32 rows (entries ~ fp32 rounding), one
// new column per step: <w_i, w_k> comes out of the same sweep as W^T q (row
// k is in the tile), so it costs no extra traffic.  This is DCGS2-style
// delayed reorthogonalisation (low-synchronisation Gram-Schmidt); it equals
// CGS2 -- and the reference's MGS + reorth (ctkrylov/arnoldi.py:66-82) -- in
// exact arithmetic.  ||q2||^2 follows from the reduced values,
//   est = ||q||^2 - 2 c.h1 + c.c + c.(E c),
// so 1/||q2|| is known before q2 is formed and the update writes the
// normalised row directly (no norm reduction, no scale pass); when est <=
// 1e-8 ||q||^2 (cancellation would cost fp64 digits) the kernels fall back to
// an explicit fp64 norm of the stored q2.
//
// Per-CTA (every CTA computes the same values in the same order, so the
// fallback decision below is grid-uniform): h2[i] = -(E h1)_i,
// cc[i] = h1[i] + h2[i], *est; CTA 0 appends E's column / row k to `gram`.
// E[i][j] with i, j < k was written by step max(i, j) < k; row and column k
// come from this step's g (E[k][j] = E[j][k] = g[j], E[k][k] = g[k] - 1).
// `Es` (row stride es_ld): the i, j < k block, in shared memory when the
// caller staged it (es_smem), else `gram` itself.
// E's entries are fp32-rounding sized (~1e-7), so E h1 and E c are formed in
// fp32: each product keeps ~7 significant digits of a term 1e-7 |h1| small,
// i.e. ~1e-14 |h1| absolute -- far below what c needs -- and the passes run
// on the fp32 pipe with no fp64 conversions (the dots, c.h1 and c.c that
// cancel stay in fp64).
__device__ __forceinline__ float gram_entry(const float* Es, int es_ld, bool es_smem, int i, int j,
                                            int k, const float* gf) {
    if (j == k) return gf[i];
    if (i == k) return gf[j];
    const float* p = Es + (size_t)i * es_ld + j;
    return es_smem ? *p : __ldcg(p);
}

template <bool ES_SMEM>
__device__ void gram_coefs(float* gram, const float* Es, int es_ld, int k,
                           const double* h1, const double* g, double* h2, double* cc,
                           double* red, double* s_est) {
    // four threads per row (nb <= 128 rows on 512 threads): each sums a
    // quarter of the row in fp32, two shuffles finish it.  Fixed order:
    // bitwise the same in every CTA.
    constexpr int TPR = 4;
    __shared__ float s_f[3][GRAM_LD];                 // h1, column k of E, c (fp32)
    const int nb = k + 1, lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    float* h1f = s_f[0];
    float* gf = s_f[1];
    float* cf = s_f[2];
    for (int r = threadIdx.x; r < nb; r += blockDim.x) {
        h1f[r] = (float)h1[r];
        gf[r] = (float)(g[r] - (r == k ? 1.0 : 0.0));
    }
    __syncthreads();
    const int i = threadIdx.x / TPR, sub = threadIdx.x % TPR;
    // E in global memory (streamed path): this thread's <= GRAM_LD / TPR
    // entries of row i go to registers with all loads issued before the first
    // use -- one L2 round trip for both products instead of one per entry
    // (4-9 -> 2-3 us per step; same summation order as the shared-memory
    // loop, j = sub, sub + TPR, ...)
    constexpr int EMAX = GRAM_LD / TPR;
    float er[ES_SMEM ? 1 : EMAX];
    if (!ES_SMEM) {
#pragma unroll
        for (int q = 0; q < EMAX; ++q) {
            const int j = sub + q * TPR;
            er[q] = (i < nb && j < nb) ? gram_entry(Es, es_ld, false, i, j, k, gf) : 0.f;
        }
    }
    float t = 0.f;
    if (ES_SMEM) {
        if (i < nb)
            for (int j = sub; j < nb; j += TPR)
                t = fmaf(gram_entry(Es, es_ld, true, i, j, k, gf), h1f[j], t);
    } else if (i < nb) {
#pragma unroll
        for (int q = 0; q < EMAX; ++q) {
            const int j = sub + q * TPR;
            if (j < nb) t = fmaf(er[q], h1f[j], t);
        }
    }
    t += __shfl_xor_sync(0xffffffffu, t, 1);
    t += __shfl_xor_sync(0xffffffffu, t, 2);
    if (i < nb && sub == 0) {
        h2[i] = -(double)t;
        cc[i] = h1[i] - (double)t;
        cf[i] = (float)cc[i];
    }
    if (blockIdx.x == 0)
        for (int r = threadIdx.x; r <= k; r += blockDim.x) {
            gram[(size_t)k * GRAM_LD + r] = gf[r];
            gram[(size_t)r * GRAM_LD + k] = gf[r];
        }
    __syncthreads();
    float u = 0.f;
    if (ES_SMEM) {
        if (i < nb)
            for (int j = sub; j < nb; j += TPR)
                u = fmaf(gram_entry(Es, es_ld, true, i, j, k, gf), cf[j], u);
    } else if (i < nb) {
#pragma unroll
        for (int q = 0; q < EMAX; ++q) {
            const int j = sub + q * TPR;
            if (j < nb) u = fmaf(er[q], cf[j], u);
        }
    }
    u += __shfl_xor_sync(0xffffffffu, u, 1);
    u += __shfl_xor_sync(0xffffffffu, u, 2);
    // this row's share of  c.(E c) + c.c - 2 c.h1  (the last two in fp64)
    double part = (i < nb && sub == 0) ? cc[i] * (double)u + cc[i] * cc[i] - 2.0 * cc[i] * h1[i] : 0.0;
    part = warp_sum(part);
    if (lane == 0) red[warp] = part;
    __syncthreads();
    if (threadIdx.x == 0) {
        double tt = 0.0;
        for (int w = 0; w < nw; ++w) tt += red[w];
        *s_est = h1[nb] + tt;
    }
    __syncthreads();
}

// v <- v - sum_j c[j] Ws[j] over the chunk (fp64 accumulate, fp32 result);
// returns this thread's part of ||v||^2 (of the rounded values).  The chunk
// has fewer float4 than the CTA has threads, so the rows are split over
// ngrp = ST / cn4 thread groups (row j -> group j % ngrp) whose fp64 partial
// sums meet in SMEM (acc[g][i]) and are added in group order.
__device__ __forceinline__ double smem_update(const float* Ws, int cpad, int nb, const double* c,
                                              float* v, double* vd, int cn, double4* acc,
                                              double scale = 1.0) {
    const int cn4 = cn >> 2;
    int ngrp = cn4 > 0 ? ST / cn4 : 1;
    ngrp = ngrp < 1 ? 1 : (ngrp > 8 ? 8 : ngrp);
    if (cn4 > ST / 2) {          // wide chunk: one thread per float4, all rows
        double nrm = 0.0;
        for (int t = threadIdx.x; t < cn4; t += ST) {
            const float4 b = reinterpret_cast<const float4*>(v)[t];
            double a0 = b.x, a1 = b.y, a2 = b.z, a3 = b.w;
#pragma unroll 4
            for (int j = 0; j < nb; ++j) {
                const float4 w = reinterpret_cast<const float4*>(Ws + (size_t)j * cpad)[t];
                const double cj = c[j];
                a0 = fma(-cj, (double)w.x, a0); a1 = fma(-cj, (double)w.y, a1);
                a2 = fma(-cj, (double)w.z, a2); a3 = fma(-cj, (double)w.w, a3);
            }
            const float4 o = make_float4((float)(a0 * scale), (float)(a1 * scale),
                                         (float)(a2 * scale), (float)(a3 * scale));
            reinterpret_cast<float4*>(v)[t] = o;
            const double4 od = make_double4(o.x, o.y, o.z, o.w);
            if (vd) {
                reinterpret_cast<double2*>(vd)[2 * t] = make_double2(od.x, od.y);
                reinterpret_cast<double2*>(vd)[2 * t + 1] = make_double2(od.z, od.w);
            }
            nrm = fma(od.x, od.x, nrm); nrm = fma(od.y, od.y, nrm);
            nrm = fma(od.z, od.z, nrm); nrm = fma(od.w, od.w, nrm);
        }
        for (int t = (cn4 << 2) + threadIdx.x; t < cn; t += ST) {
            double a = (double)v[t];
            for (int j = 0; j < nb; ++j) a = fma(-c[j], (double)Ws[(size_t)j * cpad + t], a);
            const float o = (float)(a * scale);
            v[t] = o;
            if (vd) vd[t] = (double)o;
            nrm = fma((double)o, (double)o, nrm);
        }
        return nrm;
    }
    const int g = threadIdx.x / (cn4 > 0 ? cn4 : 1);
    const int i = threadIdx.x - g * cn4;
    if (g < ngrp && i < cn4) {
        double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll 4
        for (int j = g; j < nb; j += ngrp) {
            const float4 w = reinterpret_cast<const float4*>(Ws + (size_t)j * cpad)[i];
            const double cj = c[j];
            a0 = fma(-cj, (double)w.x, a0); a1 = fma(-cj, (double)w.y, a1);
            a2 = fma(-cj, (double)w.z, a2); a3 = fma(-cj, (double)w.w, a3);
        }
        acc[g * cn4 + i] = make_double4(a0, a1, a2, a3);
    }
    __syncthreads();
    double nrm = 0.0;
    for (int t = threadIdx.x; t < cn4; t += ST) {
        const float4 b = reinterpret_cast<const float4*>(v)[t];
        double a0 = b.x, a1 = b.y, a2 = b.z, a3 = b.w;
        for (int q = 0; q < ngrp; ++q) {
            const double4 p = acc[q * cn4 + t];
            a0 += p.x; a1 += p.y; a2 += p.z; a3 += p.w;
        }
        const float4 o = make_float4((float)(a0 * scale), (float)(a1 * scale),
                                     (float)(a2 * scale), (float)(a3 * scale));
        reinterpret_cast<float4*>(v)[t] = o;
        const double4 od = make_double4(o.x, o.y, o.z, o.w);
        if (vd) {
            reinterpret_cast<double2*>(vd)[2 * t] = make_double2(od.x, od.y);
            reinterpret_cast<double2*>(vd)[2 * t + 1] = make_double2(od.z, od.w);
        }
        nrm = fma(od.x, od.x, nrm); nrm = fma(od.y, od.y, nrm);
        nrm = fma(od.z, od.z, nrm); nrm = fma(od.w, od.w, nrm);
    }
    for (int t = (cn4 << 2) + threadIdx.x; t < cn; t += ST) {
        double a = (double)v[t];
        for (int j = 0; j < nb; ++j) a = fma(-c[j], (double)Ws[(size_t)j * cpad + t], a);
        const float o = (float)(a * scale);
        v[t] = o;
        if (vd) vd[t] = (double)o;
        nrm = fma((double)o, (double)o, nrm);
    }
    return nrm;
}

// tm (when use_tma): 3-D tensor map over the basis rows as 64-float panels,
// dims {64, panels, k+1}; one box {64, chunk / 64, k+1} is this CTA's whole
// [k+1][chunk] block -- one TMA copy instead of k+1 row copies.
#ifdef CTK_GS_PROF
__device__ unsigned long long g_gs_prof[160 * 16];
#define GS_STAMP(i) do { if (threadIdx.x == 0) { unsigned long long t_; \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_)); g_gs_prof[blockIdx.x * 16 + (i)] = t_; } } while (0)
extern "C" int ctk_gs_prof_read(unsigned long long* out) {
    return cudaMemcpyFromSymbol(out, g_gs_prof, sizeof(g_gs_prof)) == cudaSuccess ? 0 : -1;
}
#else
#define GS_STAMP(i) do {} while (0)
#endif

__global__ void __launch_bounds__(ST, 1) k_gs_smem(float* W, int64_t ld, int k, int64_t L,
                                                   const float* __restrict__ q, int passes,
                                                   int64_t chunk, double* h, double* stat,
                                                   double* partial, ctk_stage_dst sd,
                                                   double* hm, int stat_off, int use_tma,
                                                   float* gram,
                                                   const __grid_constant__ CUtensorMap tm) {
    cg::grid_group grid = cg::this_grid();
    GS_STAMP(0);
    ctk_pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    const int nb = k + 1;
    const int cpad = (int)((chunk + 3) & ~3LL);
    const int64_t start = (int64_t)blockIdx.x * chunk;
    const int64_t rem = L - start;
    const int cn = rem <= 0 ? 0 : (int)(rem < chunk ? rem : chunk);
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem_raw);
    double* h1 = reinterpret_cast<double*>(smem_raw + 16);          // [2 nb + 2]: h1, ||q||^2, g
    double* h2 = h1 + (2 * nb + 2);                                 // [nb + 1]: h2, ||q1||^2
    double* cc = h2 + nb + 1;                                       // [nb + 1]: h1 + h2 (gram)
    double* red = cc + nb + 1;                                      // [SW]
    float* qv = reinterpret_cast<float*>(
        smem_raw + ((16 + sizeof(double) * (4 * nb + 4 + SW) + 15) & ~(size_t)15));
    double* qd = reinterpret_cast<double*>(qv + cpad);               // [cpad]: qv in fp64
    double* wkd = qd + cpad;                                         // [cpad]: row k in fp64 (gram)
    float* Es = reinterpret_cast<float*>(wkd + cpad);                // [k][k]: E block (gram)
    const int es_n = gram && passes == 2 ? k : 0;
    unsigned char* ws_raw = reinterpret_cast<unsigned char*>(Es + ((es_n * es_n + 3) & ~3));
    ws_raw += (128u - (smem_u32(ws_raw) & 127u)) & 127u;           // TMA destination alignment
    float* Ws = reinterpret_cast<float*>(ws_raw);                   // [nb][cpad]
    double4* acc = reinterpret_cast<double4*>(                      // [ST], 32-B aligned
        (reinterpret_cast<uintptr_t>(Ws + (size_t)nb * cpad) + 31) & ~(uintptr_t)31);
    const unsigned bar_a = smem_u32(bar);
    const unsigned row_bytes = (unsigned)(((cn + 3) & ~3) * 4);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_a) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    ctk_pdl_wait();
    GS_STAMP(1);                     // q (and, transitively, the basis) from the previous kernels
    if (use_tma) {
        if (threadIdx.x == 0 && row_bytes > 0) {
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                         "r"((unsigned)(cpad * 4) * (unsigned)nb)
                         : "memory");
            asm volatile(
                "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(Ws)),
                "l"(reinterpret_cast<uint64_t>(&tm)), "r"(0), "r"((int)(start / 64)), "r"(0),
                "r"(bar_a)
                : "memory");
        }
    } else if (threadIdx.x < 32 && row_bytes > 0) {
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a),
                         "r"(row_bytes * (unsigned)nb)
                         : "memory");
        __syncwarp();
        for (int j = threadIdx.x; j < nb; j += 32)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
                "[%3];" ::"r"(smem_u32(Ws + (size_t)j * cpad)),
                "l"(W + (size_t)j * ld + start), "r"(row_bytes), "r"(bar_a)
                : "memory");
    }
    for (int i = threadIdx.x; i < cn; i += ST) {                     // (16-B alignment of q
        const float v = q[start + i];
        qv[i] = v;
        qd[i] = v;
    }                                                                //  not assumed here)
    for (int e = threadIdx.x; e < es_n * es_n; e += ST) {            // E's i, j < k block
        const int i = e / es_n, j = e - i * es_n;                    // (written by earlier steps)
        Es[e] = __ldcg(gram + (size_t)i * GRAM_LD + j);
    }
    if (row_bytes > 0) mbar_wait(bar_a, 0);
    __syncthreads();
    GS_STAMP(2);

    double* P1 = partial;                                    // [nb + 1][G] (gram: [2 nb + 1][G])
    double* P2 = P1 + (size_t)(nb + 1) * gridDim.x;          // [nb + 1][G]
    double* P3 = P2 + (size_t)(nb + 1) * gridDim.x;          // [G]
    __shared__ double s_n2;
    bool need_norm = true, prescaled = false, staged = false;
    double nrm = 0.0;
    if (gram && passes == 2) {
        // Gram-corrected CGS2 (see gram_coefs): one sweep, one reduction
        for (int i = threadIdx.x; i < cn; i += ST) wkd[i] = (double)Ws[(size_t)k * cpad + i];
        __syncthreads();
        smem_dots2(Ws, cpad, nb, qv, qd, wkd, cn, P1);    // h1, ||q||^2, <W_j, w_k>
        GS_STAMP(3);
        grid.sync();
        GS_STAMP(4);
        all_reduce_rows(P1, 2 * nb + 1, h1);
        __syncthreads();
        GS_STAMP(6);
        __shared__ double s_est;
        gram_coefs<true>(gram, Es, es_n, k, h1, h1 + nb + 1, h2, cc, red, &s_est);
        GS_STAMP(5);
        const double est = s_est, a = h1[nb];
        if (a > 0.0 && est > 1e-8 * a) {
            nrm = smem_update(Ws, cpad, nb, cc, qv, nullptr, cn, acc, 1.0 / sqrt(est));
            if (threadIdx.x == 0) s_n2 = est;
            need_norm = false;
            prescaled = true;
        } else {
            nrm = smem_update(Ws, cpad, nb, cc, qv, nullptr, cn, acc);
        }
        GS_STAMP(10);
    } else {
    smem_dots(Ws, cpad, nb + 1, nb, qv, qd, cn, P1);             // h1 = W^T q, ||q||^2
    GS_STAMP(3);
    grid.sync();
    GS_STAMP(4);
    all_reduce_rows(P1, nb + 1, h1);
    __syncthreads();
    GS_STAMP(5);
    nrm = smem_update(Ws, cpad, nb, h1, qv, qd, cn, acc);      // q1 = q - W h1
    GS_STAMP(6);
    if (passes == 2) {
        __syncthreads();
        smem_dots(Ws, cpad, nb + 1, nb, qv, qd, cn, P2);         // h2 = W^T q1, ||q1||^2
        GS_STAMP(7);
        grid.sync();
        GS_STAMP(8);
        all_reduce_rows(P2, nb + 1, h2);
        __syncthreads();
        GS_STAMP(9);
        nrm = smem_update(Ws, cpad, nb, h2, qv, nullptr, cn, acc);         // q2 = q1 - W h2
        GS_STAMP(10);
        // ||q2||^2 = ||q1||^2 - ||h2||^2 for orthonormal W: after the first pass
        // h2 is at rounding level, so there is no cancellation and the third
        // grid-wide reduction is skipped.  Every CTA holds the same h2, so the
        // (never expected) fallback branch below is grid-uniform.
        double t = 0.0;
        for (int j = 0; j < nb; ++j) t = fma(h2[j], h2[j], t);
        if (h2[nb] > 0.0 && t <= 0.25 * h2[nb]) {
            if (threadIdx.x == 0) s_n2 = h2[nb] - t;
            need_norm = false;
        }
    }
    }
    if (need_norm) {
        nrm = warp_sum(nrm);
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = nrm;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < SW; ++w) t += red[w];
            P3[blockIdx.x] = t;
        }
        grid.sync();
        if (threadIdx.x < 32) all_reduce_rows(P3, 1, &s_n2);
    }
    __syncthreads();
    const double hk = sqrt(s_n2);
    const double qn = sqrt(h1[nb]);
    const bool broke = hk <= 1e-14 * qn;                     // BREAKDOWN_RTOL, arnoldi.py:17,80
    const float sc = broke ? 0.f : prescaled ? 1.f : (float)(1.0 / hk);
    float* wnext = W + (size_t)(k + 1) * ld + start;
    if (sd.P) {     // also stage w_{k+1} for the next K1 apply (zero-padded P and PT)
        const int pP = sd.nx + 2 * sd.pad, pT = sd.ny + 2 * sd.pad;
        for (int i = threadIdx.x; i < cn; i += ST) {
            const float v = qv[i] * sc;
            wnext[i] = v;
            const int e = (int)(start + i);
            const int iy = e / sd.nx, ix = e - iy * sd.nx;
            sd.P[(size_t)iy * pP + ix + sd.pad] = v;
            sd.PT[(size_t)ix * pT + iy + sd.pad] = v;
        }
    } else {
        for (int i = threadIdx.x; i < cn; i += ST) wnext[i] = qv[i] * sc;
    }
    if (blockIdx.x == 0) {
        // hm: optional host-mapped (page-locked) mirror of the column, written
        // here instead of a D2H copy on the Arnoldi stream.
        for (int i = threadIdx.x; i <= k; i += ST) {
            const double v = passes == 2 ? h1[i] + h2[i] : h1[i];
            h[i] = v;
            if (hm) hm[i] = v;
        }
        if (threadIdx.x == 0) {
            const double st4[4] = {qn, broke ? 1.0 : 0.0, broke ? 0.0 : 1.0 / hk, hk};
            h[k + 1] = hk;
            for (int q = 0; q < 4; ++q) stat[q] = st4[q];
            if (hm) {
                hm[k + 1] = hk;
                for (int q = 0; q < 4; ++q) hm[stat_off + q] = st4[q];
            }
        }
    }
    GS_STAMP(11);
}

// ---------------------------------------------------------------------------
// Streamed Gram-Schmidt step for Krylov vectors too long for the SMEM-resident
// path (c4: L = 2.1M, c5: L = 4.2M).  One cooperative CTA per SM owns a
// contiguous run of TW-float tiles; every sweep streams the k+1 basis rows
// and one vector of its tiles through a double-buffered shared-memory ring
// filled by bulk async copies (one mbarrier per buffer, issued by warp 0), so
// the basis is read from HBM once per sweep with a whole tile in flight while
// the other is consumed:
//   A: h1 = W^T q, ||q||^2                                   | grid barrier
//   B: q1 = q - W h1 -> row k+1; h2 = W^T q1 (q1 from SMEM)  | grid barrier  (passes == 2)
//   C: q2 = q1 - W h2 -> row k+1, ||q2||^2                   | grid barrier
//   scale row k+1 by 1/||q2|| (+ the K1 staged copies, host-mapped column)
// Three reads of the basis instead of the register-streamed kernel's four,
// and the input q is never written (AB keeps A B w_j without a copy).
// Every CTA reduces the chunk partials in the same fixed order.
// ---------------------------------------------------------------------------
constexpr int TS_RPW = 8;                        // dot rows per warp: 16 warps x 8 = 128
constexpr int TS_MAXROWS = SW * TS_RPW;          // basis rows + the vector row
// Ring depth: 4 slots of 256-float tiles while they fit beside the reduction
// scratch (k <= ~48), else 2 -- a compile-time choice per instantiation: the
// slot / phase arithmetic (g % NBUF, g / NBUF) sits on every tile's critical
// path, and with a run-time depth its divisions cost what the deeper ring
// gains (the sweeps are bound by the per-warp instruction stream, DESIGN 9.2).
constexpr int TS_MAXBUF = 4;

// Ring slot b: buffer ring + b (rows) tw floats, mbarrier bar0 + 8 b.
struct TsRing {
    float* ring;
    unsigned bar0;
    int stride;                                  // floats per slot: (nb + 1) * tw
    __device__ float* buf(int b) const { return ring + (size_t)b * stride; }
    __device__ unsigned bar(int b) const { return bar0 + 8u * (unsigned)b; }
};

// Queue tile e0 into ring slot b: thread 0 (part 0) the basis rows 0..nb-1
// (one 2-D tensor box of tw x nb floats), thread 32 (part 1) the same tile of
// the vector (a tw x 1 box, row nb of the slot).  Each issuer arrives on the
// slot's mbarrier (count 2) with its own transaction bytes: issuing a tensor
// copy costs the issuing thread ~90 ns, and the issuing warp is on the
// CTA's critical path (every tile ends in a barrier), so the two copies go
// out from two warps side by side.  Out-of-range columns of the last tile
// are zero-filled by the TMA unit and still count toward the bytes.
__device__ __forceinline__ bool ts_issuer() { return (threadIdx.x & ~32u) == 0; }

__device__ __forceinline__ void ts_issue(const TsRing& R, int b, int tw, int nb,
                                         const CUtensorMap* tmW, const float* vsrc,
                                         int64_t e0, int64_t L) {
    const unsigned bar = R.bar(b);
    float* dst = R.buf(b);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"((unsigned)(tw * nb * 4))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
            "l"(reinterpret_cast<uint64_t>(tmW)), "r"((int)e0), "r"(0), "r"(bar)
            : "memory");
    } else {
        // the vector tile is contiguous: a plain bulk copy (no tensor box;
        // columns past L stay unwritten and are never read)
        const int64_t left = L - e0;
        const unsigned bytes = (unsigned)((left < tw ? left : (int64_t)tw) * 4);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
            "[%3];" ::"r"(smem_u32(dst + (size_t)nb * tw)),
            "l"(vsrc + e0), "r"(bytes), "r"(bar)
            : "memory");
    }
}

// Gram variant: also gacc[r] += <row (warp + SW r), row grow> for rows < grow + 1.
// NR = this warp's row count (rows warp, warp + SW, ... below nrows), a
// template parameter picked by one warp-uniform switch per tile: a guard per
// row inside the unrolled loop cost a branch region (BSSY / BRA / BSYNC,
// ~25 cycles of branch latency) for each of the up-to-8 rows a warp does NOT
// have, twice per tile -- most of a tile's time at small k.
template <int NR>
__device__ __forceinline__ void ts_dots2_nr(const float* tile, int tw, int vrow, int grow, int cn,
                                            double* acc, double* gacc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* vr = tile + (size_t)vrow * tw;
    const float* gr = tile + (size_t)grow * tw;
#pragma unroll
    for (int c4 = 0; c4 < 2; ++c4) {
        const int e = c4 * 128 + lane * 4;       // a warp's LDS.128: 512 contiguous bytes
        if (c4 * 128 >= tw || e >= cn) break;
        const float4 v = *reinterpret_cast<const float4*>(vr + e);
        const float4 u = *reinterpret_cast<const float4*>(gr + e);
        const double v0 = v.x, v1 = v.y, v2 = v.z, v3 = v.w;
        const double u0 = u.x, u1 = u.y, u2 = u.z, u3 = u.w;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int j = warp + SW * r;
            const float4 w = *reinterpret_cast<const float4*>(tile + (size_t)j * tw + e);
            const double x0 = w.x, x1 = w.y, x2 = w.z, x3 = w.w;
            double a = acc[r];
            a = fma(x0, v0, a);
            a = fma(x1, v1, a);
            a = fma(x2, v2, a);
            a = fma(x3, v3, a);
            acc[r] = a;
            double b = gacc[r];
            b = fma(x0, u0, b);
            b = fma(x1, u1, b);
            b = fma(x2, u2, b);
            b = fma(x3, u3, b);
            gacc[r] = b;
        }
    }
}

__device__ __forceinline__ void ts_dots2(const float* tile, int tw, int nrows, int vrow, int grow,
                                         int cn, double* acc, double* gacc) {
    const int warp = threadIdx.x >> 5;
    const int nr = nrows > warp ? (nrows - warp + SW - 1) / SW : 0;     // warp-uniform
    switch (nr) {
        case 0: break;
        case 1: ts_dots2_nr<1>(tile, tw, vrow, grow, cn, acc, gacc); break;
        case 2: ts_dots2_nr<2>(tile, tw, vrow, grow, cn, acc, gacc); break;
        case 3: ts_dots2_nr<3>(tile, tw, vrow, grow, cn, acc, gacc); break;
        case 4: ts_dots2_nr<4>(tile, tw, vrow, grow, cn, acc, gacc); break;
        case 5: ts_dots2_nr<5>(tile, tw, vrow, grow, cn, acc, gacc); break;
        case 6: ts_dots2_nr<6>(tile, tw, vrow, grow, cn, acc, gacc); break;
        case 7: ts_dots2_nr<7>(tile, tw, vrow, grow, cn, acc, gacc); break;
        default: ts_dots2_nr<TS_RPW>(tile, tw, vrow, grow, cn, acc, gacc); break;
    }
}

// acc[r] += <row (warp + SW r), vector row> over one tile (fp64 products);
// NR as in ts_dots2_nr.
template <int NR>
__device__ __forceinline__ void ts_dots_nr(const float* tile, int tw, int vrow, int cn,
                                           double* acc) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const float* vr = tile + (size_t)vrow * tw;
#pragma unroll
    for (int c4 = 0; c4 < 2; ++c4) {
        const int e = c4 * 128 + lane * 4;       // a warp's LDS.128: 512 contiguous bytes
        if (c4 * 128 >= tw || e >= cn) break;
        const float4 v = *reinterpret_cast<const float4*>(vr + e);
        const double v0 = v.x, v1 = v.y, v2 = v.z, v3 = v.w;
#pragma unroll
        for (int r = 0; r < NR; ++r) {
            const int j = warp + SW * r;
            const float4 w = *reinterpret_cast<const float4*>(tile + (size_t)j * tw + e);
            double a = acc[r];
            a = fma((double)w.x, v0, a);
            a = fma((double)w.y, v1, a);
            a = fma((double)w.z, v2, a);
            a = fma((double)w.w, v3, a);
            acc[r] = a;
        }
    }
}

__device__ __forceinline__ void ts_dots(const float* tile, int tw, int nrows, int vrow, int cn,
                                        double* acc) {
    const int warp = threadIdx.x >> 5;
    const int nr = nrows > warp ? (nrows - warp + SW - 1) / SW : 0;     // warp-uniform
    switch (nr) {
        case 0: break;
        case 1: ts_dots_nr<1>(tile, tw, vrow, cn, acc); break;
        case 2: ts_dots_nr<2>(tile, tw, vrow, cn, acc); break;
        case 3: ts_dots_nr<3>(tile, tw, vrow, cn, acc); break;
        case 4: ts_dots_nr<4>(tile, tw, vrow, cn, acc); break;
        case 5: ts_dots_nr<5>(tile, tw, vrow, cn, acc); break;
        case 6: ts_dots_nr<6>(tile, tw, vrow, cn, acc); break;
        case 7: ts_dots_nr<7>(tile, tw, vrow, cn, acc); break;
        default: ts_dots_nr<TS_RPW>(tile, tw, vrow, cn, acc); break;
    }
}

// out[e] = vector[e] - sum_j c[j] W_j[e] over one tile: the ST threads split
// the rows into ST / tw groups whose fp64 partials meet in red[] and are
// summed in group order.  The rounded result goes to dst (global) and, when
// keep, back into the tile's vector row.  Returns this thread's ||out||^2 part.
// sdp != NULL: also write the result's K1 staged copies (element e0 + e of
// the image: P row-major, PT transposed -- 4-byte stores one row apart, which
// L2 merges into whole sectors before they reach HBM).
__device__ __forceinline__ double ts_update(float* tile, int tw, int nb, const double* c, int cn,
                                            float* dst, bool keep, double* red,
                                            double scale = 1.0,
                                            const ctk_stage_dst* sdp = nullptr, int iy0 = 0,
                                            int ix0 = 0) {
    const int ng = ST / tw;
    const int g = threadIdx.x / tw, e = threadIdx.x - g * tw;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;       // four independent chains
    if (e < cn) {
        const float* col = tile + e;
        int j = g;
        for (; j + 3 * ng < nb; j += 4 * ng) {
            a0 = fma(c[j], (double)col[(size_t)j * tw], a0);
            a1 = fma(c[j + ng], (double)col[(size_t)(j + ng) * tw], a1);
            a2 = fma(c[j + 2 * ng], (double)col[(size_t)(j + 2 * ng) * tw], a2);
            a3 = fma(c[j + 3 * ng], (double)col[(size_t)(j + 3 * ng) * tw], a3);
        }
        for (; j < nb; j += ng) a0 = fma(c[j], (double)col[(size_t)j * tw], a0);
    }
    red[threadIdx.x] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    double nrm = 0.0;
    if (g == 0 && e < cn) {
        double t = 0.0;
        for (int q = 0; q < ng; ++q) t += red[q * tw + e];
        const float o = (float)(((double)tile[(size_t)nb * tw + e] - t) * scale);
        dst[e] = o;
        if (keep) tile[(size_t)nb * tw + e] = o;
        nrm = (double)o * (double)o;
        if (sdp) {
            int iy = iy0, ix = ix0 + e;          // element (iy0, ix0) + e of the image
            while (ix >= sdp->nx) {
                ix -= sdp->nx;
                ++iy;
            }
            sdp->P[(size_t)iy * (sdp->nx + 2 * sdp->pad) + ix + sdp->pad] = o;
            sdp->PT[(size_t)ix * (sdp->ny + 2 * sdp->pad) + iy + sdp->pad] = o;
        }
    }
    __syncthreads();
    return nrm;
}

struct TsMaps {
    CUtensorMap W;          // rows 0..k of the basis, box tw x (k+1)
};

template <int TW, int NBUF>         // tile width (floats), ring depth: compile-time index arithmetic
__global__ void __launch_bounds__(ST, 1) k_gs_stream(float* W, int64_t ld, int k, int64_t L,
                                                     const float* __restrict__ q, int passes,
                                                     double* h, double* stat,
                                                     double* partial, ctk_stage_dst sd,
                                                     double* hm, int stat_off, float* gram,
                                                     const __grid_constant__ TsMaps tm) {
    cg::grid_group grid = cg::this_grid();
    GS_STAMP(0);
    ctk_pdl_trigger();
    extern __shared__ __align__(16) unsigned char smem_raw[];
    constexpr int tw = TW;
    const int nb = k + 1;
    constexpr int TS_NBUF = NBUF;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem_raw);                 // [TS_MAXBUF]
    double* h1 = reinterpret_cast<double*>(smem_raw + 8 * TS_MAXBUF);       // [2 nb + 2]
    double* h2 = h1 + (2 * nb + 2);                                         // [nb + 1]
    double* cc = h2 + (nb + 1);                                             // [nb + 1]
    double* red = cc + (nb + 1);                                            // [ST]
    // ring slots: 128-B aligned for the tensor copies
    unsigned char* ring_raw = smem_raw + 8 * TS_MAXBUF + sizeof(double) * (4 * (size_t)nb + 4 + ST);
    ring_raw += (128u - (smem_u32(ring_raw) & 127u)) & 127u;
    float* ring = reinterpret_cast<float*>(ring_raw);
    TsRing R;
    R.ring = ring;
    R.bar0 = smem_u32(bars);
    R.stride = (nb + 1) * tw;
    if (threadIdx.x == 0) {
        for (int b = 0; b < TS_NBUF; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(R.bar(b)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    ctk_pdl_wait();                  // q (and, transitively, the basis) from the previous kernels
    GS_STAMP(1);

    const int64_t ntiles = (L + tw - 1) / tw;
    const int64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * per, t1 = min(ntiles, t0 + per);
    const int nt = t1 > t0 ? (int)(t1 - t0) : 0;
    float* wnext = W + (size_t)(k + 1) * ld;
    double* P1 = partial;                                    // [nb + 1][G]
    double* P2 = P1 + (size_t)(nb + 1) * gridDim.x;          // [nb + 1][G]
    double* P3 = P2 + (size_t)(nb + 1) * gridDim.x;          // [G]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // One sweep over this CTA's tiles.  mode 0: dots with the vector (row nb,
    // + its norm); 1: update -> wnext, then dots with the result; 2: update ->
    // wnext (times `scale`) and its norm; 3: mode 0 plus the Gram dots
    // <W_j, w_k> (rows nb + 1 + j of P).
    // The ring runs continuously across sweeps: tile number g (counted from
    // the kernel's first) uses slot g % TS_NBUF at mbarrier phase (g / TS_NBUF) & 1.
    int gbase = 0;
    auto sweep = [&](int mode, const float* vmap, const double* coef, double* P,
                     double scale, const ctk_stage_dst* stage = nullptr) -> double {
        double acc[TS_RPW], gacc[TS_RPW];
#pragma unroll
        for (int r = 0; r < TS_RPW; ++r) acc[r] = gacc[r] = 0.0;
        double nrm = 0.0;
        if (ts_issuer())
            for (int i = 0; i < TS_NBUF && i < nt; ++i)
                ts_issue(R, (gbase + i) % TS_NBUF, tw, nb, &tm.W, vmap, (t0 + i) * tw, L);
        // image position of the tile's first element for the staged copies,
        // advanced tile by tile (no division per element)
        int st_iy = 0, st_ix = 0;
        if (stage) {
            const int64_t f = t0 * tw;
            st_iy = (int)(f / stage->nx);
            st_ix = (int)(f - (int64_t)st_iy * stage->nx);
        }
        for (int i = 0; i < nt; ++i) {
            const int g = gbase + i, b = g % TS_NBUF;
            const int64_t e0 = (t0 + i) * tw;
            const int cn = (int)min((int64_t)tw, L - e0);
            mbar_wait(R.bar(b), (unsigned)(g / TS_NBUF) & 1u);
            float* tile = R.buf(b);
            if (mode == 0) {
                ts_dots(tile, tw, nb + 1, nb, cn, acc);
            } else if (mode == 3) {
                ts_dots2(tile, tw, nb + 1, nb, nb - 1, cn, acc, gacc);
            } else {
                nrm += ts_update(tile, tw, nb, coef, cn, wnext + e0, mode == 1, red, scale, stage,
                                 st_iy, st_ix);
                if (mode == 1) ts_dots(tile, tw, nb, nb, cn, acc);
                if (stage) {
                    st_ix += tw;
                    while (st_ix >= stage->nx) {
                        st_ix -= stage->nx;
                        ++st_iy;
                    }
                }
            }
            // everyone is done with slot b (mode 2: ts_update ended in a barrier)
            if (mode != 2) __syncthreads();
            if (ts_issuer() && i + TS_NBUF < nt)
                ts_issue(R, b, tw, nb, &tm.W, vmap, (t0 + i + TS_NBUF) * tw, L);
        }
        gbase += nt;
        if (mode != 2) {
            const int rows = mode == 1 ? nb : nb + 1;
#pragma unroll
            for (int r = 0; r < TS_RPW; ++r) {
                const int j = warp + SW * r;
                if (j >= rows) break;                      // warp-uniform
                const double t = warp_sum(acc[r]);
                if (lane == 0) P[(size_t)j * gridDim.x + blockIdx.x] = t;
            }
            if (mode == 3) {
#pragma unroll
                for (int r = 0; r < TS_RPW; ++r) {
                    const int j = warp + SW * r;
                    if (j >= nb) break;                    // warp-uniform
                    const double t = warp_sum(gacc[r]);
                    if (lane == 0) P[(size_t)(nb + 1 + j) * gridDim.x + blockIdx.x] = t;
                }
            }
        }
        return nrm;
    };

    __shared__ double s_n2;
    bool need_norm = true, prescaled = false, staged = false;
    double nrm = 0.0;
    if (gram && passes == 2) {
        // Gram-corrected CGS2 (see gram_coefs): two sweeps, one reduction --
        // h1, ||q||^2 and <W_j, w_k> in one read of the basis, then
        // q2 = (q - W c) / ||q2|| straight into row k+1
        sweep(3, q, nullptr, P1, 1.0);
        GS_STAMP(2);
        grid.sync();
        GS_STAMP(3);
        all_reduce_rows(P1, 2 * nb + 1, h1);
        __syncthreads();
        GS_STAMP(4);
        __shared__ double s_est;
        gram_coefs<false>(gram, gram, GRAM_LD, k, h1, h1 + nb + 1, h2, cc, red, &s_est);
        GS_STAMP(5);
        const double est = s_est, a = h1[nb];
        if (a > 0.0 && est > 1e-8 * a) {
            // the final scale is known here: the K1 staged copies of w_{k+1}
            // are written in the same sweep (no re-read, no extra barrier),
            // unless the step breaks down (hk is only known after the sweep)
            const bool fold = sd.P && sqrt(est) > 1e-14 * sqrt(a);
            sweep(2, q, cc, nullptr, 1.0 / sqrt(est), fold ? &sd : nullptr);
            if (threadIdx.x == 0) s_n2 = est;
            need_norm = false;
            prescaled = true;
            staged = fold;
        } else {
            nrm = sweep(2, q, cc, nullptr, 1.0);
        }
    } else {
        sweep(0, q, nullptr, P1, 1.0);                   // h1 = W^T q, ||q||^2
        grid.sync();
        all_reduce_rows(P1, nb + 1, h1);
        __syncthreads();
        const double* cfin = h1;
        const float* vfin = q;
        if (passes == 2) {
            sweep(1, q, h1, P2, 1.0);                    // q1 -> wnext, h2 = W^T q1
            asm volatile("fence.proxy.async.global;" ::: "memory");   // q1: generic writes, bulk reads
            grid.sync();
            all_reduce_rows(P2, nb, h2);
            __syncthreads();
            cfin = h2;
            vfin = wnext;
        }
        nrm = sweep(2, vfin, cfin, nullptr, 1.0);            // q2 -> wnext, ||q2||^2
    }
    GS_STAMP(6);
    if (need_norm) {
        nrm = warp_sum(nrm);
        if (lane == 0) red[warp] = nrm;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < SW; ++w) t += red[w];
            P3[blockIdx.x] = t;
        }
        grid.sync();
        if (threadIdx.x < 32) all_reduce_rows(P3, 1, &s_n2);
        __syncthreads();
    } else if (sd.P && !staged) {
        grid.sync();                 // the staging tiles below span other CTAs' rows
    }
    const double hk = sqrt(s_n2);
    const double qn = sqrt(h1[nb]);
    const bool broke = hk <= 1e-14 * qn;                     // BREAKDOWN_RTOL, arnoldi.py:17,80
    const float sc = broke ? 0.f : prescaled ? 1.f : (float)(1.0 / hk);
    if (staged) {
        // w_{k+1} and its staged copies were written by the update sweep
    } else if (!sd.P) {
        if (!prescaled && nt > 0) {
            const int64_t e0 = t0 * tw, e1 = min(L, t1 * tw);
            for (int64_t i = e0 + threadIdx.x; i < e1; i += ST) wnext[i] *= sc;
        }
    } else {
        // Scale and stage w_{k+1} for the next K1 apply by 32 x 32 image tiles
        // (each tile owned by one CTA): coalesced P rows, and the transposed
        // copy PT through a shared-memory tile instead of strided stores.
        float (*tr)[33] = reinterpret_cast<float (*)[33]>(ring);
        const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;      // 32 x 16
        const int tnx = (sd.nx + 31) >> 5, tny = (sd.ny + 31) >> 5;
        const int pP = sd.nx + 2 * sd.pad, pT = sd.ny + 2 * sd.pad;
        for (int t = blockIdx.x; t < tnx * tny; t += gridDim.x) {
            const int bx = (t % tnx) << 5, by = (t / tnx) << 5;
            for (int r = ty; r < 32; r += SW) {
                const int iy = by + r, ix = bx + tx;
                float v = 0.f;
                if (iy < sd.ny && ix < sd.nx) {
                    const size_t o = (size_t)iy * sd.nx + ix;
                    v = wnext[o] * sc;
                    if (!prescaled) wnext[o] = v;
                    sd.P[(size_t)iy * pP + ix + sd.pad] = v;
                }
                tr[r][tx] = v;
            }
            __syncthreads();
            for (int r = ty; r < 32; r += SW) {
                const int ix = bx + r, iy = by + tx;
                if (ix < sd.nx && iy < sd.ny) sd.PT[(size_t)ix * pT + iy + sd.pad] = tr[tx][r];
            }
            __syncthreads();
        }
    }
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i <= k; i += ST) {
            const double v = passes == 2 ? h1[i] + h2[i] : h1[i];
            h[i] = v;
            if (hm) hm[i] = v;
        }
        if (threadIdx.x == 0) {
            const double st4[4] = {qn, broke ? 1.0 : 0.0, broke ? 0.0 : 1.0 / hk, hk};
            h[k + 1] = hk;
            for (int c = 0; c < 4; ++c) stat[c] = st4[c];
            if (hm) {
                hm[k + 1] = hk;
                for (int c = 0; c < 4; ++c) hm[stat_off + c] = st4[c];
            }
        }
    }
    GS_STAMP(7);
}

}  // namespace ctk

using namespace ctk;

// Cooperative fused path when L is small and the device supports it.
static int try_cgs2_fused(float* W, int64_t ld, int k, int64_t L, float* q, double* h,
                          double* stat, Scratch s, cudaStream_t st, bool* done) {
    *done = false;
    if (L > FUSED_MAX_L) return CTK_OK;
    static int coop = -1, sms = 0, per_sm = 0;
    if (coop < 0) {
        const char* off = getenv("CTK_NO_FUSED_CGS2");
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cgs2_fused, FT,
                                                      sizeof(double) * 512 * (FW + 1));
        cudaGetLastError();
        if (off && off[0] == '1') coop = 0;
    }
    if (coop != 1 || per_sm < 1 || k + 2 > 512) return CTK_OK;
    int64_t G = ((L >> 2) + FT - 1) / FT;            // >= one float4 per thread
    static int cap = -1, mult = 1;
    if (cap < 0) {
        const char* e = getenv("CTK_FUSED_CTAS");
        cap = e ? atoi(e) : 0;
        const char* m = getenv("CTK_FUSED_PER_SM");      // tuning override (CTAs per SM)
        mult = m && atoi(m) > 0 ? atoi(m) : 1;
        if (mult > per_sm) mult = per_sm;
    }
    if (G > (int64_t)sms * mult) G = (int64_t)sms * mult;
    if (cap > 0 && G > cap) G = cap;
    if (G < 1) G = 1;
    double* red = s.tmp;
    void* args[] = {&W, &ld, &k, &L, &q, &h, &stat, &s.partial, &red};
    const size_t smem = sizeof(double) * ((size_t)(k + 1) + (size_t)(k + 2) * FW);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_cgs2_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(sizeof(double) * 512 * (FW + 1)));
        attr = true;
    }
    cudaError_t e = cudaLaunchCooperativeKernel((const void*)k_cgs2_fused, dim3((unsigned)G),
                                                dim3(FT), args, smem, st);
    ctk_count_launch();
    if (e != cudaSuccess) return ctk_check_cuda(e, "k_cgs2_fused");
    *done = true;
    return CTK_OK;
}

// SMEM-resident path when every CTA's chunk of the k+1 rows fits in shared
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult qr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr) !=
                cudaSuccess ||
            qr != cudaDriverEntryPointSuccess)
            p = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// fp32 2-D map over `rows` rows of length L (pitch ld floats), box tw x rows.
static bool encode_rows(CUtensorMap* m, const float* base, int64_t L, int64_t ld, int rows, int tw) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)L, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * sizeof(float)};
    cuuint32_t box[2] = {(cuuint32_t)tw, (cuuint32_t)rows};
    cuuint32_t es[2] = {1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
               es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// memory with one CTA per SM.
static size_t gs_smem_bytes(int k, int64_t chunk) {
    const int nb = k + 1;
    const size_t head = (16 + sizeof(double) * (4 * (size_t)nb + 4 + SW) + 15) & ~(size_t)15;
    return head + sizeof(float) * (size_t)chunk * (nb + 1) + 2 * sizeof(double) * (size_t)chunk +
           sizeof(float) * (((size_t)k * k + 3) & ~(size_t)3) + sizeof(double) * 4 * ST + 32 + 128;
}

static bool gs_smem_plan(int64_t L, int k, int64_t* Gp, int64_t* chunkp, size_t* smemp) {
    static int coop = -1, sms = 0, gcap = 0;
    if (coop < 0) {
        const char* off = getenv("CTK_NO_SMEM_GS");
        const char* e = getenv("CTK_GS_CTAS");             // tuning override
        gcap = e ? atoi(e) : 0;
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaFuncSetAttribute(k_gs_smem, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_LIMIT) != cudaSuccess)
            coop = 0;
        cudaGetLastError();
        if (off && off[0] == '1') coop = 0;
    }
    if (coop != 1 || L < 4 || k < 0) return false;
    // chunk: a multiple of 64 floats (the TMA panel), at most 256 panels
    int64_t G = gcap > 0 && gcap < sms ? gcap : sms;
    int64_t chunk = ((L + G - 1) / G + 63) & ~63LL;
    if (chunk > 64 * 256 || k + 1 > 256) return false;
    G = (L + chunk - 1) / chunk;
    if (G > GS_MAXG) return false;
    const size_t smem = gs_smem_bytes(k, chunk);
    if (smem > SMEM_LIMIT) return false;
    // partials: (nb + 1) + (nb + 1) + 1 rows of G doubles within carve(scratch, k + 3)
    if ((size_t)(2 * k + 5) * G > (size_t)MAXCH * (size_t)(k + 3)) return false;
    *Gp = G;
    *chunkp = chunk;
    *smemp = smem;
    return true;
}

static int try_gs_smem(float* W, int64_t ld, int k, int64_t L, float* q, int passes, double* h,
                       double* stat, Scratch s, cudaStream_t st, const ctk_stage_dst* sdp,
                       double* hm, float* gram, bool* done) {
    *done = false;
    int64_t G, chunk;
    size_t smem;
    if (!gs_smem_plan(L, k, &G, &chunk, &smem)) return CTK_OK;
    double* partial = s.partial;
    ctk_stage_dst sd = {};
    if (sdp && sdp->P && (int64_t)sdp->nx * sdp->ny == L) sd = *sdp;
    int stat_off = (int)(stat - h);
    // the CTA blocks of the k+1 rows as one 3-D TMA box each (64-float panels)
    CUtensorMap tm;
    memset(&tm, 0, sizeof(tm));
    int use_tma = 0;
    if (auto enc = tensor_map_encoder()) {
        cuuint64_t dims[3] = {64, (cuuint64_t)((L + 63) / 64), (cuuint64_t)(k + 1)};
        cuuint64_t strides[2] = {64 * sizeof(float), (cuuint64_t)ld * sizeof(float)};
        cuuint32_t box[3] = {64, (cuuint32_t)(chunk / 64), (cuuint32_t)(k + 1)};
        cuuint32_t es[3] = {1, 1, 1};
        use_tma = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, W, dims, strides, box, es,
                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    // cooperative (grid barriers) and programmatic: the launch and the
    // prologue overlap the producer of q (K2 / K1), which triggers at entry
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(ST);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(&cfg, k_gs_smem, W, ld, k, L, (const float*)q, passes, chunk,
                                       h, stat, partial, sd, hm, stat_off, use_tma, gram, tm);
    ctk_count_launch();
    if (e != cudaSuccess) return ctk_check_cuda(e, "k_gs_smem");
    *done = true;
    return CTK_OK;
}

bool ctk_gs_smem_ok(int64_t L, int k) {
    int64_t G, chunk;
    size_t smem;
    return gs_smem_plan(L, k, &G, &chunk, &smem);
}

// Streamed path: L a multiple of 4 (16-B row pitch of q), at most TS_MAXROWS
// rows, two ring buffers of the widest tile (256 or 128 floats) that fit.
static size_t gs_stream_bytes(int k, int tw, int nbuf) {
    const int nb = k + 1;
    const size_t head = 8 * TS_MAXBUF + sizeof(double) * (4 * (size_t)nb + 4 + ST) + 128;
    return head + nbuf * sizeof(float) * (size_t)(nb + 1) * tw;
}

static bool gs_stream_plan(int64_t L, int k, int* twp, size_t* smemp, int* Gp, int* nbufp) {
    static int coop = -1, sms = 0;
    if (coop < 0) {
        const char* off = getenv("CTK_NO_STREAM_GS");
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaFuncSetAttribute(k_gs_stream<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_LIMIT) != cudaSuccess ||
            cudaFuncSetAttribute(k_gs_stream<256, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_LIMIT) != cudaSuccess ||
            cudaFuncSetAttribute(k_gs_stream<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)SMEM_LIMIT) != cudaSuccess)
            coop = 0;
        cudaGetLastError();
        if (off && off[0] == '1') coop = 0;
    }
    if (coop != 1 || k < 0 || (L & 3) || k + 2 > TS_MAXROWS || sms > GS_MAXG) return false;
    if (L >= (1LL << 31) || !tensor_map_encoder()) return false;   // 32-bit TMA coordinates
    if (L < (int64_t)sms * 1024) return false;           // short vectors: SMEM / fused paths
    static const int max_buf = [] {
        const char* e = getenv("CTK_TS_NBUF");            // tuning override: 2 = never 4 slots
        return e && atoi(e) == 2 ? 2 : TS_MAXBUF;
    }();
    for (int tw = 256; tw >= 128; tw >>= 1) {         // ts_dots: 4 or 8 floats per lane
        if (gs_stream_bytes(k, tw, 2) > SMEM_LIMIT) continue;
        const int nbuf =
            tw == 256 && max_buf == 4 && gs_stream_bytes(k, tw, 4) <= SMEM_LIMIT ? 4 : 2;
        *twp = tw;
        *smemp = gs_stream_bytes(k, tw, nbuf);
        *Gp = sms;
        *nbufp = nbuf;
        return true;
    }
    return false;
}

bool ctk_gs_stream_ok(int64_t L, int k) {
    int tw, G, nbuf;
    size_t smem;
    return !ctk_gs_smem_ok(L, k) && gs_stream_plan(L, k, &tw, &smem, &G, &nbuf);
}

static int try_gs_stream(float* W, int64_t ld, int k, int64_t L, const float* q, int passes,
                         double* h, double* stat, Scratch s, cudaStream_t st,
                         const ctk_stage_dst* sdp, double* hm, float* gram, bool* done) {
    *done = false;
    int tw, G, nbuf;
    size_t smem;
    if (!gs_stream_plan(L, k, &tw, &smem, &G, &nbuf)) return CTK_OK;
    if ((size_t)(2 * k + 5) * G > (size_t)MAXCH * (size_t)(k + 3)) return CTK_OK;
    ctk_stage_dst sd = {};
    if (sdp && sdp->P && (int64_t)sdp->nx * sdp->ny == L) sd = *sdp;
    const int stat_off = (int)(stat - h);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(ST);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    TsMaps tm;
    if (!encode_rows(&tm.W, W, L, ld, k + 1, tw))
        return CTK_OK;                                   // no TMA encoder: other paths
    auto kern = tw == 256 ? (nbuf == 4 ? k_gs_stream<256, 4> : k_gs_stream<256, 2>)
                          : k_gs_stream<128, 2>;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, W, ld, k, L, q, passes, h, stat, s.partial, sd,
                                       hm, stat_off, gram, tm);
    ctk_count_launch();
    if (e != cudaSuccess) return ctk_check_cuda(e, "k_gs_stream");
    *done = true;
    return CTK_OK;
}

static int check_vec(const void* p, const char* what) {
    if (!p) return ctk_fail(CTK_ERR_ARG, "%s is NULL", what);
    if (((uintptr_t)p) & 15) return ctk_fail(CTK_ERR_ARG, "%s is not 16-byte aligned", what);
    return CTK_OK;
}

extern "C" size_t ctk_reduce_scratch_bytes(int nvec, int64_t L) {
    (void)L;
    const int cap = nvec + 3;
    return 256 + GRAM_BYTES + sizeof(double) * ((size_t)MAXCH * cap + 3 * (size_t)cap) + 256;
}

static int launch_dots(const float* W, int64_t ld, int nvec, const float* v, int64_t L,
                       int want_norm, double* out, Scratch s, cudaStream_t st) {
    const int nv = nvec + (want_norm ? 1 : 0);
    if (nv > s.nvec_cap || nv > KMAX_VEC) return ctk_fail(CTK_ERR_ARG, "too many vectors (%d)", nv);
    const int64_t L4 = L >> 2;
    const int64_t ch = chunk_len(L4);
    int64_t nch = (L4 + ch - 1) / ch;
    if (nch < 1) nch = 1;
    dim3 grid((unsigned)nch, (unsigned)((nv + JG - 1) / JG));
    k_dots<<<grid, KT, 0, st>>>(W, ld, nvec, v, L, want_norm, ch, out, s.partial, s.ticket);
    CTK_LAUNCH_CHECK("k_dots");
    return CTK_OK;
}

static int combine_ctas(int64_t L) {
    int64_t G = ((L >> 2) + 31) / 32;                 // 32-float4 column tiles
    if (G > MAXCH / 2) G = MAXCH / 2;
    return G < 1 ? 1 : (int)G;
}

static int launch_combine(const float* W, int64_t ld, int nvec, const double* coef, double sgn,
                          const float* base, float* dst, int64_t L, double* norm_out, Scratch s,
                          cudaStream_t st) {
    if (nvec > KMAX_VEC) return ctk_fail(CTK_ERR_ARG, "too many vectors (%d)", nvec);
    CombineJob j0 = {W, ld, sgn, base, dst, L, norm_out, s.partial, s.ticket, combine_ctas(L)};
    CombineJob j1 = j0;
    j1.G = 0;
    const size_t smem = sizeof(double) * (size_t)(nvec > 0 ? nvec : 1);
    CoefPack cp;
    k_combine<<<(unsigned)j0.G, CT, smem, st>>>(j0, j1, nvec, coef, cp);
    CTK_LAUNCH_CHECK("k_combine");
    return CTK_OK;
}

// x = x0 + sum y_j X_j (norm -> n_x) and r = d0 - sum y_j AX_j (norm -> n_r)
// in one launch (ctk_iterate's linear path).
int ctk_combine_pair(const float* X, int64_t ldx, const float* x0, float* x, int64_t Lx,
                     double* n_x, const float* AX, int64_t ldax, const float* d0, float* r,
                     int64_t Lr, double* n_r, int k, const double* y, void* scratch,
                     void* stream, const double* y_host) {
    if (k > KMAX_VEC) return ctk_fail(CTK_ERR_ARG, "too many vectors (%d)", k);
    if ((ldx & 3) || (ldax & 3)) return ctk_fail(CTK_ERR_ARG, "ld must be a multiple of 4");
    Scratch s = carve(scratch, k + 3);
    CombineJob j0 = {X, ldx, 1.0, x0, x, Lx, n_x, s.partial, s.ticket, combine_ctas(Lx)};
    CombineJob j1 = {AX, ldax, -1.0, d0, r, Lr, n_r, s.partial + j0.G, s.ticket + 1,
                     combine_ctas(Lr)};
    const size_t smem = sizeof(double) * (size_t)(k > 0 ? k : 1);
    CoefPack cp;
    const bool byval = y_host && k <= COEF_BYVAL;     // no H2D copy of y on the stream
    if (byval) memcpy(cp.c, y_host, sizeof(double) * (size_t)k);
    k_combine<<<(unsigned)(j0.G + j1.G), CT, smem, ctk_stream(stream)>>>(j0, j1, k,
                                                                         byval ? nullptr : y, cp);
    CTK_LAUNCH_CHECK("k_combine");
    return CTK_OK;
}

static int iter_batch_ctas(int64_t L) {
    int64_t G = ((L >> 2) + IB_T - 1) / IB_T;
    if (G > CTK_IB_GCAP * 148) G = CTK_IB_GCAP * 148;
    return (int)(G < 1 ? 1 : G);
}

bool ctk_iterate_batch_ok(int k0, int nb, int nvec_cap, int64_t Lx, int64_t Lr) {
    if (nb < 1 || nb > IB_NB || k0 < 1 || k0 + nb - 1 > IB_MAXK) return false;
    const int64_t need = (int64_t)IB_NB * (iter_batch_ctas(Lx) + iter_batch_ctas(Lr));
    return need <= (int64_t)MAXCH * (nvec_cap + 3);
}

extern "C" int ctk_iterate_batch(const float* X, int64_t ldx, const float* x0, float* x,
                                 int64_t Lx, const float* AX, int64_t ldax, const float* d0,
                                 float* r, int64_t Lr, int k0, int nb, const double* y,
                                 int ystride, double* norms, void* scratch, int nvec_cap,
                                 void* stream) {
    if (!X || !AX || !d0 || !y || !norms || !scratch)
        return ctk_fail(CTK_ERR_ARG, "null argument");
    if ((ldx & 3) || (ldax & 3)) return ctk_fail(CTK_ERR_ARG, "ld must be a multiple of 4");
    if (!ctk_iterate_batch_ok(k0, nb, nvec_cap, Lx, Lr))
        return ctk_fail(CTK_ERR_ARG, "bad iterate batch (k0 %d, nb %d)", k0, nb);
    Scratch s = carve(scratch, nvec_cap + 3);
    IterBatchJob j0 = {X, ldx, x0, x, Lx, norms + 1, s.partial, s.ticket, iter_batch_ctas(Lx)};
    IterBatchJob j1 = {AX, ldax, d0, r, Lr, norms, s.partial + (size_t)IB_NB * j0.G, s.ticket + 1,
                       iter_batch_ctas(Lr)};
    const int ph = ctk_prof_open(3, ctk_stream(stream));
    static const int ibv = [] {                 // floats per thread and row (tuning override)
        const char* e = getenv("CTK_IB_V");
        return e && atoi(e) == 2 ? 2 : 4;
    }();
    if (ibv == 4)
        k_iter_batch<4><<<(unsigned)(j0.G + j1.G), IB_T, 0, ctk_stream(stream)>>>(j0, j1, y, ystride,
                                                                                k0, nb);
    else
        k_iter_batch<2><<<(unsigned)(j0.G + j1.G), IB_T, 0, ctk_stream(stream)>>>(j0, j1, y, ystride,
                                                                                k0, nb);
    CTK_LAUNCH_CHECK("k_iter_batch");
    ctk_prof_close(ph, ctk_stream(stream));
    return CTK_OK;
}

extern "C" int ctk_dots(const float* W, int64_t ld, int nvec, const float* v, int64_t L,
                        int want_norm, double* out, void* scratch, void* stream) {
    int rc;
    if (nvec > 0 && (rc = check_vec(W, "W"))) return rc;
    if ((rc = check_vec(v, "v"))) return rc;
    if (!out || !scratch) return ctk_fail(CTK_ERR_ARG, "null output/scratch");
    if (ld & 3) return ctk_fail(CTK_ERR_ARG, "ld must be a multiple of 4");
    return launch_dots(W, ld, nvec, v, L, want_norm, out, carve(scratch, nvec + 3),
                       ctk_stream(stream));
}

extern "C" int ctk_update(const float* W, int64_t ld, int nvec, const double* coef,
                          const float* v, float* dst, int64_t L, double* norm2_out, void* scratch,
                          void* stream) {
    int rc;
    if (nvec > 0 && (rc = check_vec(W, "W"))) return rc;
    if ((rc = check_vec(v, "v")) || (rc = check_vec(dst, "dst"))) return rc;
    if (ld & 3) return ctk_fail(CTK_ERR_ARG, "ld must be a multiple of 4");
    if (!scratch || (nvec > 0 && !coef)) return ctk_fail(CTK_ERR_ARG, "null coef/scratch");
    return launch_combine(W, ld, nvec, coef, -1.0, v, dst, L, norm2_out, carve(scratch, nvec + 3),
                          ctk_stream(stream));
}

extern "C" int ctk_combine(const float* W, int64_t ld, int k, const double* y, const float* x0,
                           float* dst, int64_t L, double* norm2_out, void* scratch, void* stream) {
    int rc;
    if (k > 0 && (rc = check_vec(W, "W"))) return rc;
    if ((rc = check_vec(dst, "dst"))) return rc;
    if (x0 && (rc = check_vec(x0, "x0"))) return rc;
    if (ld & 3) return ctk_fail(CTK_ERR_ARG, "ld must be a multiple of 4");
    if (!scratch || (k > 0 && !y)) return ctk_fail(CTK_ERR_ARG, "null y/scratch");
    return launch_combine(W, ld, k, y, 1.0, x0, dst, L, norm2_out, carve(scratch, k + 3),
                          ctk_stream(stream));
}

extern "C" int ctk_norm2(const float* v, int64_t L, double* out, void* scratch, void* stream) {
    int rc;
    if ((rc = check_vec(v, "v"))) return rc;
    if (!out || !scratch) return ctk_fail(CTK_ERR_ARG, "null output/scratch");
    return launch_dots(nullptr, 4, 0, v, L, 1, out, carve(scratch, 3), ctk_stream(stream));
}

extern "C" int ctk_scale(const float* v, float* dst, int64_t L, const double* scale_dev,
                         void* stream) {
    if (!v || !dst || !scale_dev) return ctk_fail(CTK_ERR_ARG, "null argument");
    int blocks = (int)((L + 255) / 256);
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    k_scale<<<blocks, 256, 0, ctk_stream(stream)>>>(v, dst, L, scale_dev);
    CTK_LAUNCH_CHECK("k_scale");
    return CTK_OK;
}

extern "C" int ctk_cgs2_step(float* W, int64_t ld, int k, int64_t L, float* q, double* h,
                             double* stat, void* scratch, void* stream) {
    return ctk_gs_step(W, ld, k, L, q, 2, h, stat, scratch, stream);
}

extern "C" int ctk_gs_step(float* W, int64_t ld, int k, int64_t L, float* q, int passes,
                           double* h, double* stat, void* scratch, void* stream) {
    return ctk_gs_step_ex(W, ld, k, L, q, passes, h, stat, scratch, stream, nullptr, nullptr);
}

// Gram-matrix bookkeeping (host side, per scratch buffer): the Gram-corrected
// path needs E's columns 0..k-1, which exist when the previous calls on this
// scratch were steps 0..k-1 of the same basis (same W, ld, L), each on a
// single-launch path.  Launches on one scratch are stream-ordered, so the
// issue order here is the execution order.  Anything else (a first call at
// k > 0, another basis, a fallback path in between) runs the classic CGS2
// kernels for this step and restarts the chain at the next k = 0.
// CTK_NO_GRAM_GS=1 disables the Gram path (classic 2-reduction CGS2).
struct GramChain {
    const float* W;
    int64_t ld, L;
    int next_k;
};

static bool gram_track(void* scratch, const float* W, int64_t ld, int64_t L, int k, bool single) {
    static const bool off = [] {
        const char* e = getenv("CTK_NO_GRAM_GS");
        return e && e[0] == '1';
    }();
    static std::mutex mu;
    static std::unordered_map<void*, GramChain> chains;
    std::lock_guard<std::mutex> lk(mu);
    if (off || !single || k + 1 >= GRAM_LD) {
        chains.erase(scratch);
        return false;
    }
    auto it = chains.find(scratch);
    if (k == 0) {
        chains[scratch] = GramChain{W, ld, L, 1};
        return true;
    }
    if (it == chains.end() || it->second.W != W || it->second.ld != ld || it->second.L != L ||
        it->second.next_k != k) {
        chains.erase(scratch);
        return false;
    }
    it->second.next_k = k + 1;
    return true;
}

int ctk_gs_step_ex(float* W, int64_t ld, int k, int64_t L, float* q, int passes, double* h,
                   double* stat, void* scratch, void* stream, const ctk_stage_dst* sd,
                   double* h_mirror, const ctk_comm* comm) {
    int rc;
    if ((rc = check_vec(W, "W")) || (rc = check_vec(q, "q"))) return rc;
    if (ld & 3) return ctk_fail(CTK_ERR_ARG, "ld must be a multiple of 4");
    if (k < 0 || !h || !stat || !scratch) return ctk_fail(CTK_ERR_ARG, "bad cgs2 arguments");
    if (L > ld) return ctk_fail(CTK_ERR_SHAPE, "L (%lld) exceeds ld (%lld)", (long long)L,
                                (long long)ld);
    cudaStream_t st = ctk_stream(stream);
    Scratch s = carve(scratch, k + 3);
    if (passes != 1 && passes != 2) return ctk_fail(CTK_ERR_ARG, "passes must be 1 or 2");
    bool fused = false;
    const bool single =
        !comm && passes == 2 && (ctk_gs_smem_ok(L, k) || ctk_gs_stream_ok(L, k));
    float* gram = gram_track(scratch, W, ld, L, k, single) ? s.gram : nullptr;
    if (!comm) {
        if ((rc = try_gs_smem(W, ld, k, L, q, passes, h, stat, s, st, sd, h_mirror, gram, &fused)))
            return rc;
        if (fused) return CTK_OK;
        if ((rc = try_gs_stream(W, ld, k, L, q, passes, h, stat, s, st, sd, h_mirror, gram,
                                &fused)))
            return rc;
        if (fused) return CTK_OK;
        if (passes == 2 && (rc = try_cgs2_fused(W, ld, k, L, q, h, stat, s, st, &fused))) return rc;
        if (fused) return CTK_OK;
    }
    // multi-kernel CGS2; sharded vectors: every dot / norm summed over ranks
    auto sum = [&](double* v, int64_t cnt) { return comm ? ctk_comm_sum_f64(comm, v, cnt, st) : 0; };
    double* h1 = s.tmp;                   // k+2: h1[0..k], ||q||^2
    double* h2 = s.tmp + s.nvec_cap;      // k+1
    double* n2 = s.tmp + 2 * s.nvec_cap;  // 1
    const int nb = k + 1;
    float* wnext = W + (size_t)(k + 1) * ld;
    if ((rc = launch_dots(W, ld, nb, q, L, 1, h1, s, st))) return rc;            // h1, ||Mw||^2
    if ((rc = sum(h1, nb + 1))) return rc;
    if (passes == 1) {        // classical Gram-Schmidt, no reorthogonalisation pass
        if ((rc = launch_combine(W, ld, nb, h1, -1.0, q, wnext, L, n2, s, st))) return rc;
        if ((rc = sum(n2, 1))) return rc;
        k_cgs2_finalize<<<1, 128, 0, st>>>(h1, nullptr, n2, k, h, stat);
        CTK_LAUNCH_CHECK("k_cgs2_finalize");
        return ctk_scale(wnext, wnext, L, stat + 2, stream);
    }
    if ((rc = launch_combine(W, ld, nb, h1, -1.0, q, q, L, nullptr, s, st))) return rc;  // q1
    if ((rc = launch_dots(W, ld, nb, q, L, 0, h2, s, st))) return rc;            // h2
    if ((rc = sum(h2, nb))) return rc;
    if ((rc = launch_combine(W, ld, nb, h2, -1.0, q, wnext, L, n2, s, st))) return rc;   // q2
    if ((rc = sum(n2, 1))) return rc;
    k_cgs2_finalize<<<1, 128, 0, st>>>(h1, h2, n2, k, h, stat);
    CTK_LAUNCH_CHECK("k_cgs2_finalize");
    return ctk_scale(wnext, wnext, L, stat + 2, stream);
}
