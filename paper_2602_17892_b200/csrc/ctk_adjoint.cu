// ctk_adjoint.cu -- K7: the exact adjoint A^T of the Siddon forward projector
// (matched mode, LSQR/LSMR).  Reference: ctkrylov/ct.py:248-264
// (`matched_back` = the transpose of the assembled Siddon CSR, ct.py:182-201).
//
// Pixel-driven gather: for pixel p and angle a, every ray j whose line
// x cos + y sin = s_j crosses the pixel square contributes len(ray ∩ p) u[a, j].
// Siddon's segment inside a (convex) pixel is exactly that chord, whose length
// as a function of the signed distance d between the line and the pixel centre
// is a trapezoid:
//     len(d) = min(h / max(|c|,|s|), max(0, (P - |d|) / (|c| |s|))),
//     P = (|c| + |s|) h / 2  (half-width of the pixel's shadow).
// The reference drops segments <= 1e-15 (ct.py:178); the difference is below
// fp32 resolution.  Angles the reference treats as axis-aligned (K1d: rays can
// lie exactly on grid lines, and the midpoint/floor/clip rule decides which
// column gets them) use the literal fp64 segment lists of K1d, transposed once
// into per-pixel CSR lists (ray, length) on first use.
//
// B200 mapping mirrors K2: a CTA per 32 x 16 (32 x 32 for >= 512^2) pixel
// tile, 2 (4) pixels per thread;
// per 32-angle chunk the detector window of the tile is staged into SMEM with
// coalesced loads (zero outside [0, D)), then each pixel evaluates the 4
// candidate rays j0-1..j0+2 around g = j0 + f.  Away from the axes
// (min(|c|,|s|) >= 0.02, i.e. the slope region is >= 0.02 h wide) g comes
// from K2's fixed point and the four weights, normalised by the flat-top
// length (folded into the staged window), are one FFMA.SAT each:
//     w_k / Lm = sat(Q_k -/+ f B),  B = s ics / Lm,  Q_k per angle;
// near-axis angles evaluate g and the trapezoid in fp64 (their slope region
// is ~|sin| h wide, below fp32 resolution of g).  Small images split angles
// over blockIdx.z into partial images reduced in a fixed order.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <vector>

#include "ctk_common.cuh"

namespace ctk {

constexpr int JTX = 32, JROWS = 8, JCA = 32;     // tile JTX x (JROWS * JPPT), JPPT = K2's
constexpr int JTHREADS = JTX * JROWS;
#ifndef CTK_ADJ_FAST_MIN
#define CTK_ADJ_FAST_MIN 0.02
#endif

struct AdjArgs {
    const double* cs;        // [n_angles] bitwise np.cos
    const double* sn;        // [n_angles] bitwise np.sin
    const int* deg_slot;     // [n_angles] -> degenerate slot or -1
    const float* u;          // row a at u + (a - a0) * D
    const float* x0;         // optional
    float* out;              // final image (split == 0) or partials [S][n]
    float* x;                // final image (split)
    unsigned* cnt;           // split: per-tile tickets (zeroed once)
    const long long* dt_ptr; // [n_deg][n + 1] transposed degenerate lists
    const int* dt_ray;
    const float* dt_len;
    const int* deg_angle;    // slot -> angle
    int n_deg;
    int nx, ny, D, a0, a1, per_split, wmax, split, fbits;
    int qm;                  // TAPS == 1: candidates j0 - qm .. j0 + 1 + qm
    double h, sp, xmin, ymax, center;
};

// TAPS: candidate rays per pixel-angle.  With R = max (|c|+|s|) h / (2 s), the
// half-width of a pixel's shadow in bins: 2 (j0, j0+1) when R <= 1, 4
// (j0-1 .. j0+2) when R <= 2 -- the staged window holds, per bin i, the taps
// (u[i], u[i+1]) or (u[i-1] .. u[i+2]) so one LDS.64 / LDS.128 fetches them --
// and 1 for bins narrower than that (s < 0.354 h): a plain window and the
// fp64 trapezoid over j0 - qm .. j0 + 1 + qm, qm = ceil(R) - 1, for every
// angle (no fixed-point fast path).
template <int TAPS>
struct TapT {
    typedef float4 type;
};
template <>
struct TapT<2> {
    typedef float2 type;
};
template <>
struct TapT<1> {
    typedef float type;
};

// Resident CTAs per SM: 6 (40 registers; the few spills sit in the fp64
// near-axis branch).  Unconstrained the kernels take 109 registers (2 CTAs):
// At per apply at c2 / c3 / c4 / c5 0.070 / 0.243 / 1.61 / 7.68 ms against
// 0.045 / 0.182 / 1.27 / 6.02 ms with 6 (4: 0.051 / 0.198 / 1.27 / 6.04).
#ifndef CTK_ADJ_MINB
#define CTK_ADJ_MINB 6
#endif
template <int JPPT, int TAPS>
__global__ void __launch_bounds__(JTHREADS, CTK_ADJ_MINB) k_adjoint(AdjArgs A) {
    constexpr int JTY = JROWS * JPPT;
    typedef typename TapT<TAPS>::type tap_t;
    extern __shared__ __align__(16) unsigned char wraw[];
    tap_t* winq = reinterpret_cast<tap_t*>(wraw);    // [JCA][wmax] taps per window bin
    __shared__ double s_cg[JCA], s_sg[JCA], s_P[JCA], s_Lm[JCA], s_ics[JCA];
    __shared__ int s_w0[JCA], s_skip[JCA];      // skip: 0 fp64 path, 1 K1d, 2 fp32 fixed point
    __shared__ int4 s_fx[JCA];                  // fast path: T0, C, S (fixed point), unused
    __shared__ float4 s_q[JCA];                 // fast path: weight offsets of the 4 candidates
    __shared__ float s_b[JCA];                  //            and slope (weights / Lm)

    const int tx = threadIdx.x, ty = threadIdx.y, tid = ty * JTX + tx;
    const int ix0 = blockIdx.x * JTX, iy0 = blockIdx.y * JTY;
    const int ix = ix0 + tx;
    const double X = A.xmin + ((double)ix + 0.5) * A.h;
    double Y[JPPT];
#pragma unroll
    for (int r = 0; r < JPPT; ++r) Y[r] = A.ymax - ((double)(iy0 + ty + r * JROWS) + 0.5) * A.h;
    const double Xlo = A.xmin + ((double)ix0 + 0.5) * A.h;
    const double Xhi = A.xmin + ((double)(ix0 + JTX - 1) + 0.5) * A.h;
    const double Yhi = A.ymax - ((double)iy0 + 0.5) * A.h;
    const double Ylo = A.ymax - ((double)(iy0 + JTY - 1) + 0.5) * A.h;

    const int aS = A.a0 + blockIdx.z * A.per_split;
    const int aE = min(A.a1, aS + A.per_split);
    const int D = A.D, wmax = A.wmax;
    const double sp = A.sp;
    const int F = A.fbits, I = 32 - A.fbits;

    double acc[JPPT];
#pragma unroll
    for (int r = 0; r < JPPT; ++r) acc[r] = 0.0;
    for (int ac = aS; ac < aE; ac += JCA) {
        const int na = min(JCA, aE - ac);
        if (tid < na) {
            const int a = ac + tid;
            const double c = A.cs[a], s = A.sn[a];
            const double cg = c / sp, sg = s / sp;
            const double ac_ = fabs(c), as_ = fabs(s);
            s_cg[tid] = cg;
            s_sg[tid] = sg;
            s_P[tid] = 0.5 * (ac_ + as_) * A.h;
            s_Lm[tid] = A.h / fmax(ac_, as_);
            s_ics[tid] = ac_ * as_ > 0.0 ? 1.0 / (ac_ * as_) : 0.0;
            const double g00 = fma(Xlo, cg, fma(Ylo, sg, A.center));
            const double g01 = fma(Xlo, cg, fma(Yhi, sg, A.center));
            const double g10 = fma(Xhi, cg, fma(Ylo, sg, A.center));
            const double g11 = fma(Xhi, cg, fma(Yhi, sg, A.center));
            const int w0 = (int)floor(fmin(fmin(g00, g01), fmin(g10, g11))) -
                           (TAPS == 1 ? A.qm + 1 : 2);
            s_w0[tid] = w0;
            // fp32 fixed-point path away from the axes (slope region >= 0.02 h
            // wide): normalised weights sat(Q_k -/+ f B) by FFMA.SAT
            const bool fast = TAPS != 1 && fmin(ac_, as_) >= CTK_ADJ_FAST_MIN;
            s_skip[tid] = A.deg_slot[a] >= 0 ? 1 : (fast ? 2 : 0);
            if (fast) {
                const double scale = ldexp(1.0, A.fbits);
                s_fx[tid] = make_int4((int)(unsigned)llrint((g01 - (double)w0) * scale),
                                      (int)llrint(cg * A.h * scale), (int)llrint(-sg * A.h * scale), 0);
                const double ics = 1.0 / (ac_ * as_), Lm = A.h / fmax(ac_, as_);
                const double A0 = 0.5 * (ac_ + as_) * A.h * ics / Lm, B0 = sp * ics / Lm;
                s_q[tid] = make_float4((float)(A0 - B0), (float)A0, (float)(A0 - B0),
                                       (float)(A0 - 2.0 * B0));
                s_b[tid] = (float)B0;
            }
        }
        __syncthreads();
        for (int ai = ty; ai < na; ai += JROWS) {
            const float* row = A.u + (size_t)(ac + ai - A.a0) * D;
            const int w0 = s_w0[ai];
            tap_t* dst = winq + ai * wmax;
            const float lsc = s_skip[ai] == 2 ? (float)s_Lm[ai] : 1.f;   // fast: pre-scale by Lm
            for (int i = tx; i < wmax; i += JTX) {
                float v4[4];
                constexpr int first = TAPS == 4 ? -1 : 0;
#pragma unroll
                for (int q = 0; q < TAPS; ++q) {
                    const int b = w0 + i + first + q;
                    v4[q] = (b >= 0 && b < D) ? lsc * __ldg(row + b) : 0.f;
                }
                if constexpr (TAPS == 1)
                    dst[i] = v4[0];
                else if constexpr (TAPS == 2)
                    dst[i] = make_float2(v4[0], v4[1]);
                else
                    dst[i] = make_float4(v4[0], v4[1], v4[2], v4[3]);
            }
        }
        __syncthreads();
        float fa[JPPT];
#pragma unroll
        for (int r = 0; r < JPPT; ++r) fa[r] = 0.f;
        for (int ai = 0; ai < na; ++ai) {
            const int mode = s_skip[ai];
            if (mode == 1) continue;                   // K1d angles: transposed lists below
            if (TAPS != 1 && mode == 2) {
                const int4 fx = s_fx[ai];
                const float4 qw = s_q[ai];
                const float bw = s_b[ai];
                const tap_t* wr = winq + ai * wmax;
                const unsigned T0 = (unsigned)fx.x + (unsigned)tx * (unsigned)fx.y +
                                    (unsigned)ty * (unsigned)fx.z;
#pragma unroll
                for (int r = 0; r < JPPT; ++r) {
                    const unsigned T = T0 + (unsigned)(r * JROWS) * (unsigned)fx.z;
                    const int idx = (int)(T >> F);
                    const float f = __uint_as_float(0x3f800000u | ((T << I) >> 9)) - 1.f;
                    const tap_t v = wr[idx];
                    float t = fa[r];
                    // |k - f| for k = -1, 0, 1, 2 is 1 + f, f, 1 - f, 2 - f
                    if constexpr (TAPS == 2) {
                        t = fmaf(__saturatef(fmaf(f, -bw, qw.y)), v.x, t);
                        t = fmaf(__saturatef(fmaf(f, bw, qw.z)), v.y, t);
                    } else if constexpr (TAPS == 4) {
                        t = fmaf(__saturatef(fmaf(f, -bw, qw.x)), v.x, t);
                        t = fmaf(__saturatef(fmaf(f, -bw, qw.y)), v.y, t);
                        t = fmaf(__saturatef(fmaf(f, bw, qw.z)), v.z, t);
                        t = fmaf(__saturatef(fmaf(f, bw, qw.w)), v.w, t);
                    }
                    fa[r] = t;
                }
                continue;
            }
            const double cg = s_cg[ai], sg = s_sg[ai], P = s_P[ai], Lm = s_Lm[ai], ics = s_ics[ai];
            const tap_t* wq = winq + ai * wmax - s_w0[ai];
#pragma unroll
            for (int r = 0; r < JPPT; ++r) {
                const double g = fma(X, cg, fma(Y[r], sg, A.center));   // ray index at the centre
                const int j0 = (int)floor(g);
                const int qlo = TAPS == 1 ? -A.qm : -1, qhi = TAPS == 1 ? A.qm + 1 : 2;
                for (int q = qlo; q <= qhi; ++q) {
                    const int j = j0 + q;
                    const double a = P - fabs((double)j - g) * sp;
                    if (a > 0.0) {
                        float uj;
                        if constexpr (TAPS == 1) uj = wq[j];
                        else if constexpr (TAPS == 2) uj = wq[j].x;
                        else uj = wq[j].y;
                        acc[r] = fma(fmin(Lm, a * ics), (double)uj, acc[r]);
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < JPPT; ++r) acc[r] += (double)fa[r];
        __syncthreads();
    }
    // degenerate angles of this split range: per-pixel transposed lists
    const size_t n = (size_t)A.nx * A.ny;
    for (int sl = 0; sl < A.n_deg; ++sl) {
        const int a = A.deg_angle[sl];
        if (a < aS || a >= aE) continue;
        const float* urow = A.u + (size_t)(a - A.a0) * D;
#pragma unroll
        for (int r = 0; r < JPPT; ++r) {
            const int iy = iy0 + ty + r * JROWS;
            if (ix >= A.nx || iy >= A.ny) continue;
            const size_t p = (size_t)iy * A.nx + ix;
            const long long* pp = A.dt_ptr + (size_t)sl * (n + 1);
            for (long long e = pp[p]; e < pp[p + 1]; ++e)
                acc[r] = fma((double)A.dt_len[e], (double)__ldg(urow + A.dt_ray[e]), acc[r]);
        }
    }
    if (A.split) {
        float* part = A.out;
        const bool inx = ix < A.nx;
#pragma unroll
        for (int r = 0; r < JPPT; ++r) {
            const int iy = iy0 + ty + r * JROWS;
            if (inx && iy < A.ny) part[(size_t)blockIdx.z * n + (size_t)iy * A.nx + ix] = (float)acc[r];
        }
        __syncthreads();
        __shared__ unsigned s_last;
        unsigned* ticket = A.cnt + (size_t)blockIdx.y * gridDim.x + blockIdx.x;
        if (tid == 0) s_last = ctk_ticket_arrive(ticket, gridDim.z);
        __syncthreads();
        if (!s_last) return;
        if (inx) {
            for (int r = 0; r < JPPT; ++r) {
                const int iy = iy0 + ty + r * JROWS;
                if (iy >= A.ny) continue;
                const size_t o = (size_t)iy * A.nx + ix;
                double t = 0.0;
                for (unsigned z = 0; z < gridDim.z; ++z) t += (double)__ldcg(part + z * n + o);
                A.x[o] = (float)((A.x0 ? (double)A.x0[o] : 0.0) + t);
            }
        }
        if (tid == 0) *ticket = 0u;
    } else {
        if (ix >= A.nx) return;
#pragma unroll
        for (int r = 0; r < JPPT; ++r) {
            const int iy = iy0 + ty + r * JROWS;
            if (iy >= A.ny) continue;
            const size_t o = (size_t)iy * A.nx + ix;
            A.out[o] = (float)((A.x0 ? (double)A.x0[o] : 0.0) + acc[r]);
        }
    }
}

static int adj_tiles_y(const ctk_geom* g) {
    const int jty = JROWS * (g->back_ppt == 4 ? 4 : 2);      // the kernels' JPPT
    return (g->ny + jty - 1) / jty;
}

int adj_splits(const ctk_geom* g, int a0, int a1) {
    const int tiles = ((g->nx + JTX - 1) / JTX) * adj_tiles_y(g);
    int S = (148 * 8 + tiles - 1) / tiles;
    const int max_s = (a1 - a0 + JCA - 1) / JCA;
    if (S > max_s) S = max_s;
    return S < 1 ? 1 : S;
}

// Transposed K1d lists (pixel -> (ray, length)), built on the host once per
// geometry in ray order (deterministic summation order).
struct DegT {
    long long* ptr = nullptr;
    int* ray = nullptr;
    float* len = nullptr;
    int* angle = nullptr;
    int n_deg = 0;
};

std::mutex g_degt_mu;

int degt_get(ctk_geom* g, DegT* out) {
    std::lock_guard<std::mutex> lk(g_degt_mu);
    if (g->d_degt_ptr || g->n_degenerate == 0) {
        out->ptr = g->d_degt_ptr;
        out->ray = g->d_degt_ray;
        out->len = g->d_degt_len;
        out->angle = g->d_degt_angle;
        out->n_deg = g->d_degt_ptr ? g->n_degenerate : 0;
        return CTK_OK;
    }
    const int D = g->det_count, nd = g->n_degenerate;
    const size_t n = (size_t)g->nx * g->ny;
    std::vector<int> slot(g->n_angles);
    CTK_CUDA(cudaMemcpy(slot.data(), g->d_deg_slot, sizeof(int) * g->n_angles,
                        cudaMemcpyDeviceToHost));
    std::vector<int> angle(nd, -1);
    for (int a = 0; a < g->n_angles; ++a)
        if (slot[a] >= 0 && slot[a] < nd) angle[slot[a]] = a;
    const size_t rays = (size_t)nd * D;
    const size_t entries = (size_t)nd * g->deg_maxseg * D;
    std::vector<long long> cnt(rays);
    std::vector<int> pix(entries);
    std::vector<float> len(entries);
    CTK_CUDA(cudaMemcpy(cnt.data(), g->d_deg_ptr, sizeof(long long) * rays, cudaMemcpyDeviceToHost));
    CTK_CUDA(cudaMemcpy(pix.data(), g->d_deg_pix, sizeof(int) * entries, cudaMemcpyDeviceToHost));
    CTK_CUDA(cudaMemcpy(len.data(), g->d_deg_len, sizeof(float) * entries, cudaMemcpyDeviceToHost));
    std::vector<long long> ptr((size_t)nd * (n + 1), 0);
    for (int sl = 0; sl < nd; ++sl) {
        long long* P = ptr.data() + (size_t)sl * (n + 1);
        for (int j = 0; j < D; ++j)
            for (long long e = 0; e < cnt[(size_t)sl * D + j]; ++e)
                ++P[(size_t)pix[((size_t)sl * g->deg_maxseg + e) * D + j] + 1];
        for (size_t p = 0; p < n; ++p) P[p + 1] += P[p];
    }
    // global offsets: slot sl's entries follow slot sl-1's
    long long base = 0;
    for (int sl = 0; sl < nd; ++sl) {
        long long* P = ptr.data() + (size_t)sl * (n + 1);
        const long long tot = P[n];
        for (size_t p = 0; p <= n; ++p) P[p] += base;
        base += tot;
    }
    std::vector<int> tray(base > 0 ? base : 1);
    std::vector<float> tlen(base > 0 ? base : 1);
    std::vector<long long> fill(ptr);
    for (int sl = 0; sl < nd; ++sl) {
        long long* F = fill.data() + (size_t)sl * (n + 1);
        for (int j = 0; j < D; ++j)
            for (long long e = 0; e < cnt[(size_t)sl * D + j]; ++e) {
                const size_t idx = ((size_t)sl * g->deg_maxseg + e) * D + j;
                const long long at = F[pix[idx]]++;
                tray[at] = j;
                tlen[at] = len[idx];
            }
    }
    cudaError_t e = cudaMalloc(&g->d_degt_ptr, sizeof(long long) * ptr.size());
    if (e == cudaSuccess) e = cudaMalloc(&g->d_degt_ray, sizeof(int) * tray.size());
    if (e == cudaSuccess) e = cudaMalloc(&g->d_degt_len, sizeof(float) * tlen.size());
    if (e == cudaSuccess) e = cudaMalloc(&g->d_degt_angle, sizeof(int) * nd);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_degt_ptr, ptr.data(), sizeof(long long) * ptr.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_degt_ray, tray.data(), sizeof(int) * tray.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_degt_len, tlen.data(), sizeof(float) * tlen.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_degt_angle, angle.data(), sizeof(int) * nd, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) return ctk_check_cuda(e, "transposed degenerate lists");
    out->ptr = g->d_degt_ptr;
    out->ray = g->d_degt_ray;
    out->len = g->d_degt_len;
    out->angle = g->d_degt_angle;
    out->n_deg = nd;
    return CTK_OK;
}

}  // namespace ctk

using namespace ctk;

// Work buffer (split launches): [one arrival ticket per tile, 16-float
// aligned] [S partial images] -- the tickets at a fixed offset, so calls with
// different split counts sharing one zero-filled buffer agree on them.
static int64_t adj_ticket_floats(const ctk_geom* g) {
    const int64_t tiles = (int64_t)((g->nx + JTX - 1) / JTX) * adj_tiles_y(g);
    return (tiles + 15) / 16 * 16;
}

extern "C" int64_t ctk_adjoint_work_floats(const ctk_geom_t* g, int a0, int a1) {
    if (!g || a0 < 0 || a1 > g->n_angles || a0 >= a1) return 0;
    const int S = adj_splits(g, a0, a1);
    return S > 1 ? adj_ticket_floats(g) + (int64_t)S * g->nx * g->ny : 0;
}

extern "C" int ctk_adjoint(const ctk_geom_t* gc, const float* u, float* x, int a0, int a1,
                           const float* x0, float* work, void* stream) {
    ctk_geom* g = const_cast<ctk_geom*>(gc);
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
    DegT dt;
    int rc = degt_get(g, &dt);
    if (rc) return rc;
    const int S = adj_splits(g, a0, a1);
    if (S > 1 && !work)
        return ctk_fail(CTK_ERR_ARG, "ctk_adjoint needs %lld work floats",
                        (long long)ctk_adjoint_work_floats(g, a0, a1));
    AdjArgs A;
    A.cs = g->d_cos;
    A.sn = g->d_sin;
    A.deg_slot = g->d_deg_slot;
    A.u = u;
    A.x0 = x0;
    A.out = S > 1 ? work + adj_ticket_floats(g) : x;
    A.x = x;
    A.cnt = S > 1 ? reinterpret_cast<unsigned*>(work) : nullptr;
    A.dt_ptr = dt.ptr;
    A.dt_ray = dt.ray;
    A.dt_len = dt.len;
    A.deg_angle = dt.angle;
    A.n_deg = dt.n_deg;
    A.nx = g->nx;
    A.ny = g->ny;
    A.D = g->det_count;
    A.a0 = a0;
    A.a1 = a1;
    A.per_split = (a1 - a0 + S - 1) / S;
    // Candidates and window.  R: half-width of a pixel's shadow in bins, at
    // most h / (sqrt 2 s); the window must hold this kernel's own tile
    // (32 x 8 JPPT pixels: K2's bound is for K2's tile, which is half as tall
    // for small images) plus the candidates' margins on both sides.
    const int jppt = g->back_ppt == 4 ? 4 : 2;
    const double rmax = 0.5 * 1.41421356237309515 * g->h / g->det_spacing;
    static int force4 = -1;
    if (force4 < 0) {
        const char* e = getenv("CTK_ADJ_TAPS4");          // test hook: the 4-tap path
        force4 = e && e[0] == '1';
    }
    const int taps = rmax > 2.0 - 1e-9 ? 1 : (!force4 && rmax <= 1.0) ? 2 : 4;
    A.qm = taps == 1 ? (int)ceil(rmax) - 1 : 1;
    A.wmax = (int)ceil(sqrt((double)JTX * JTX + (double)(JROWS * jppt) * (JROWS * jppt)) * g->h /
                       g->det_spacing) + 2 * (A.qm + 1) + 3;
    {   // fixed-point fraction bits: window coordinates [0, wmax] need I bits
        int I = 1;
        while ((1 << I) <= A.wmax + 1) ++I;
        A.fbits = 32 - I;
    }
    A.split = S > 1;
    A.h = g->h;
    A.sp = g->det_spacing;
    A.xmin = g->xmin;
    A.ymax = g->ymax;
    A.center = g->center;
    dim3 grid((g->nx + JTX - 1) / JTX, adj_tiles_y(g), S), block(JTX, JROWS);
    const size_t smem = (size_t)JCA * A.wmax *
                        (taps == 1 ? sizeof(float) : taps == 2 ? sizeof(float2) : sizeof(float4));
    if (smem > 200 * 1024)
        return ctk_fail(CTK_ERR_GEOMETRY, "adjoint: detector windows of %d bins per tile do not fit "
                        "in shared memory (pixel size %g, bin spacing %g)", A.wmax, g->h,
                        g->det_spacing);
    const bool p4 = g->back_ppt == 4;
    auto kern = p4 ? (taps == 1 ? k_adjoint<4, 1> : taps == 2 ? k_adjoint<4, 2> : k_adjoint<4, 4>)
                   : (taps == 1 ? k_adjoint<2, 1> : taps == 2 ? k_adjoint<2, 2> : k_adjoint<2, 4>);
    // Opt in early (the 48 KB default also counts the static arrays) and always
    // to the same value, the largest window any geometry may have: the limit
    // is per function, so concurrent launches for geometries with different
    // window sizes must not lower it under each other.
    if (smem > 40 * 1024)
        CTK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
    kern<<<grid, block, smem, st>>>(A);
    CTK_LAUNCH_CHECK("k_adjoint");
    return CTK_OK;
}
