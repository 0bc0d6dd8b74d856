// ctk_forward.cu -- K1 / K1d / K6: the Siddon forward projector A on sm_100a.
//
// Reference semantics: ctkrylov/ct.py:137-201 (exact ray/pixel intersection
// lengths, pixel chosen by the segment midpoint, segments <= 1e-15 dropped).
//
// K1 (generic angles) restates Siddon as a row walk.  For a ray whose walk
// axis is the image row (|cos| >= |sin|) the cross coordinate advances by
// sigma = |tan| <= 1 pixel per row, so each row holds one segment, or two
// split at one vertical grid line.  The walk keeps the cross coordinate in
// 32.32 fixed point (integer adds, no division, no fp64 in the loop):
//     c = floor(u), f = frac(u); crossing iff floor(u + sigma) != c
//     w_c = crossing ? (1 - f) * Lx : L,  w_{c+1} = L - w_c
// which are the reference's segment lengths up to ~1e-7 relative (fp32
// weights).  Near-horizontal rays walk the columns of a transposed copy, so
// every gather of a warp (32 adjacent bins of one angle) touches 2-3 adjacent
// 32-B sectors of one image row.  Both copies carry a one-pixel zero border so
// rays entering/leaving through the side need no masks.
//
// K1d: angles the reference treats as axis-aligned (|sin| or |cos| < 1e-14,
// ct.py:153-155,165,168) are traced by a literal fp64 emulation of
// _siddon_ray with explicit round-to-nearest intrinsics (no FMA contraction),
// because there a whole ray lies on a grid line and the reference's
// midpoint/floor/clip sequence decides which column or row receives it.
#include <math.h>

#include "ctk_common.cuh"

namespace ctk {

struct ExactGrid {
    int nx, ny;
    double h, xmin, xmax, ymin, ymax;
};

// Literal restatement of _siddon_ray (ct.py:137-179) in strict IEEE fp64.
// Calls sink(pixel, length) for every kept segment in increasing t.
template <class Sink>
__device__ __forceinline__ void trace_exact(const ExactGrid& g, double ct, double st, double off,
                                            Sink& sink) {
    const double px = __dmul_rn(off, ct), py = __dmul_rn(off, st);
    const double dx = -st, dy = ct;
    double t_lo = -INFINITY, t_hi = INFINITY;
    // x slab
    if (fabs(dx) < 1e-14) {
        if (px < g.xmin || px > g.xmax) return;
    } else {
        double t0 = __ddiv_rn(__dsub_rn(g.xmin, px), dx);
        double t1 = __ddiv_rn(__dsub_rn(g.xmax, px), dx);
        if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
        if (t0 > t_lo) t_lo = t0;
        if (t1 < t_hi) t_hi = t1;
    }
    // y slab
    if (fabs(dy) < 1e-14) {
        if (py < g.ymin || py > g.ymax) return;
    } else {
        double t0 = __ddiv_rn(__dsub_rn(g.ymin, py), dy);
        double t1 = __ddiv_rn(__dsub_rn(g.ymax, py), dy);
        if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
        if (t0 > t_lo) t_lo = t0;
        if (t1 < t_hi) t_hi = t1;
    }
    if (t_hi <= t_lo) return;

    const bool use_x = fabs(dx) >= 1e-14, use_y = fabs(dy) >= 1e-14;
    const int nxi = use_x ? g.nx + 1 : 0, nyi = use_y ? g.ny + 1 : 0;
    int ix_i = (use_x && dx < 0) ? g.nx : 0, ix_s = (use_x && dx < 0) ? -1 : 1;
    int iy_i = (use_y && dy < 0) ? g.ny : 0, iy_s = (use_y && dy < 0) ? -1 : 1;
    int kx = 0, ky = 0;
    double prev = t_lo;
    auto emit = [&](double t_next) {
        const double len = __dsub_rn(t_next, prev);
        const double tm = __dmul_rn(0.5, __dadd_rn(prev, t_next));
        const double fx = floor(__ddiv_rn(__dsub_rn(__dadd_rn(px, __dmul_rn(tm, dx)), g.xmin), g.h));
        const double fy = floor(__ddiv_rn(__dsub_rn(g.ymax, __dadd_rn(py, __dmul_rn(tm, dy))), g.h));
        long long ix = (long long)fx, iy = (long long)fy;
        ix = ix < 0 ? 0 : (ix > g.nx - 1 ? g.nx - 1 : ix);
        iy = iy < 0 ? 0 : (iy > g.ny - 1 ? g.ny - 1 : iy);
        if (len > 1e-15) sink(iy * g.nx + ix, len);
        prev = t_next;
    };
    double tx = INFINITY, ty = INFINITY;
    bool have_x = false, have_y = false;
    for (;;) {
        while (!have_x && kx < nxi) {
            double v = __ddiv_rn(__dsub_rn(__dadd_rn(g.xmin, __dmul_rn((double)ix_i, g.h)), px), dx);
            if (v > t_lo && v < t_hi) { tx = v; have_x = true; } else { ix_i += ix_s; ++kx; }
        }
        while (!have_y && ky < nyi) {
            double v = __ddiv_rn(__dsub_rn(__dadd_rn(g.ymin, __dmul_rn((double)iy_i, g.h)), py), dy);
            if (v > t_lo && v < t_hi) { ty = v; have_y = true; } else { iy_i += iy_s; ++ky; }
        }
        if (!have_x && !have_y) break;
        double v;
        if (have_x && (!have_y || tx <= ty)) {
            v = tx; have_x = false; ix_i += ix_s; ++kx;
        } else {
            v = ty; have_y = false; iy_i += iy_s; ++ky;
        }
        if (v != prev) emit(v);     // np.unique: exact duplicates collapse
    }
    if (t_hi != prev) emit(t_hi);
}

struct SumSink {
    const float* x;
    double acc;
    __device__ void operator()(long long pix, double len) { acc += len * (double)__ldg(x + pix); }
};

struct CountSink {
    long long raw = 0, nnz = 0, last = -1;
    __device__ void operator()(long long pix, double) {
        ++raw;
        if (pix != last) ++nnz;   // identical (ray, pixel) pairs are consecutive
        last = pix;
    }
};

// ---- K1 staging: zero-bordered row-major copy P and transposed copy PT ----
// P : ny rows x (nx+2), P[iy][ix+1]  = x[iy][ix]
// PT: nx rows x (ny+2), PT[ix][iy+1] = x[iy][ix]
__global__ void __launch_bounds__(256) k_stage(const float* __restrict__ x, float* __restrict__ P,
                                               float* __restrict__ PT, int nx, int ny) {
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    const int pP = nx + 2, pT = ny + 2;
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        int iy = by + r, ix = bx + tx;
        float v = (iy < ny && ix < nx) ? x[(size_t)iy * nx + ix] : 0.f;
        tile[r][tx] = v;
        if (iy < ny && ix < nx) P[(size_t)iy * pP + ix + 1] = v;
    }
    // zero borders owned by edge tiles
    if (blockIdx.x == 0) {
        for (int r = ty * 32 + tx; r < 32; r += 256) {
            int iy = by + r;
            if (iy < ny) P[(size_t)iy * pP] = 0.f;
        }
    }
    if (blockIdx.x == gridDim.x - 1) {
        for (int r = ty * 32 + tx; r < 32; r += 256) {
            int iy = by + r;
            if (iy < ny) P[(size_t)iy * pP + nx + 1] = 0.f;
        }
    }
    if (blockIdx.y == 0) {
        for (int r = ty * 32 + tx; r < 32; r += 256) {
            int ix = bx + r;
            if (ix < nx) PT[(size_t)ix * pT] = 0.f;
        }
    }
    if (blockIdx.y == gridDim.y - 1) {
        for (int r = ty * 32 + tx; r < 32; r += 256) {
            int ix = bx + r;
            if (ix < nx) PT[(size_t)ix * pT + ny + 1] = 0.f;
        }
    }
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        int ix = bx + r, iy = by + tx;
        if (ix < nx && iy < ny) PT[(size_t)ix * pT + iy + 1] = tile[tx][r];
    }
}

constexpr int FWD_THREADS = 128;

struct FwdArgs {
    const AngleParams* ap;
    const double* offsets;
    const double* cos_tab;
    const double* sin_tab;
    const float* x;    // original image (exact path)
    const float* P;
    const float* PT;
    const float* b;    // optional: y = b - A x
    float* y;
    ExactGrid eg;
    int D, a0;
    int all_exact;
};

// Row walk of one ray.  Returns sum of segment length * pixel value.
__device__ __forceinline__ double walk_ray(const AngleParams& p, double s, const float* __restrict__ base,
                                           int R, int C) {
    const double sigma = (double)p.sigma_fx * (1.0 / 4294967296.0);
    double u0 = fma(p.beta, s, p.alpha);
    // the ray meets the image iff u(k) in (0, C) for some k in [0, R]
    if (!(u0 < (double)C + 1.0) || !(u0 + (double)R * sigma > -1.0)) return 0.0;
    const long long Sg = p.sigma_fx;
    const long long U0 = llrint(u0 * 4294967296.0);
    const long long C2 = (long long)C << 32;
    // rows k with u(k+1) > 0 and u(k) < C  (=> floor(u(k)) in [-1, C-1])
    long long kb, ke;
    if (U0 + Sg > 0) kb = 0;
    else if (Sg == 0) return 0.0;
    else kb = (-U0) / Sg;                       // smallest k with U0 + (k+1) Sg > 0
    if (U0 >= C2) return 0.0;
    if (Sg == 0) ke = R;
    else ke = (C2 - U0 + Sg - 1) / Sg;          // smallest k with U0 + k Sg >= C
    if (kb < 0) kb = 0;
    if (ke > R) ke = R;
    if (kb >= ke) return 0.0;

    const int pitch = C + 2;
    const int dir = p.mirror ? -1 : 1;
    const float* rowp = base + (size_t)kb * pitch + (p.mirror ? C : 1);
    long long u = U0 + kb * Sg;
    const float L = p.L, Lx = p.Lx;
    double acc = 0.0;
    int k = (int)kb;
    const int kend = (int)ke;
    while (k < kend) {
        const int kstop = min(kend, k + 64);
        float a32 = 0.f;
#pragma unroll 4
        for (; k < kstop; ++k) {
            const int c = (int)(u >> 32);
            const float f = (float)(unsigned)(u & 0xffffffffll) * 2.3283064365386963e-10f;
            const long long un = u + Sg;
            const bool cross = (int)(un >> 32) != c;
            const float wa = cross ? (1.f - f) * Lx : L;
            const float wb = L - wa;
            const float* pp = rowp + dir * c;
            const float v0 = __ldg(pp);
            const float v1 = __ldg(pp + dir);
            a32 = fmaf(wa, v0, fmaf(wb, v1, a32));
            u = un;
            rowp += pitch;
        }
        acc += (double)a32;
    }
    return acc;
}

__global__ void __launch_bounds__(FWD_THREADS) k_forward(FwdArgs A) {
    const int a = A.a0 + blockIdx.y;
    const int j = blockIdx.x * FWD_THREADS + threadIdx.x;
    if (j >= A.D) return;
    const AngleParams p = A.ap[a];
    const double s = A.offsets[j];
    double acc;
    if (p.degenerate || A.all_exact) {
        SumSink sink{A.x, 0.0};
        trace_exact(A.eg, A.cos_tab[a], A.sin_tab[a], s, sink);
        acc = sink.acc;
    } else if (p.frame == 0) {
        acc = walk_ray(p, s, A.P, A.eg.ny, A.eg.nx);
    } else {
        acc = walk_ray(p, s, A.PT, A.eg.nx, A.eg.ny);
    }
    const size_t o = (size_t)blockIdx.y * A.D + j;
    float r = (float)acc;
    if (A.b) r = (float)((double)A.b[o] - acc);
    A.y[o] = r;
}

__global__ void __launch_bounds__(FWD_THREADS) k_count(FwdArgs A, unsigned long long* counts) {
    const int a = A.a0 + blockIdx.y;
    const int j = blockIdx.x * FWD_THREADS + threadIdx.x;
    long long raw = 0, nnz = 0;
    if (j < A.D) {
        CountSink sink;
        trace_exact(A.eg, A.cos_tab[a], A.sin_tab[a], A.offsets[j], sink);
        raw = sink.raw;
        nnz = sink.nnz;
    }
    // warp reduce then one integer atomic per warp (integer: order-free)
    for (int o = 16; o > 0; o >>= 1) {
        raw += __shfl_down_sync(0xffffffffu, raw, o);
        nnz += __shfl_down_sync(0xffffffffu, nnz, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(counts, (unsigned long long)raw);
        atomicAdd(counts + 1, (unsigned long long)nnz);
    }
}

static FwdArgs make_args(const ctk_geom* g, const float* x, float* y, int a0, const float* b) {
    FwdArgs A;
    A.ap = g->d_ap;
    A.offsets = g->d_offsets;
    A.cos_tab = g->d_cos;
    A.sin_tab = g->d_sin;
    A.x = x;
    A.P = nullptr;
    A.PT = nullptr;
    A.b = b;
    A.y = y;
    A.eg = ExactGrid{g->nx, g->ny, g->h, g->xmin, g->xmax, g->ymin, g->ymax};
    A.D = g->det_count;
    A.a0 = a0;
    A.all_exact = 0;
    return A;
}

}  // namespace ctk

using namespace ctk;

static int check_range(const ctk_geom* g, int a0, int a1) {
    if (!g) return ctk_fail(CTK_ERR_ARG, "null geometry");
    if (a0 < 0 || a1 > g->n_angles || a0 > a1)
        return ctk_fail(CTK_ERR_SHAPE, "angle range [%d, %d) outside [0, %d)", a0, a1, g->n_angles);
    return CTK_OK;
}

extern "C" int ctk_forward(const ctk_geom_t* g, const float* x, float* y, int a0, int a1,
                           const float* b, float* work, void* stream) {
    int rc = check_range(g, a0, a1);
    if (rc) return rc;
    if (!x || !y) return ctk_fail(CTK_ERR_ARG, "null vector");
    if (a1 == a0) return CTK_OK;
    if (!work) return ctk_fail(CTK_ERR_ARG, "ctk_forward needs a stage work buffer");
    CTK_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = ctk_stream(stream);
    float* P = work;
    float* PT = work + (size_t)g->ny * (g->nx + 2);
    dim3 sg((g->nx + 31) / 32, (g->ny + 31) / 32), sb(32, 8);
    k_stage<<<sg, sb, 0, st>>>(x, P, PT, g->nx, g->ny);
    CTK_LAUNCH_CHECK("k_stage");
    FwdArgs A = make_args(g, x, y, a0, b);
    A.P = P;
    A.PT = PT;
    dim3 grid((g->det_count + FWD_THREADS - 1) / FWD_THREADS, a1 - a0);
    k_forward<<<grid, FWD_THREADS, 0, st>>>(A);
    CTK_LAUNCH_CHECK("k_forward");
    return CTK_OK;
}

extern "C" int ctk_forward_exact(const ctk_geom_t* g, const float* x, float* y, int a0, int a1,
                                 void* stream) {
    int rc = check_range(g, a0, a1);
    if (rc) return rc;
    if (!x || !y) return ctk_fail(CTK_ERR_ARG, "null vector");
    if (a1 == a0) return CTK_OK;
    CTK_CUDA(cudaSetDevice(g->device));
    FwdArgs A = make_args(g, x, y, a0, nullptr);
    A.all_exact = 1;
    dim3 grid((g->det_count + FWD_THREADS - 1) / FWD_THREADS, a1 - a0);
    k_forward<<<grid, FWD_THREADS, 0, ctk_stream(stream)>>>(A);
    CTK_LAUNCH_CHECK("k_forward(exact)");
    return CTK_OK;
}

extern "C" int ctk_count_segments(const ctk_geom_t* g, int a0, int a1, int64_t* counts_dev,
                                  void* stream) {
    int rc = check_range(g, a0, a1);
    if (rc) return rc;
    if (!counts_dev) return ctk_fail(CTK_ERR_ARG, "null counts");
    CTK_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = ctk_stream(stream);
    CTK_CUDA(cudaMemsetAsync(counts_dev, 0, 2 * sizeof(int64_t), st));
    if (a1 == a0) return CTK_OK;
    FwdArgs A = make_args(g, nullptr, nullptr, a0, nullptr);
    dim3 grid((g->det_count + FWD_THREADS - 1) / FWD_THREADS, a1 - a0);
    k_count<<<grid, FWD_THREADS, 0, st>>>(A, reinterpret_cast<unsigned long long*>(counts_dev));
    CTK_LAUNCH_CHECK("k_count");
    return CTK_OK;
}
