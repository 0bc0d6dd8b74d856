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
// That trace runs once, at geometry creation, into per-ray segment lists;
// an apply sums them warp-per-ray inside the same launch as K1.
#include <cooperative_groups.h>
#include <math.h>

#include <vector>

#include "ctk_common.cuh"

namespace ctk {

struct ExactGrid {
    int nx, ny;
    double h, xmin, xmax, ymin, ymax;
    double inv_h;
    int h_pow2;
};

// IEEE a / b.  When |b| is a power of two, a * (1/b) is the same double
// (both are exact scalings), and avoids the long fp64 division sequence --
// this is the common case on the degenerate angles (dx = -1, dy = 1) and for
// unit pixels.
__device__ __forceinline__ double xdiv(double a, double b, double inv_b, bool pow2) {
    return pow2 ? __dmul_rn(a, inv_b) : __ddiv_rn(a, b);
}

// Literal restatement of _siddon_ray (ct.py:137-179) in strict IEEE fp64.
// Calls sink(pixel, length) for every kept segment in increasing t.
template <class Sink>
__device__ __forceinline__ void trace_exact(const ExactGrid& g, double ct, double st, double off,
                                            const AngleParams& p, Sink& sink) {
    const double px = __dmul_rn(off, ct), py = __dmul_rn(off, st);
    const double dx = -st, dy = ct;
    const bool xp2 = p.exact_flags & 1, yp2 = (p.exact_flags >> 1) & 1, hp2 = g.h_pow2;
    const double idx = p.inv_dx, idy = p.inv_dy, ih = g.inv_h;
    double t_lo = -INFINITY, t_hi = INFINITY;
    // x slab
    if (fabs(dx) < 1e-14) {
        if (px < g.xmin || px > g.xmax) return;
    } else {
        double t0 = xdiv(__dsub_rn(g.xmin, px), dx, idx, xp2);
        double t1 = xdiv(__dsub_rn(g.xmax, px), dx, idx, xp2);
        if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
        if (t0 > t_lo) t_lo = t0;
        if (t1 < t_hi) t_hi = t1;
    }
    // y slab
    if (fabs(dy) < 1e-14) {
        if (py < g.ymin || py > g.ymax) return;
    } else {
        double t0 = xdiv(__dsub_rn(g.ymin, py), dy, idy, yp2);
        double t1 = xdiv(__dsub_rn(g.ymax, py), dy, idy, yp2);
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
        const double fx = floor(xdiv(__dsub_rn(__dadd_rn(px, __dmul_rn(tm, dx)), g.xmin), g.h, ih, hp2));
        const double fy = floor(xdiv(__dsub_rn(g.ymax, __dadd_rn(py, __dmul_rn(tm, dy))), g.h, ih, hp2));
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
            double v = xdiv(__dsub_rn(__dadd_rn(g.xmin, __dmul_rn((double)ix_i, g.h)), px), dx, idx, xp2);
            if (v > t_lo && v < t_hi) { tx = v; have_x = true; } else { ix_i += ix_s; ++kx; }
        }
        while (!have_y && ky < nyi) {
            double v = xdiv(__dsub_rn(__dadd_rn(g.ymin, __dmul_rn((double)iy_i, g.h)), py), dy, idy, yp2);
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

struct FillSink {          // segment i of a ray -> entry i * stride of its column
    int* pix;
    float* len;
    long long i;
    long long stride;
    __device__ void operator()(long long p, double l) {
        pix[i] = (int)p;
        len[i] = (float)l;
        i += stride;
    }
};

// ---- K1 staging: zero-padded row-major copy P and transposed copy PT ----
// P : ny rows x (nx + 2 pad), P[iy][ix + pad]  = x[iy][ix]
// PT: nx rows x (ny + 2 pad), PT[ix][iy + pad] = x[iy][ix]
__global__ void __launch_bounds__(256) k_stage(const float* __restrict__ x, float* __restrict__ P,
                                               float* __restrict__ PT, int nx, int ny, int pad) {
    ctk_pdl_trigger();
    __shared__ float tile[32][33];
    const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;   // 32 x 8
    const int tid = ty * 32 + tx;
    const int pP = nx + 2 * pad, pT = ny + 2 * pad;
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        int iy = by + r, ix = bx + tx;
        float v = (iy < ny && ix < nx) ? x[(size_t)iy * nx + ix] : 0.f;
        tile[r][tx] = v;
        if (iy < ny && ix < nx) P[(size_t)iy * pP + ix + pad] = v;
    }
    // zero padding owned by the edge tiles
    if (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1) {
        const int c0 = blockIdx.x == 0 ? 0 : nx + pad;
        for (int e = tid; e < 32 * pad; e += 256) {
            const int iy = by + e / pad;
            if (iy < ny) P[(size_t)iy * pP + c0 + e % pad] = 0.f;
        }
        if (gridDim.x == 1)
            for (int e = tid; e < 32 * pad; e += 256) {
                const int iy = by + e / pad;
                if (iy < ny) P[(size_t)iy * pP + nx + pad + e % pad] = 0.f;
            }
    }
    if (blockIdx.y == 0 || blockIdx.y == gridDim.y - 1) {
        const int c0 = blockIdx.y == 0 ? 0 : ny + pad;
        for (int e = tid; e < 32 * pad; e += 256) {
            const int ix = bx + e / pad;
            if (ix < nx) PT[(size_t)ix * pT + c0 + e % pad] = 0.f;
        }
        if (gridDim.y == 1)
            for (int e = tid; e < 32 * pad; e += 256) {
                const int ix = bx + e / pad;
                if (ix < nx) PT[(size_t)ix * pT + ny + pad + e % pad] = 0.f;
            }
    }
    __syncthreads();
#pragma unroll
    for (int r = ty; r < 32; r += 8) {
        int ix = bx + r, iy = by + tx;
        if (ix < nx && iy < ny) PT[(size_t)ix * pT + iy + pad] = tile[tx][r];
    }
}

constexpr int FWD_THREADS = 32 * CTK_FWD_APB;
#ifndef CTK_FWD_UNROLL
#define CTK_FWD_UNROLL 16
#endif
constexpr int FWD_UNROLL = CTK_FWD_UNROLL;     // rows per unrolled batch of the walk

struct FwdArgs {
    const AngleParams* ap;
    const double* offsets;
    const double* cos_tab;
    const double* sin_tab;
    const float* x;          // original image (degenerate lists / exact path)
    const float* P;          // zero-bordered row-major copy
    const float* PT;         // zero-bordered transposed copy
    const float* b;          // optional: y = b - A x
    float* y;
    int split;               // row chunks per ray (blockIdx.z), small-problem parallelism
    const int* deg_slot;
    const long long* deg_cnt;   // segments per degenerate ray [slot * D + j]
    const int* deg_pix;         // [slot][maxseg][D]: ray-interleaved, coalesced per warp
    const float* deg_len;
    int deg_maxseg;
    ExactGrid eg;
    int D, a0, a1, pad;
    unsigned* done;          // optional: per 4-angle group, finished CTAs (K2 chaining)
    int pair;                // warp = 2 angles x 16 bins (else 1 angle x 32 bins)
};

// One ray of the row walk (see the header comment).  base/pitch/C describe
// the zero-padded copy the ray walks; MIRROR reverses the cross axis.
//
// The lanes of a warp (32 adjacent bins of one angle) walk the SAME rows in
// lockstep: each lane's own row range [kb, ke) is widened to the warp's
// union [kw, kW), and outside its range a lane's taps fall into the zero
// padding (pad >= the cross-axis spread of the warp's rays, set at geometry
// creation), so they add exact zeros and need no predicate.  Rays entering
// through the side of the image otherwise start on different rows, which
// turns each warp gather into ~10 scattered sectors instead of 2-3.
// One row step.  frac += sigma; the carry moves the pair one column:
// q += pitch + carry.  MIRROR (the pair's second tap is to the LEFT) keeps
// fr = ~frac instead: fr -= sigma borrows exactly when frac + sigma carries,
// and the carry flag after a subtract is "no borrow", so
// q += (pitch - 1) + !borrow = pitch - carry.  Both are two integer ops.
template <bool MIRROR>
__device__ __forceinline__ void walk_step(unsigned& fr, int& q, unsigned Sf, int pitch) {
    if (MIRROR)
        asm("sub.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;"
            : "+r"(fr), "+r"(q) : "r"(Sf), "r"(pitch - 1));
    else
        asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;"
            : "+r"(fr), "+r"(q) : "r"(Sf), "r"(pitch));
}

// Second-tap weight from the step state: w = sat(f + sigma - 1) with
// f1 = 1 + f from the top fraction bits (no I2F); MIRROR holds ~frac, i.e.
// f' = 1 - f - 2^-32, so w = sat((sigma + 1) - (1 + f')) (free negation).
template <bool MIRROR>
__device__ __forceinline__ float walk_weight(unsigned fr, float sm2, float sp1) {
    const float f1 = __uint_as_float(0x3f800000u | (fr >> 9));
    return MIRROR ? __saturatef(sp1 - f1) : __saturatef(f1 + sm2);
}

template <bool MIRROR>
__device__ __forceinline__ double walk_ray(const AngleParams& p, double s,
                                           const float* __restrict__ base, int R, int C, int pad,
                                           int krow0, int krow1) {
    const double sigma = (double)p.sigma_fx * (1.0 / 4294967296.0);
    const double u0 = fma(p.beta, s, p.alpha);
    const long long Sg = p.sigma_fx;
    const long long U0 = llrint(u0 * 4294967296.0);
    const long long C2 = (long long)C << 32;
    // the ray meets the image iff u(k) in (0, C) for some k in [0, R]
    bool hit = (u0 < (double)C + 1.0) && (u0 + (double)R * sigma > -1.0) && U0 < C2;
    // rows k with u(k+1) > 0 and u(k) < C  (=> floor(u(k)) in [-1, C-1])
    // fp64 estimates of the integer quotients, then exact integer fix-ups
    // (cheaper than two 64-bit integer divisions per ray)
    long long kb = 0, ke = R;
    if (hit) {
        if (U0 + Sg <= 0) {
            if (Sg == 0) {
                hit = false;
            } else {
                kb = (long long)floor((double)(-U0) * p.inv_sg);   // smallest k: U0 + (k+1) Sg > 0
                while (U0 + (kb + 1) * Sg <= 0) ++kb;
                while (kb > 0 && U0 + kb * Sg > 0) --kb;
            }
        }
        if (Sg != 0) {
            ke = (long long)ceil((double)(C2 - U0) * p.inv_sg);    // smallest k: U0 + k Sg >= C
            while (U0 + ke * Sg < C2) ++ke;
            while (ke > 0 && U0 + (ke - 1) * Sg >= C2) --ke;
        }
        if (kb < krow0) kb = krow0;           // this block's row chunk only
        if (ke > krow1) ke = krow1;
        if (kb >= ke) hit = false;
    }
    const unsigned lanes = __activemask();
    const int kw = __reduce_min_sync(lanes, hit ? (int)kb : 0x7fffffff);
    const int kW = __reduce_max_sync(lanes, hit ? (int)ke : (int)0x80000000);
    if (!hit) return 0.0;
    ctk_pdl_wait();                                  // P / PT come from the previous kernel

    const int pitch = C + 2 * pad;
    // sigma < 1 here (the host clamps sigma_fx below 2^32), so the cross
    // coordinate is (column c, 32-bit fraction) and a row splits exactly when
    // the fraction add carries.  q = flat index of the pair's first tap:
    // row k, padded column c + pad (MIRROR: padded column C - 1 - c + pad,
    // second tap one to the left).
    const long long u = U0 + (long long)kw * Sg;
    unsigned frac = MIRROR ? ~(unsigned)u : (unsigned)u;      // see walk_step
    const unsigned Sf = (unsigned)Sg;
    const int c0 = (int)(u >> 32);
    // the carry moves the pair one column right (MIRROR: left: subtract it)
    int q = kw * pitch + (MIRROR ? C - 1 - c0 + pad : c0 + pad);
    // Second-tap length wb = max(0, f + sigma - 1) * Lx, the part of the row
    // past the grid line (0 when it does not reach it), and wa = L - wb, so
    //   wa v0 + wb v1 = L v0 + Lx w (v1 - v0),  w = sat(f1 + (sigma - 2)),
    // f1 = 1 + f (w < sigma <= 1: the saturation only clamps at 0).  Per row:
    // frac add + carry, address, two taps, 1 + f, FADD.SAT, and the two sums.
    const float sm2 = (float)((double)Sg * (1.0 / 4294967296.0) - 2.0);
    const float sp1 = (float)((double)Sg * (1.0 / 4294967296.0) + 1.0);
    double acc = 0.0;
    int k = kw;
#ifndef CTK_FWD_PAIRED
#define CTK_FWD_PAIRED 1
#endif
    while (k < kW) {
        const int kstop = min(kW, k + 48);
        float s0 = 0.f, s1 = 0.f;
        if (CTK_FWD_PAIRED) {
            // two rows per step in packed fp32x2 (FADD2 / FFMA2): rows k, k+1
            // share one add for the v0 sums, one for the differences and one
            // FMA for the weighted sums.
            float2 S0 = make_float2(0.f, 0.f), S1 = make_float2(0.f, 0.f);
            const float2 m1 = make_float2(-1.f, -1.f);
#pragma unroll FWD_UNROLL / 2
            for (; k + 1 < kstop; k += 2) {
                float2 v0, v1, w;
                {
                    w.x = walk_weight<MIRROR>(frac, sm2, sp1);
                    const float* pp = base + q;
                    v0.x = __ldg(pp);
                    v1.x = __ldg(pp + (MIRROR ? -1 : 1));
                    walk_step<MIRROR>(frac, q, Sf, pitch);
                }
                {
                    w.y = walk_weight<MIRROR>(frac, sm2, sp1);
                    const float* pp = base + q;
                    v0.y = __ldg(pp);
                    v1.y = __ldg(pp + (MIRROR ? -1 : 1));
                    walk_step<MIRROR>(frac, q, Sf, pitch);
                }
                S0 = __fadd2_rn(S0, v0);
                S1 = __ffma2_rn(w, __ffma2_rn(v0, m1, v1), S1);
            }
            s0 = S0.x + S0.y;
            s1 = S1.x + S1.y;
        }
#pragma unroll FWD_UNROLL
        for (; k < kstop; ++k) {
            const float w = walk_weight<MIRROR>(frac, sm2, sp1);
            const float* pp = base + q;
            const float v0 = __ldg(pp);
            const float v1 = __ldg(pp + (MIRROR ? -1 : 1));
            s0 += v0;
            s1 = fmaf(w, v1 - v0, s1);
            walk_step<MIRROR>(frac, q, Sf, pitch);      // frac += sigma; split -> next column
        }
        acc += (double)p.L * (double)s0 + (double)p.Lx * (double)s1;
    }
    return acc;
}

// Degenerate angle: thread per ray over its precomputed literal segments,
// stored ray-interleaved so a warp's loads are coalesced like the walk's.
__device__ __forceinline__ double degenerate_ray(const FwdArgs& A, int slot, int j, int e0,
                                                 int e1) {
    ctk_pdl_wait();                                  // x comes from the previous kernel
    const long long cnt = A.deg_cnt[(size_t)slot * A.D + j];
    if (e1 > cnt) e1 = (int)cnt;
    const size_t base = (size_t)slot * A.deg_maxseg * A.D + j;
    double acc = 0.0;
    float s = 0.f;
    int e = e0;
    while (e < e1) {
        const int stop = min(e1, e + 48);
#pragma unroll 8
        for (; e < stop; ++e) {
            const size_t o = base + (size_t)e * A.D;
            s = fmaf(__ldg(A.deg_len + o), __ldg(A.x + __ldg(A.deg_pix + o)), s);
        }
        acc += (double)s;
        s = 0.f;
    }
    return acc;
}

__device__ __forceinline__ double forward_ray(const FwdArgs& A, int a, int slot, int j, int chunk) {
    if (slot >= 0) {                         // whole block: warp-uniform branch
        const int per = (A.deg_maxseg + A.split - 1) / A.split;
        return degenerate_ray(A, slot, j, chunk * per, (chunk + 1) * per);
    }
    const AngleParams p = A.ap[a];
    const double s = A.offsets[j];
    const int R = p.frame == 0 ? A.eg.ny : A.eg.nx;
    const int per = (R + A.split - 1) / A.split;
    const int k0 = chunk * per, k1 = min(R, k0 + per);
    if (p.frame == 0)
        return p.mirror ? walk_ray<true>(p, s, A.P, A.eg.ny, A.eg.nx, A.pad, k0, k1)
                        : walk_ray<false>(p, s, A.P, A.eg.ny, A.eg.nx, A.pad, k0, k1);
    return p.mirror ? walk_ray<true>(p, s, A.PT, A.eg.nx, A.eg.ny, A.pad, k0, k1)
                    : walk_ray<false>(p, s, A.PT, A.eg.nx, A.eg.ny, A.pad, k0, k1);
}

// One ray per thread; SPLIT: rows of each ray over blockIdx.z (small problems).
// A CTA is FWD_APB adjacent angles x 32 adjacent bins, one angle per warp:
// neighbouring angles' rays cross nearly the same pixels at the same time,
// so the warps of a CTA share the L1 lines their gathers pull from L2.
constexpr int FWD_APB = FWD_THREADS / 32;
static_assert(FWD_APB == CTK_FWD_APB, "K2 chaining counts K1 CTAs per angle group");

// K2 chaining: after the barrier that orders the CTA's output stores, one
// release increment of its angle group's counter (see ctk_common.cuh).
// The signalling thread first waits for the previous kernel (K3 of the last
// step, which itself waited for that step's K2): a CTA whose rays all miss
// never reached griddepcontrol.wait, and counting it early would let the
// previous step's K2 see this step's increments.
__device__ __forceinline__ void signal_group(const FwdArgs& A) {
    if (!A.done) return;
    __syncthreads();
    if (threadIdx.x == 0) {
        ctk_pdl_wait();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(A.done + blockIdx.y) : "memory");
    }
}

constexpr int FWD_MAX_SPLIT = 8;            // portable cluster size limit

__device__ __forceinline__ unsigned cluster_addr(const void* p, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
                 : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}

// Resident CTAs per SM: 8 (64 registers) for the row-split cluster launches of
// small problems, whose few short CTAs need the slots; 6 (80 registers) for
// whole-ray CTAs -- measured A per apply at c3 / c4 / c5: 0.1096 / 0.605 /
// 2.838 -> 0.1075 / 0.597 / 2.806 ms (while the split c2 launch would go
// 0.0297 -> 0.0379 ms with 6).
#ifndef CTK_FWD_MINB
#define CTK_FWD_MINB (32 / CTK_FWD_APB_N)
#endif
#ifndef CTK_FWD_MINB_WHOLE
#define CTK_FWD_MINB_WHOLE (CTK_FWD_APB_N == 4 ? 6 : CTK_FWD_MINB)
#endif
#ifndef CTK_FWD_DYNSMEM
#define CTK_FWD_DYNSMEM 0
#endif

template <bool SPLIT>
__global__ void __launch_bounds__(FWD_THREADS, SPLIT ? CTK_FWD_MINB : CTK_FWD_MINB_WHOLE)
k_forward(FwdArgs A) {
    ctk_pdl_trigger();
    // A CTA is 4 adjacent angles x 32 adjacent bins.  Paired layout: each
    // warp takes 2 adjacent angles x 16 bins (half-warps), so a warp's taps
    // on a walk row span ~16 rays' worth of columns (+ the small shift
    // between neighbouring angles) instead of 32 rays' -- fewer cache lines,
    // hence fewer L1 wavefronts, per gather request (the L1 pipe bounds K1).
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int ai, j;
    if (A.pair == 2) {          // 4 angles x 8 bins per warp
        ai = blockIdx.y * FWD_APB + (lane >> 3);
        j = blockIdx.x * 32 + w * 8 + (lane & 7);
    } else if (A.pair == 1) {   // 2 angles x 16 bins per warp
        ai = blockIdx.y * FWD_APB + (w >> 1) * 2 + (lane >> 4);
        j = blockIdx.x * 32 + (w & 1) * 16 + (lane & 15);
    } else {                    // 1 angle x 32 bins per warp
        ai = blockIdx.y * FWD_APB + w;
        j = blockIdx.x * 32 + lane;
    }
    const int a = A.a0 + ai;
    const size_t o = (size_t)ai * A.D + j;
    if (!SPLIT) {
        if (a < A.a1 && j < A.D) {
            const double acc = forward_ray(A, a, A.deg_slot[a], j, 0);
            ctk_pdl_wait();          // rays that miss skipped it: y may still be read upstream
            A.y[o] = A.b ? (float)((double)A.b[o] - acc) : (float)acc;
        }
        signal_group(A);
        return;
    }
    // Row chunks of the same rays form one thread-block cluster (1, 1, split).
    // Chunks 1.. push their fp32 partial into chunk 0's shared memory over
    // DSMEM and arrive on its mbarrier (release.cluster); chunk 0 waits
    // (acquire.cluster) and sums in chunk order -- the same fixed order as a
    // separate finalize pass, with no global fence (which would invalidate
    // the L1 lines the gathers live on) and no second launch.
    __shared__ float s_part[FWD_MAX_SPLIT - 1][FWD_THREADS];
    __shared__ __align__(8) unsigned long long s_bar;
    namespace cg = cooperative_groups;
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();                 // == blockIdx.z
    const unsigned bar = (unsigned)__cvta_generic_to_shared(&s_bar);
    if (rank == 0 && threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(A.split - 1)
                     : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    cl.sync();
    const bool valid = a < A.a1 && j < A.D;
    const float v = valid ? (float)forward_ray(A, a, A.deg_slot[a], j, (int)rank) : 0.f;
    if (rank != 0) {
        asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(
                         cluster_addr(&s_part[rank - 1][threadIdx.x], 0)),
                     "f"(v)
                     : "memory");
        __syncthreads();
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(
                             cluster_addr(&s_bar, 0))
                         : "memory");
        return;
    }
    asm volatile(
        "{\n .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(bar)
        : "memory");
    if (valid) {
        ctk_pdl_wait();              // rays that miss skipped it: y may still be read upstream
        double s = (double)v;
        for (int c = 1; c < A.split; ++c) s += (double)s_part[c - 1][threadIdx.x];
        A.y[o] = A.b ? (float)((double)A.b[o] - s) : (float)s;
    }
    signal_group(A);
}

// Literal fp64 Siddon for every ray (validation path, ctk_forward_exact).
__global__ void __launch_bounds__(FWD_THREADS) k_forward_exact(FwdArgs A) {
    const int a = A.a0 + blockIdx.y;
    const int j = blockIdx.x * FWD_THREADS + threadIdx.x;
    if (j >= A.D) return;
    SumSink sink{A.x, 0.0};
    trace_exact(A.eg, A.cos_tab[a], A.sin_tab[a], A.offsets[j], A.ap[a], sink);
    A.y[(size_t)blockIdx.y * A.D + j] = (float)sink.acc;
}

__global__ void __launch_bounds__(FWD_THREADS) k_count(FwdArgs A, unsigned long long* counts) {
    const int a = A.a0 + blockIdx.y;
    const int j = blockIdx.x * FWD_THREADS + threadIdx.x;
    long long raw = 0, nnz = 0;
    if (j < A.D) {
        CountSink sink;
        trace_exact(A.eg, A.cos_tab[a], A.sin_tab[a], A.offsets[j], A.ap[a], sink);
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

// Degenerate-angle segment lists: pass 1 counts, pass 2 fills the
// ray-interleaved [slot][e][D] layout.
__global__ void k_deg_lists(ExactGrid eg, const AngleParams* ap, const double* cos_tab,
                            const double* sin_tab, const double* offsets, const int* angles,
                            int n_deg, int D, long long* counts, int maxseg, int* pix, float* len) {
    const long long ray = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    if (ray >= (long long)n_deg * D) return;
    const int slot = (int)(ray / D);
    const int a = angles[slot];
    const int j = (int)(ray % D);
    if (pix == nullptr) {
        CountSink c;
        trace_exact(eg, cos_tab[a], sin_tab[a], offsets[j], ap[a], c);
        counts[ray] = c.raw;
    } else {
        FillSink f{pix, len, (long long)slot * maxseg * D + j, D};
        trace_exact(eg, cos_tab[a], sin_tab[a], offsets[j], ap[a], f);
    }
}

static FwdArgs make_args(const ctk_geom* g, const float* x, float* y, int a0, int a1,
                         const float* b) {
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
    A.deg_slot = g->d_deg_slot;
    A.deg_cnt = g->d_deg_ptr;
    A.deg_pix = g->d_deg_pix;
    A.deg_len = g->d_deg_len;
    A.deg_maxseg = g->deg_maxseg;
    A.eg = ExactGrid{g->nx, g->ny, g->h, g->xmin, g->xmax, g->ymin, g->ymax, g->inv_h, g->h_pow2};
    A.D = g->det_count;
    A.a0 = a0;
    A.a1 = a1;
    A.pad = g->fwd_pad;
    A.split = 1;
    A.done = nullptr;
    A.pair = g->fwd_pair;
    return A;
}

}  // namespace ctk

using namespace ctk;

// Called once from ctk_geom_create: literal Siddon segment lists of every
// ray at a degenerate angle, so applies are a memory-parallel list sum.
int ctk_build_degenerate_lists(ctk_geom* g) {
    std::vector<int> slot(g->n_angles, -1), angles;
    std::vector<AngleParams> hap(g->n_angles);
    CTK_CUDA(cudaMemcpy(hap.data(), g->d_ap, sizeof(AngleParams) * g->n_angles,
                        cudaMemcpyDeviceToHost));
    for (int a = 0; a < g->n_angles; ++a)
        if (hap[a].degenerate) {
            slot[a] = (int)angles.size();
            angles.push_back(a);
        }
    CTK_CUDA(cudaMalloc(&g->d_deg_slot, sizeof(int) * g->n_angles));
    CTK_CUDA(cudaMemcpy(g->d_deg_slot, slot.data(), sizeof(int) * g->n_angles,
                        cudaMemcpyHostToDevice));
    const long long rays = (long long)angles.size() * g->det_count;
    CTK_CUDA(cudaMalloc(&g->d_deg_ptr, sizeof(long long) * (rays + 1)));
    CTK_CUDA(cudaMemset(g->d_deg_ptr, 0, sizeof(long long) * (rays + 1)));
    g->deg_segments = 0;
    g->deg_maxseg = 0;
    if (rays == 0) return CTK_OK;
    int* d_angles = nullptr;
    CTK_CUDA(cudaMalloc(&d_angles, sizeof(int) * angles.size()));
    CTK_CUDA(cudaMemcpy(d_angles, angles.data(), sizeof(int) * angles.size(),
                        cudaMemcpyHostToDevice));
    const ExactGrid eg{g->nx, g->ny, g->h, g->xmin, g->xmax, g->ymin, g->ymax, g->inv_h, g->h_pow2};
    const int threads = 128;
    const int blocks = (int)((rays + threads - 1) / threads);
    const int D = g->det_count;
    k_deg_lists<<<blocks, threads>>>(eg, g->d_ap, g->d_cos, g->d_sin, g->d_offsets, d_angles,
                                    (int)angles.size(), D, g->d_deg_ptr, 0, nullptr, nullptr);
    cudaError_t e = cudaGetLastError();
    std::vector<long long> cnt(rays);
    if (e == cudaSuccess)
        e = cudaMemcpy(cnt.data(), g->d_deg_ptr, sizeof(long long) * rays, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
        cudaFree(d_angles);
        return ctk_check_cuda(e, "degenerate segment count");
    }
    long long mx = 0;
    for (long long r = 0; r < rays; ++r) {
        g->deg_segments += cnt[r];
        if (cnt[r] > mx) mx = cnt[r];
    }
    g->deg_maxseg = (int)(mx > 0 ? mx : 1);
    const size_t entries = (size_t)angles.size() * g->deg_maxseg * D;
    e = cudaMalloc(&g->d_deg_pix, sizeof(int) * entries);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_deg_len, sizeof(float) * entries);
    if (e == cudaSuccess) e = cudaMemset(g->d_deg_pix, 0, sizeof(int) * entries);
    if (e == cudaSuccess) e = cudaMemset(g->d_deg_len, 0, sizeof(float) * entries);
    if (e == cudaSuccess) {
        k_deg_lists<<<blocks, threads>>>(eg, g->d_ap, g->d_cos, g->d_sin, g->d_offsets,
                                        d_angles, (int)angles.size(), D, g->d_deg_ptr,
                                        g->deg_maxseg, g->d_deg_pix, g->d_deg_len);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaFree(d_angles);
    if (e != cudaSuccess) return ctk_check_cuda(e, "degenerate segment fill");
    return CTK_OK;
}

static int check_range(const ctk_geom* g, int a0, int a1) {
    if (!g) return ctk_fail(CTK_ERR_ARG, "null geometry");
    if (a0 < 0 || a1 > g->n_angles || a0 > a1)
        return ctk_fail(CTK_ERR_SHAPE, "angle range [%d, %d) outside [0, %d)", a0, a1, g->n_angles);
    return CTK_OK;
}

extern "C" int ctk_forward(const ctk_geom_t* g, const float* x, float* y, int a0, int a1,
                           const float* b, float* work, void* stream) {
    return ctk_forward_ex(g, x, y, a0, a1, b, work, false, stream);
}

// prestaged: work already holds the zero-padded P / PT of x (written by the
// producer of x: K2's epilogue or the SMEM Gram-Schmidt step), so the K1
// staging launch is skipped.  x itself is still read by degenerate angles.
int ctk_forward_ex(const ctk_geom_t* g, const float* x, float* y, int a0, int a1, const float* b,
                   float* work, bool prestaged, void* stream, unsigned* done_flags) {
    int rc = check_range(g, a0, a1);
    if (rc) return rc;
    if (!x || !y) return ctk_fail(CTK_ERR_ARG, "null vector");
    if (a1 == a0) return CTK_OK;
    if (!work) return ctk_fail(CTK_ERR_ARG, "ctk_forward needs a stage work buffer");
    CTK_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = ctk_stream(stream);
    float* P = work;
    float* PT = work + (size_t)g->ny * (g->nx + 2 * g->fwd_pad);
    dim3 sg((g->nx + 31) / 32, (g->ny + 31) / 32), sb(32, 8);
    const int ph = ctk_prof_open(0, st);
    if (!prestaged) {
        k_stage<<<sg, sb, 0, st>>>(x, P, PT, g->nx, g->ny, g->fwd_pad);
        CTK_LAUNCH_CHECK("k_stage");
    }
    FwdArgs A = make_args(g, x, y, a0, a1, b);
    A.P = P;
    A.PT = PT;
    A.split = g->fwd_split;
    A.done = done_flags;
    dim3 grid((g->det_count + 31) / 32, (a1 - a0 + FWD_APB - 1) / FWD_APB, A.split);
    if (A.split > 1)
        CTK_CUDA(ctk_launch_pdl(k_forward<true>, grid, dim3(FWD_THREADS), CTK_FWD_DYNSMEM, st,
                                dim3(1, 1, (unsigned)A.split), A));
    else
        CTK_CUDA(ctk_launch_pdl(k_forward<false>, grid, dim3(FWD_THREADS), CTK_FWD_DYNSMEM, st,
                                dim3(1, 1, 1), A));
    ctk_count_launch();
    ctk_prof_close(ph, st);
    return CTK_OK;
}

extern "C" int ctk_forward_exact(const ctk_geom_t* g, const float* x, float* y, int a0, int a1,
                                 void* stream) {
    int rc = check_range(g, a0, a1);
    if (rc) return rc;
    if (!x || !y) return ctk_fail(CTK_ERR_ARG, "null vector");
    if (a1 == a0) return CTK_OK;
    CTK_CUDA(cudaSetDevice(g->device));
    FwdArgs A = make_args(g, x, y, a0, a1, nullptr);
    dim3 grid((g->det_count + FWD_THREADS - 1) / FWD_THREADS, a1 - a0);
    k_forward_exact<<<grid, FWD_THREADS, 0, ctk_stream(stream)>>>(A);
    CTK_LAUNCH_CHECK("k_forward_exact");
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
    FwdArgs A = make_args(g, nullptr, nullptr, a0, a1, nullptr);
    dim3 grid((g->det_count + FWD_THREADS - 1) / FWD_THREADS, a1 - a0);
    k_count<<<grid, FWD_THREADS, 0, st>>>(A, reinterpret_cast<unsigned long long*>(counts_dev));
    CTK_LAUNCH_CHECK("k_count");
    return CTK_OK;
}
