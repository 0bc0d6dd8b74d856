// ctk_geom.cu -- geometry handle, per-angle tables, error plumbing.
//
// The handle captures what the reference's operator closures capture:
// ImageGrid (ctkrylov/ct.py:37-66) and ParallelGeometry (ct.py:69-96).  All
// derived per-angle constants are computed here once, on the host, in fp64
// from the bitwise numpy cos/sin values, and uploaded.
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <atomic>
#include <vector>

#include "ctk_common.cuh"

static thread_local char g_err[512] = "";
static std::atomic<long long> g_launches{0};

void ctk_count_launch(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

extern "C" int64_t ctk_launch_counter(void) { return g_launches.load(std::memory_order_relaxed); }

int ctk_fail(int code, const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return code;
}

int ctk_check_cuda(cudaError_t e, const char* what) {
    return ctk_fail(CTK_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

extern "C" int ctk_version(void) { return 1; }

extern "C" const char* ctk_last_error(void) { return g_err; }

extern "C" int ctk_device_count(int* out) {
    if (!out) return ctk_fail(CTK_ERR_ARG, "null output");
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess) {
        cudaGetLastError();
        n = 0;
    }
    *out = n;
    return CTK_OK;
}

namespace {

bool is_pow2(double v) {
    if (!(v != 0.0) || !isfinite(v)) return false;
    int e;
    return frexp(fabs(v), &e) == 0.5;
}

constexpr int BTX = 32, BCA = 32;   // must match ctk_back.cu (tile height 8 * back_ppt)

void free_geom(ctk_geom* g) {
    if (!g) return;
    cudaFree(g->d_ap);
    cudaFree(g->d_bp);
    cudaFree(g->d_cos);
    cudaFree(g->d_sin);
    cudaFree(g->d_offsets);
    cudaFree(g->d_deg_slot);
    cudaFree(g->d_deg_ptr);
    cudaFree(g->d_deg_pix);
    cudaFree(g->d_deg_len);
    cudaFree(g->d_degt_ptr);
    cudaFree(g->d_degt_ray);
    cudaFree(g->d_degt_len);
    cudaFree(g->d_degt_angle);
    delete g;
}

}  // namespace

extern "C" int ctk_geom_create(int nx, int ny, double pixel_size, int n_angles,
                               const double* cos_tab, const double* sin_tab, int det_count,
                               const double* offsets, double det_spacing, int device,
                               ctk_geom_t** out) {
    if (!out) return ctk_fail(CTK_ERR_ARG, "null output handle");
    *out = nullptr;
    if (nx <= 0 || ny <= 0 || !(pixel_size > 0))
        return ctk_fail(CTK_ERR_GEOMETRY, "invalid grid: nx=%d, ny=%d, h=%g", nx, ny, pixel_size);
    if (n_angles <= 0 || !cos_tab || !sin_tab)
        return ctk_fail(CTK_ERR_GEOMETRY, "angles must be a non-empty 1-D array");
    if (det_count <= 0 || !(det_spacing > 0) || !offsets)
        return ctk_fail(CTK_ERR_GEOMETRY, "invalid detector: count=%d, spacing=%g", det_count,
                        det_spacing);
    // K1 lockstep walk: a warp's 32 adjacent rays spread over at most
    // 31 * sqrt(2) * spacing / h cross-axis pixels; that many zero columns on
    // each side of the staged copies keep every lane's off-range taps in range.
    int64_t pad = (int64_t)ceil(31.0 * 1.4142135623730951 * det_spacing / pixel_size) + 3;
    if ((int64_t)nx + 2 * pad > (1 << 20) || (int64_t)ny + 2 * pad > (1 << 20) ||
        (int64_t)(nx > ny ? nx : ny) * ((nx > ny ? nx : ny) + 2 * pad) >= (1LL << 31))
        return ctk_fail(CTK_ERR_GEOMETRY, "grid too large for the 32.32 walk (%d x %d)", nx, ny);

    // Paired K1 warps (2 adjacent angles x 16 bins): at a common walk row the
    // two angles' rays of one bin differ by <= dtheta * r * sqrt 2 pixels
    // (r: the image half-diagonal), so the warp's spread is 15 bins plus that
    // shift; pair only where the shift is a few pixels, and pad for it.
    int pair = 0;
    {
        double shift = 0.0;
        for (int a = 0; a + 1 < n_angles; a += 2) {
            const double sd = sin_tab[a + 1] * cos_tab[a] - cos_tab[a + 1] * sin_tab[a];
            const double cd = cos_tab[a + 1] * cos_tab[a] + sin_tab[a + 1] * sin_tab[a];
            const double dth = fabs(atan2(sd, cd));
            if (dth > shift) shift = dth;
        }
        const double rmax = 0.5 * pixel_size * sqrt((double)nx * nx + (double)ny * ny);
        const double shift_px = shift * rmax * 1.4142135623730951 / pixel_size;
        // measured (tools/bench_projectors.py): 2 x 16 warps cut c4 / c5 A
        // by 5% (0.636 -> 0.603, 3.00 -> 2.83 ms) and cost 4-14% on the
        // shorter rays of c2 / c3; CTK_FWD_PAIR = 0 / 1 / 2 (4 x 8) overrides
        const char* e = getenv("CTK_FWD_PAIR");
        const int want = e ? atoi(e) : ((nx < ny ? nx : ny) >= 1024 ? 1 : 0);
        if (want > 0 && shift_px <= 8.0) {
            pair = want > 2 ? 2 : want;
            if (pair == 2 && CTK_FWD_APB != 4) pair = 1;      // 4 x 8 warps assume 4-warp CTAs
            const int64_t need = (int64_t)ceil((pair == 2 ? 7.0 : 15.0) * 1.4142135623730951 *
                                                   det_spacing / pixel_size +
                                               (pair == 2 ? 3.0 : 1.0) * shift_px) + 3;
            if (need > pad) pad = need;
        }
    }
    ctk_geom* g = new ctk_geom();
    memset(g, 0, sizeof(*g));
    g->device = device;
    g->fwd_pad = (int)pad;
    g->fwd_pair = pair;
    g->nx = nx;
    g->ny = ny;
    g->n_angles = n_angles;
    g->det_count = det_count;
    g->h = pixel_size;
    g->det_spacing = det_spacing;
    // ImageGrid.extent (ct.py:53-58): hx = 0.5 * nx * h
    const double hx = 0.5 * (double)nx * pixel_size, hy = 0.5 * (double)ny * pixel_size;
    g->xmin = -hx;
    g->xmax = hx;
    g->ymin = -hy;
    g->ymax = hy;
    g->center = 0.5 * (double)(det_count - 1);   // ct.py:215
    g->h_pow2 = is_pow2(pixel_size) ? 1 : 0;
    g->inv_h = 1.0 / pixel_size;

    std::vector<ctk::AngleParams> ap(n_angles);
    std::vector<ctk::BackParams> bp(n_angles);
    double max_span = 0.0;
    {   // K2 rows per thread: 4 (32x32 tiles, fewer per-angle setups) once the
        // image has enough tiles to fill the GPU, 2 (32x16) from 256^2, else 1
        // (32x8: more tiles for small images; c1 K2 15.5 -> 14.1 us in-solve)
        const int64_t npx = (int64_t)nx * ny;
        int ppt = npx >= 512LL * 512 ? 4 : (npx >= 256LL * 256 ? 2 : 1);
        const char* ov = getenv("CTK_BACK_PPT");          // tuning override (1, 2 or 4)
        if (ov && (atoi(ov) == 1 || atoi(ov) == 2 || atoi(ov) == 4)) ppt = atoi(ov);
        g->back_ppt = ppt;
    }
    const int bty = 8 * g->back_ppt;
    const double h = pixel_size;
    int n_near = 0;
    for (int a = 0; a < n_angles; ++a) {
        const double c = cos_tab[a], s = sin_tab[a];
        ctk::AngleParams p;
        memset(&p, 0, sizeof(p));
        // Literal path (K1d segment lists from the fp64 tracer): the angles the
        // reference treats as axis-aligned (|sin| or |cos| < 1e-14,
        // ct.py:153,165,168), and those within 1e-5 rad of an axis.  There the
        // walk's slope, quantised to 2^-32 px per row, is off by up to
        // 0.5 / (sigma 2^32) of itself (7% at 1e-9 rad), which moves the row
        // where a ray lying on a grid line changes column -- 1e-2 errors in
        // such rays (found by the random-geometry parity test).  At most
        // CTK_MAX_NEAR_AXIS such angles take the lists (each costs
        // ~8 bytes x segments per ray x bins); uniform angle sets have none.
        const bool on_axis = fabs(s) < 1e-14 || fabs(c) < 1e-14;
        const bool near_axis = !on_axis && (fabs(s) < 1e-5 || fabs(c) < 1e-5) &&
                               n_near < ctk::CTK_MAX_NEAR_AXIS;
        n_near += near_axis;
        p.degenerate = (on_axis || near_axis) ? 1 : 0;
        p.exact_flags = (is_pow2(-s) ? 1 : 0) | (is_pow2(c) ? 2 : 0);
        p.inv_dx = s != 0.0 ? 1.0 / -s : 0.0;
        p.inv_dy = c != 0.0 ? 1.0 / c : 0.0;
        if (p.degenerate && g->n_degenerate < ctk::CTK_MAX_DEG_LIST)
            g->deg_list[g->n_degenerate] = a;
        double sigma_raw, C;
        if (fabs(c) >= fabs(s)) {
            // walk image rows top->bottom; u = (x - xmin)/h at row boundary
            const double t = s / c;
            p.frame = 0;
            p.beta = 1.0 / (c * h);
            p.alpha = (-g->xmin - g->ymax * t) / h;
            sigma_raw = t;
            C = nx;
            p.L = (float)(h / fabs(c));
            p.Lx = (float)(s != 0.0 ? h / fabs(s) : 0.0);
        } else {
            // walk image columns left->right; v = (ymax - y)/h at column boundary
            const double ct = c / s;
            p.frame = 1;
            p.beta = -1.0 / (s * h);
            p.alpha = (g->ymax + g->xmin * ct) / h;
            sigma_raw = ct;
            C = ny;
            p.L = (float)(h / fabs(s));
            p.Lx = (float)(c != 0.0 ? h / fabs(c) : 0.0);
        }
        if (sigma_raw < 0) {
            p.mirror = 1;
            p.alpha = C - p.alpha;
            p.beta = -p.beta;
            sigma_raw = -sigma_raw;
        }
        if (sigma_raw > 1.0) sigma_raw = 1.0;
        p.sigma_fx = llrint(sigma_raw * 4294967296.0);
        // the walk keeps a 32-bit fraction: sigma == 1 (|tan| rounds to 1 at 45
        // degrees) becomes 1 - 2^-32, a 1e-6-pixel drift over a 4096-row walk
        if (p.sigma_fx > 0xffffffffll) p.sigma_fx = 0xffffffffll;
        p.inv_sg = p.sigma_fx > 0 ? 1.0 / (double)p.sigma_fx : 0.0;
        ap[a] = p;
        bp[a].cg = c / det_spacing;
        bp[a].sg = s / det_spacing;
        const double span = ((BTX - 1) * fabs(c) + (bty - 1) * fabs(s)) * h / det_spacing;
        if (span > max_span) max_span = span;
        g->n_degenerate += p.degenerate;
    }
    g->back_wmax = (int)ceil(max_span) + 6;
    {   // K1 row split: up to one wave of 128-thread CTAs (12 resident per SM)
        const int64_t m = (int64_t)n_angles * det_count;
        int64_t sp = (148LL * 12 * 128 + m - 1) / m;
        if (sp < 1) sp = 1;
        if (sp > 8) sp = 8;
        const int rmin = nx < ny ? nx : ny;
        if (sp > rmin / 32) sp = rmin / 32;               // >= 32 rows per chunk: the per-ray
        if (sp < 1) sp = 1;                               // setup must stay amortised
        const char* ov = getenv("CTK_FWD_SPLIT");          // tuning override (1..8)
        if (ov && atoi(ov) >= 1 && atoi(ov) <= 8) sp = atoi(ov);
        g->fwd_split = (int)sp;
    }
    if ((size_t)BCA * g->back_wmax * 2 * sizeof(float) > 200 * 1024) {
        free_geom(g);
        return ctk_fail(CTK_ERR_GEOMETRY,
                        "pixel/bin ratio too large for the staged backprojector (window %d)",
                        (int)ceil(max_span));
    }

    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_ap, sizeof(ctk::AngleParams) * n_angles);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_bp, sizeof(ctk::BackParams) * n_angles);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_cos, sizeof(double) * n_angles);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_sin, sizeof(double) * n_angles);
    if (e == cudaSuccess) e = cudaMalloc(&g->d_offsets, sizeof(double) * det_count);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_ap, ap.data(), sizeof(ctk::AngleParams) * n_angles,
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_bp, bp.data(), sizeof(ctk::BackParams) * n_angles,
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_cos, cos_tab, sizeof(double) * n_angles, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_sin, sin_tab, sizeof(double) * n_angles, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(g->d_offsets, offsets, sizeof(double) * det_count, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        free_geom(g);
        return ctk_check_cuda(e, "ctk_geom_create");
    }
    int rc = ctk_build_degenerate_lists(g);
    if (rc != CTK_OK) {
        free_geom(g);
        return rc;
    }
    *out = g;
    return CTK_OK;
}

extern "C" int ctk_geom_destroy(ctk_geom_t* g) {
    if (!g) return CTK_OK;
    cudaSetDevice(g->device);
    free_geom(g);
    return CTK_OK;
}

extern "C" int ctk_geom_info(const ctk_geom_t* g, int64_t* n, int64_t* m, int64_t* stage_floats,
                             int* n_degenerate) {
    if (!g) return ctk_fail(CTK_ERR_ARG, "null geometry");
    if (n) *n = (int64_t)g->nx * g->ny;
    if (m) *m = (int64_t)g->n_angles * g->det_count;
    if (stage_floats) *stage_floats = ctk_stage_floats(g);
    if (n_degenerate) *n_degenerate = g->n_degenerate;
    return CTK_OK;
}
