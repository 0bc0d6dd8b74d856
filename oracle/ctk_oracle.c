/*
 * ctk_oracle.c -- CPU ORACLE for the A/B projector hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker, never the product: only tests/, the
 * smoke() check in __graft_entry__.py and bench.py's cpu_baseline /
 * --impl reference legs may load it.  The product path (the CUDA library in
 * paper_2602_17892_b200/csrc) never links or calls anything here.
 *
 * It restates, in plain C with strict IEEE evaluation (-ffp-contract=off),
 * the reference's fp64 algorithms so that results are bit-identical to the
 * unmodified reference on the same inputs:
 *
 *   orc_siddon_ray      <- ctkrylov/ct.py:137-179  (_siddon_ray)
 *   orc_forward         <- ctkrylov/ct.py:182-201  (forward_ray_driven: COO -> CSR,
 *                          duplicate (ray,pixel) pairs summed, SpMV in column order)
 *   orc_csr_*           <- same operator as an assembled CSR (what the reference
 *                          builds once and applies with scipy's csr_matvec)
 *   orc_back            <- ctkrylov/ct.py:204-245  (back_pixel_driven), angle-ordered
 *                          accumulation per pixel exactly as the reference's loop
 *
 * Geometry inputs are passed from numpy bitwise (cos/sin tables evaluated
 * with scalar np.cos/np.sin as the reference does, bin offsets from
 * ParallelGeometry.bin_offsets, ctkrylov/ct.py:93-96), so no libm call here
 * can introduce a one-ulp difference.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

typedef struct {
    int nx, ny;
    double h;
    double xmin, xmax, ymin, ymax;
} orc_grid;

static orc_grid make_grid(int nx, int ny, double h) {
    /* ImageGrid.extent, ctkrylov/ct.py:53-58: hx = 0.5 * nx * h */
    orc_grid g;
    g.nx = nx;
    g.ny = ny;
    g.h = h;
    double hx = 0.5 * (double)nx * h;
    double hy = 0.5 * (double)ny * h;
    g.xmin = -hx;
    g.xmax = hx;
    g.ymin = -hy;
    g.ymax = hy;
    return g;
}

/* One ray, ctkrylov/ct.py:137-179.  Writes up to (nx+ny+2) segments.
 * t_buf must hold nx+ny+4 doubles.  Returns the kept segment count. */
static int siddon_ray(const orc_grid* g, double ct, double st, double offset,
                      int64_t* pix, double* len, double* t_buf) {
    const double h = g->h;
    const int nx = g->nx, ny = g->ny;
    double px = offset * ct, py = offset * st;
    double dx = -st, dy = ct;
    double t_lo = -INFINITY, t_hi = INFINITY;
    /* slab clip, ct.py:149-160 */
    {
        double p0s[2] = {px, py}, ds[2] = {dx, dy};
        double los[2] = {g->xmin, g->ymin}, his[2] = {g->xmax, g->ymax};
        for (int a = 0; a < 2; ++a) {
            double p0 = p0s[a], d = ds[a], lo = los[a], hi = his[a];
            if (fabs(d) < 1e-14) {
                if (p0 < lo || p0 > hi) return 0;
            } else {
                double t0 = (lo - p0) / d, t1 = (hi - p0) / d;
                if (t0 > t1) { double tmp = t0; t0 = t1; t1 = tmp; }
                /* Python max/min on floats */
                if (t0 > t_lo) t_lo = t0;
                if (t1 < t_hi) t_hi = t1;
            }
        }
    }
    if (t_hi <= t_lo) return 0;

    /* crossings, ct.py:163-171: three sorted streams merged with exact-duplicate
     * removal (np.unique).  tx_i = (xmin + i*h - px)/dx is monotone in i. */
    int nt = 0;
    t_buf[nt++] = t_lo;
    int use_x = fabs(dx) >= 1e-14, use_y = fabs(dy) >= 1e-14;
    int ix_i = 0, ix_step = 1, ix_n = use_x ? nx + 1 : 0;
    if (use_x && dx < 0) { ix_i = nx; ix_step = -1; }
    int iy_i = 0, iy_step = 1, iy_n = use_y ? ny + 1 : 0;
    if (use_y && dy < 0) { iy_i = ny; iy_step = -1; }
    int kx = 0, ky = 0;
    /* Each stream's next in-range crossing is computed once and kept until it
     * is consumed (the same value, bit for bit, as re-evaluating it every
     * merge step). */
    double tx = INFINITY, ty = INFINITY;
    int have_x = 0, have_y = 0;
    for (;;) {
        /* advance streams past values outside (t_lo, t_hi) */
        if (!have_x) {
            tx = INFINITY;
            while (kx < ix_n) {
                double v = (g->xmin + (double)ix_i * h - px) / dx;
                if (v > t_lo && v < t_hi) { tx = v; have_x = 1; break; }
                ix_i += ix_step; ++kx;
            }
        }
        if (!have_y) {
            ty = INFINITY;
            while (ky < iy_n) {
                double v = (g->ymin + (double)iy_i * h - py) / dy;
                if (v > t_lo && v < t_hi) { ty = v; have_y = 1; break; }
                iy_i += iy_step; ++ky;
            }
        }
        if (kx >= ix_n && ky >= iy_n) break;
        double v;
        if (tx <= ty) { v = tx; ix_i += ix_step; ++kx; have_x = 0; }
        else { v = ty; iy_i += iy_step; ++ky; have_y = 0; }
        if (v != t_buf[nt - 1]) t_buf[nt++] = v;
    }
    if (t_hi != t_buf[nt - 1]) t_buf[nt++] = t_hi;

    int ns = 0;
    for (int k = 0; k + 1 < nt; ++k) {
        double l = t_buf[k + 1] - t_buf[k];
        double tm = 0.5 * (t_buf[k] + t_buf[k + 1]);
        double qx = px + tm * dx - g->xmin, qy = g->ymax - (py + tm * dy);
        /* x / 1.0 == x exactly: skip the divisions at unit pixel size */
        double fx = floor(h == 1.0 ? qx : qx / h);
        double fy = floor(h == 1.0 ? qy : qy / h);
        int64_t ix = (int64_t)fx, iy = (int64_t)fy;
        if (ix < 0) ix = 0;
        if (ix > nx - 1) ix = nx - 1;
        if (iy < 0) iy = 0;
        if (iy > ny - 1) iy = ny - 1;
        if (l > 1e-15) {
            pix[ns] = iy * nx + ix;
            len[ns] = l;
            ++ns;
        }
    }
    return ns;
}

static void rev_span(int64_t* pix, double* len, int lo, int hi) {
    for (--hi; lo < hi; ++lo, --hi) {
        int64_t tp = pix[lo]; pix[lo] = pix[hi]; pix[hi] = tp;
        double tl = len[lo]; len[lo] = len[hi]; len[hi] = tl;
    }
}

/* Reverse [lo, hi) as a sequence of equal-pixel runs: run order flips, the
 * order inside each run (trace order of duplicates) is kept. */
static void rev_groups(int64_t* pix, double* len, int lo, int hi) {
    rev_span(pix, len, lo, hi);
    for (int a = lo; a < hi;) {
        int b = a + 1;
        while (b < hi && pix[b] == pix[a]) ++b;
        if (b - a > 1) rev_span(pix, len, a, b);
        a = b;
    }
}

static int is_sorted_pix(const int64_t* pix, int ns) {
    for (int i = 1; i < ns; ++i)
        if (pix[i - 1] > pix[i]) return 0;
    return 1;
}

/* CSR canonicalisation of one row (scipy csr_sort_indices + csr_sum_duplicates):
 * sort by column, sum duplicates, in place.  Returns merged count.
 * The result is what a STABLE sort gives (duplicates summed in trace order,
 * as the insertion sort this replaces did).  Along a ray the row iy and the
 * column ix of the segments are monotone, so the sorted order is reached in
 * O(ns) by flipping the row-block order and then each decreasing block (as
 * runs of equal pixels); should that not leave the row sorted, a stable
 * bottom-up merge sort of the original order runs instead.  (An insertion
 * sort is quadratic on the reversed rows of c4/c5 rays, ~3k segments.)
 * tmp_pix / tmp_len hold ns entries. */
static int canon_row(int64_t* pix, double* len, int ns, int nx, int64_t* tmp_pix,
                     double* tmp_len) {
    if (!is_sorted_pix(pix, ns)) {
        memcpy(tmp_pix, pix, sizeof(int64_t) * (size_t)ns);
        memcpy(tmp_len, len, sizeof(double) * (size_t)ns);
        if (pix[0] / nx > pix[ns - 1] / nx) rev_groups(pix, len, 0, ns);
        for (int a = 0; a < ns;) {
            int b = a + 1;
            while (b < ns && pix[b] / nx == pix[a] / nx) ++b;
            if (pix[a] > pix[b - 1]) rev_groups(pix, len, a, b);
            a = b;
        }
        if (!is_sorted_pix(pix, ns)) {
            memcpy(pix, tmp_pix, sizeof(int64_t) * (size_t)ns);
            memcpy(len, tmp_len, sizeof(double) * (size_t)ns);
            int64_t *sp = pix, *dp = tmp_pix;
            double *sl = len, *dl = tmp_len;
            for (int w = 1; w < ns; w *= 2) {
                for (int lo = 0; lo < ns; lo += 2 * w) {
                    int mid = lo + w < ns ? lo + w : ns;
                    int hi = lo + 2 * w < ns ? lo + 2 * w : ns;
                    int i = lo, j = mid, o = lo;
                    while (i < mid && j < hi) {
                        if (sp[j] < sp[i]) { dp[o] = sp[j]; dl[o++] = sl[j++]; }
                        else { dp[o] = sp[i]; dl[o++] = sl[i++]; }
                    }
                    while (i < mid) { dp[o] = sp[i]; dl[o++] = sl[i++]; }
                    while (j < hi) { dp[o] = sp[j]; dl[o++] = sl[j++]; }
                }
                int64_t* tp = sp; sp = dp; dp = tp;
                double* tl = sl; sl = dl; dl = tl;
            }
            if (sp != pix) {
                memcpy(pix, sp, sizeof(int64_t) * (size_t)ns);
                memcpy(len, sl, sizeof(double) * (size_t)ns);
            }
        }
    }
    int out = 0;
    for (int i = 0; i < ns; ++i) {
        if (out > 0 && pix[out - 1] == pix[i]) {
            len[out - 1] = len[out - 1] + len[i];
        } else {
            pix[out] = pix[i];
            len[out] = len[i];
            ++out;
        }
    }
    return out;
}

/* ---- tiny pthread parallel-for (dynamic chunks over [0, n)) ---------- */
typedef void (*orc_body_fn)(void* ctx, int64_t lo, int64_t hi, void* scratch);
typedef struct {
    orc_body_fn fn;
    void* ctx;
    int64_t n, chunk;
    int64_t next; /* guarded by mu */
    pthread_mutex_t mu;
    size_t scratch_bytes;
} orc_pool;

static void* orc_worker(void* arg) {
    orc_pool* p = (orc_pool*)arg;
    void* scratch = p->scratch_bytes ? malloc(p->scratch_bytes) : NULL;
    for (;;) {
        pthread_mutex_lock(&p->mu);
        int64_t lo = p->next;
        p->next += p->chunk;
        pthread_mutex_unlock(&p->mu);
        if (lo >= p->n) break;
        int64_t hi = lo + p->chunk < p->n ? lo + p->chunk : p->n;
        p->fn(p->ctx, lo, hi, scratch);
    }
    free(scratch);
    return NULL;
}

static void orc_parallel_for(int64_t n, int64_t chunk, int nthreads, size_t scratch_bytes,
                             orc_body_fn fn, void* ctx) {
    if (nthreads <= 0) {
        long c = sysconf(_SC_NPROCESSORS_ONLN);
        nthreads = c > 0 ? (int)c : 1;
    }
    if (nthreads > 256) nthreads = 256;
    orc_pool p;
    p.fn = fn; p.ctx = ctx; p.n = n; p.chunk = chunk > 0 ? chunk : 1; p.next = 0;
    p.scratch_bytes = scratch_bytes;
    pthread_mutex_init(&p.mu, NULL);
    if (nthreads == 1) {
        orc_worker(&p);
    } else {
        pthread_t th[256];
        for (int i = 0; i < nthreads; ++i) pthread_create(&th[i], NULL, orc_worker, &p);
        for (int i = 0; i < nthreads; ++i) pthread_join(th[i], NULL);
    }
    pthread_mutex_destroy(&p.mu);
}

/* ---- ray-parallel work ------------------------------------------------ */
typedef struct {
    orc_grid g;
    const double *cos_tab, *sin_tab, *offsets, *x;
    int det_count;
    double* y;              /* forward */
    int64_t* row_nnz;       /* csr pass 1 / counts */
    int64_t* row_raw;       /* counts */
    const int64_t* indptr;  /* csr pass 2 */
    int32_t* indices;
    double* data;
} ray_ctx;

#define RAY_SCRATCH(c) (sizeof(double) * 5 * (size_t)((c)->g.nx + (c)->g.ny + 8))

#define CANON_TMP(c, scratch) \
    (int64_t*)((double*)(scratch) + 3 * ((c)->g.nx + (c)->g.ny + 8)), \
    (double*)(scratch) + 4 * ((c)->g.nx + (c)->g.ny + 8)

static int trace_row(const ray_ctx* c, int64_t r, void* scratch, int64_t** pix, double** len) {
    const int cap = c->g.nx + c->g.ny + 8;
    *pix = (int64_t*)scratch;
    *len = (double*)scratch + cap;
    double* tb = (double*)scratch + 2 * cap;
    int a = (int)(r / c->det_count), j = (int)(r % c->det_count);
    return siddon_ray(&c->g, c->cos_tab[a], c->sin_tab[a], c->offsets[j], *pix, *len, tb);
}

static void body_forward(void* vctx, int64_t lo, int64_t hi, void* scratch) {
    ray_ctx* c = (ray_ctx*)vctx;
    for (int64_t r = lo; r < hi; ++r) {
        int64_t* pix; double* len;
        int ns = trace_row(c, r, scratch, &pix, &len);
        ns = canon_row(pix, len, ns, c->g.nx, CANON_TMP(c, scratch));
        double s = 0.0;
        for (int k = 0; k < ns; ++k) s += len[k] * c->x[pix[k]];
        c->y[r] = s;
    }
}

static void body_count(void* vctx, int64_t lo, int64_t hi, void* scratch) {
    ray_ctx* c = (ray_ctx*)vctx;
    for (int64_t r = lo; r < hi; ++r) {
        int64_t* pix; double* len;
        int ns = trace_row(c, r, scratch, &pix, &len);
        if (c->row_raw) c->row_raw[r] = ns;
        c->row_nnz[r] = canon_row(pix, len, ns, c->g.nx, CANON_TMP(c, scratch));
    }
}

static void body_fill(void* vctx, int64_t lo, int64_t hi, void* scratch) {
    ray_ctx* c = (ray_ctx*)vctx;
    for (int64_t r = lo; r < hi; ++r) {
        int64_t* pix; double* len;
        int ns = trace_row(c, r, scratch, &pix, &len);
        ns = canon_row(pix, len, ns, c->g.nx, CANON_TMP(c, scratch));
        int64_t base = c->indptr[r];
        for (int k = 0; k < ns; ++k) {
            c->indices[base + k] = (int32_t)pix[k];
            c->data[base + k] = len[k];
        }
    }
}

static ray_ctx make_ray_ctx(int nx, int ny, double h, const double* cos_tab,
                            const double* sin_tab, int det_count, const double* offsets) {
    ray_ctx c;
    memset(&c, 0, sizeof(c));
    c.g = make_grid(nx, ny, h);
    c.cos_tab = cos_tab;
    c.sin_tab = sin_tab;
    c.offsets = offsets;
    c.det_count = det_count;
    return c;
}

/* Exported: segments of one ray (for tests). */
int orc_siddon_ray(int nx, int ny, double h, double ct, double st, double offset,
                   int64_t* pix, double* len) {
    orc_grid g = make_grid(nx, ny, h);
    double* t_buf = (double*)malloc(sizeof(double) * (size_t)(nx + ny + 8));
    int n = siddon_ray(&g, ct, st, offset, pix, len, t_buf);
    free(t_buf);
    return n;
}

/* y[a*D+j] = sum over the canonical CSR row of len * x[pix] (ct.py:197-201). */
int orc_forward(int nx, int ny, double h, int n_angles, const double* cos_tab,
                const double* sin_tab, int det_count, const double* offsets,
                const double* x, double* y, int nthreads) {
    ray_ctx c = make_ray_ctx(nx, ny, h, cos_tab, sin_tab, det_count, offsets);
    c.x = x;
    c.y = y;
    orc_parallel_for((int64_t)n_angles * det_count, 64, nthreads, RAY_SCRATCH(&c),
                     body_forward, &c);
    return 0;
}

/* Per-ray segment counts: raw (kept segments, before duplicate merge) and
 * CSR nnz (after).  Either output may be NULL for raw. */
int orc_row_counts(int nx, int ny, double h, int n_angles, const double* cos_tab,
                   const double* sin_tab, int det_count, const double* offsets,
                   int64_t* row_raw, int64_t* row_nnz, int nthreads) {
    ray_ctx c = make_ray_ctx(nx, ny, h, cos_tab, sin_tab, det_count, offsets);
    c.row_raw = row_raw;
    c.row_nnz = row_nnz;
    orc_parallel_for((int64_t)n_angles * det_count, 64, nthreads, RAY_SCRATCH(&c),
                     body_count, &c);
    return 0;
}

/* Assembled CSR pass 2 (the reference's one-time build, ct.py:189-200),
 * given indptr from the cumulative row_nnz. */
int orc_csr_fill(int nx, int ny, double h, int n_angles, const double* cos_tab,
                 const double* sin_tab, int det_count, const double* offsets,
                 const int64_t* indptr, int32_t* indices, double* data, int nthreads) {
    ray_ctx c = make_ray_ctx(nx, ny, h, cos_tab, sin_tab, det_count, offsets);
    c.indptr = indptr;
    c.indices = indices;
    c.data = data;
    orc_parallel_for((int64_t)n_angles * det_count, 64, nthreads, RAY_SCRATCH(&c),
                     body_fill, &c);
    return 0;
}

/* scipy csr_matvec: the row sum starts at 0 and accumulates in stored
 * (column-sorted) order. */
typedef struct {
    const int64_t* indptr;
    const int32_t* indices;
    const double *data, *x;
    double* y;
} spmv_ctx;

static void body_spmv(void* vctx, int64_t lo, int64_t hi, void* scratch) {
    (void)scratch;
    spmv_ctx* c = (spmv_ctx*)vctx;
    for (int64_t r = lo; r < hi; ++r) {
        double s = 0.0;
        for (int64_t k = c->indptr[r]; k < c->indptr[r + 1]; ++k)
            s += c->data[k] * c->x[c->indices[k]];
        c->y[r] = s;
    }
}

int orc_csr_spmv(int64_t m, const int64_t* indptr, const int32_t* indices,
                 const double* data, const double* x, double* y, int nthreads) {
    spmv_ctx c = {indptr, indices, data, x, y};
    orc_parallel_for(m, 1024, nthreads, 0, body_spmv, &c);
    return 0;
}

/* Pixel-driven backprojection, ct.py:204-245.  out[p] accumulates the
 * per-angle terms in angle order, exactly as the reference's angle loop. */
typedef struct {
    orc_grid g;
    int n_angles, det_count;
    const double *cos_tab, *sin_tab, *u;
    double det_spacing, center;
    double* out;
} back_ctx;

static void body_back(void* vctx, int64_t lo, int64_t hi, void* scratch) {
    (void)scratch;
    back_ctx* c = (back_ctx*)vctx;
    const int D = c->det_count;
    const double h = c->g.h;
    for (int64_t p = lo; p < hi; ++p) {
        int iy = (int)(p / c->g.nx), ix = (int)(p % c->g.nx);
        /* ImageGrid.pixel_centers, ct.py:60-66 */
        double X = c->g.xmin + ((double)ix + 0.5) * h;
        double Y = c->g.ymax - ((double)iy + 0.5) * h;
        double acc = 0.0;
        for (int a = 0; a < c->n_angles; ++a) {
            double gg = (X * c->cos_tab[a] + Y * c->sin_tab[a]) / c->det_spacing + c->center;
            int64_t i0 = (int64_t)floor(gg);
            double w1 = gg - (double)i0;
            const double* row = c->u + (int64_t)a * D;
            /* ct.py:227,231: idx0 = clip(i0); idx1 = clip(idx0 + 1) -- the second
             * tap is indexed from the CLIPPED first tap, so i0 == -1 reads
             * row[1] (row[0] when D == 1), not row[0].  Kept verbatim. */
            int64_t idx0 = i0 < 0 ? 0 : (i0 > D - 1 ? D - 1 : i0);
            int64_t idx1 = idx0 + 1 > D - 1 ? D - 1 : idx0 + 1;
            double v0 = (i0 >= 0 && i0 <= D - 1) ? row[idx0] : 0.0;
            double v1 = (i0 + 1 >= 0 && i0 + 1 <= D - 1) ? row[idx1] : 0.0;
            acc += h * ((1.0 - w1) * v0 + w1 * v1);
        }
        c->out[p] = acc;
    }
}

int orc_back(int nx, int ny, double h, int n_angles, const double* cos_tab,
             const double* sin_tab, int det_count, double det_spacing,
             const double* u, double* out, int nthreads) {
    back_ctx c;
    c.g = make_grid(nx, ny, h);
    c.n_angles = n_angles;
    c.det_count = det_count;
    c.cos_tab = cos_tab;
    c.sin_tab = sin_tab;
    c.u = u;
    c.det_spacing = det_spacing;
    c.center = 0.5 * (double)(det_count - 1);
    c.out = out;
    orc_parallel_for((int64_t)nx * ny, 256, nthreads, 0, body_back, &c);
    return 0;
}
