/*
 * ctk.h -- C ABI of the B200-native projector / Krylov library (libctk.so).
 *
 * Drop-in boundary for the hot path of ctkrylov's hybrid AB-/BA-GMRES
 * (reference paths relative to pkg/src of arxiv/paper_2602_17892):
 *
 *   ctk_geom_create   replaces the geometry captured by the closures built in
 *                     forward_ray_driven / back_pixel_driven
 *                     (ctkrylov/ct.py:182-201, 204-245; ImageGrid ct.py:37-66,
 *                     ParallelGeometry ct.py:69-96)
 *   ctk_forward       replaces A.apply: `lambda v: mat @ v`        (ct.py:201)
 *                     optionally fused with the residual b - A x   (gmres.py:174,209)
 *   ctk_forward_exact literal fp64 Siddon (ct.py:137-179), every angle
 *   ctk_count_segments  segment / CSR-nnz counts of A               (ct.py:178,197-200)
 *   ctk_back          replaces B.apply: the angle loop            (ct.py:234-245)
 *                     optionally fused with x0 + B(.)              (gmres.py:207)
 *   ctk_cgs2_step     replaces arnoldi_step's MGS + reorth sweeps  (arnoldi.py:66-82)
 *   ctk_combine       replaces W = column_stack(basis); W @ y; x0 + (.)
 *                                                                  (gmres.py:205-207)
 *   ctk_dots / ctk_update / ctk_norm2   the vector primitives behind the above
 *                     (np.linalg.norm at arnoldi.py:42,67,77, gmres.py:210,251)
 *
 * Conventions
 *   - Every vector is caller-owned device memory, fp32, contiguous.  Images are
 *     row-major (ny, nx) with row 0 at the top; sinograms are angle-major
 *     (a * det_count + j), exactly the reference layout (ct.py:10-18).
 *   - Calls are asynchronous and stream-ordered on `stream` (a cudaStream_t
 *     passed as void*; NULL = legacy default stream).  Nothing allocates on the
 *     hot path.  Reductions are deterministic (fixed trees, no float atomics).
 *   - Return 0 on success, a negative CTK_ERR_* code otherwise;
 *     ctk_last_error() returns a thread-local message for the last failure.
 *   - A geometry handle is immutable after creation and may be shared across
 *     host threads and streams.  Scratch buffers are per call site (one per
 *     stream in flight) and must be zero-filled once when allocated.
 */
#ifndef CTK_H_
#define CTK_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CTK_OK 0
#define CTK_ERR_ARG (-1)      /* invalid argument (ValueError)                        */
#define CTK_ERR_SHAPE (-2)    /* inconsistent dimensions (OperatorShapeError)         */
#define CTK_ERR_GEOMETRY (-3) /* invalid grid / geometry (GeometryError)              */
#define CTK_ERR_CUDA (-4)     /* CUDA runtime failure (RuntimeError)                  */

typedef struct ctk_geom ctk_geom_t;

int ctk_version(void);
const char* ctk_last_error(void);

/* Geometry.  cos_tab/sin_tab are the bitwise host values np.cos(theta) /
 * np.sin(theta) for each angle; offsets are ParallelGeometry.bin_offsets()
 * (ct.py:93-96).  Angles must already satisfy the reference's validation
 * (strictly increasing in [0, pi)); the library checks sizes and positivity. */
int ctk_geom_create(int nx, int ny, double pixel_size, int n_angles,
                    const double* cos_tab, const double* sin_tab, int det_count,
                    const double* offsets, double det_spacing, int device,
                    ctk_geom_t** out);
int ctk_geom_destroy(ctk_geom_t* g);
/* n = nx*ny, m = n_angles*det_count, stage_floats = workspace for ctk_forward,
 * n_degenerate = angles taking the literal segment-list path (axis-aligned,
 * or within 1e-5 rad of an axis). */
int ctk_geom_info(const ctk_geom_t* g, int64_t* n, int64_t* m, int64_t* stage_floats,
                  int* n_degenerate);

/* y = A x for angles [a0, a1): y holds (a1-a0)*det_count samples, row a at
 * y + (a-a0)*det_count.  If b is non-NULL, writes y = b - A x instead (b laid
 * out like y).  work: ctk_geom_info().stage_floats fp32 scratch. */
int ctk_forward(const ctk_geom_t* g, const float* x, float* y, int a0, int a1,
                const float* b, float* work, void* stream);

/* Literal fp64 Siddon for every angle (same output layout, no work buffer). */
/* Exact adjoint of A (Siddon transpose; matched mode):
 * x = (x0 ? x0 : 0) + A^T u over angles [a0, a1).  Replaces
 * matched_back(forward) = CSR transpose, ctkrylov/ct.py:248-264.  `work` holds
 * ctk_adjoint_work_floats(g, a0, a1) floats (zero-filled once; may be NULL when
 * that is 0). */
int ctk_adjoint(const ctk_geom_t* g, const float* u, float* x, int a0, int a1,
                const float* x0, float* work, void* stream);
int64_t ctk_adjoint_work_floats(const ctk_geom_t* g, int a0, int a1);

int ctk_forward_exact(const ctk_geom_t* g, const float* x, float* y, int a0, int a1,
                      void* stream);

/* Kept segments (length > 1e-15, ct.py:178) and CSR nnz (duplicate (ray, pixel)
 * pairs merged, ct.py:197-200) over angles [a0, a1).  counts_dev: 2 int64 of
 * device memory, overwritten.  Synchronous-free: read back after the stream. */
int ctk_count_segments(const ctk_geom_t* g, int a0, int a1, int64_t* counts_dev,
                       void* stream);

/* x = (x0 ? x0 : 0) + B u, summing angles [a0, a1) (u row a at
 * u + (a-a0)*det_count).  work: ctk_back_work_floats() fp32 scratch,
 * zero-filled once: [K1 -> K2 chaining counters of the native BA Arnoldi
 * step][per-tile tickets][split partial images] -- counters and tickets at
 * offsets fixed by the geometry, so one buffer serves every angle range.  A
 * plain apply may pass NULL when the geometry needs no angle split. */
int64_t ctk_back_work_floats(const ctk_geom_t* g, int a0, int a1);
/* Layout of that buffer (introspection for protocol tests): out[0] = counter
 * words (one per 4-angle K1 group, padded), out[1] = ticket words (one per
 * K2 tile, padded), out[2] = K1 CTAs per group (a chained step j leaves every
 * group's counter at out[2] * (j + 1)), out[3] = K2 tiles. */
int ctk_back_work_layout(const ctk_geom_t* g, int64_t* out4);
int ctk_back(const ctk_geom_t* g, const float* u, float* x, int a0, int a1,
             const float* x0, float* work, void* stream);

/* ---- Krylov vector kernels.  W: basis rows of length L with row pitch ld
 * (floats, multiple of 4); device pointers throughout. */
size_t ctk_reduce_scratch_bytes(int nvec, int64_t L);

/* out[j] = <W_j, v> for j < nvec, and out[nvec] = <v, v> if want_norm. */
int ctk_dots(const float* W, int64_t ld, int nvec, const float* v, int64_t L,
             int want_norm, double* out, void* scratch, void* stream);
/* dst = v - sum_j coef[j] W_j   (dst may alias v); norm2_out[0] = ||dst||^2 if
 * norm2_out is non-NULL. */
int ctk_update(const float* W, int64_t ld, int nvec, const double* coef, const float* v,
               float* dst, int64_t L, double* norm2_out, void* scratch, void* stream);
/* out[0] = ||v||^2 (fp64). */
int ctk_norm2(const float* v, int64_t L, double* out, void* scratch, void* stream);
/* dst = v * (*scale_dev) with scale read on device. */
int ctk_scale(const float* v, float* dst, int64_t L, const double* scale_dev, void* stream);

/* One Arnoldi step's orthogonalisation (CGS2, equal in exact arithmetic to
 * the reference's MGS + reorthogonalisation, arnoldi.py:66-82):
 *   in : W rows 0..k (orthonormal basis), q = M w_k (overwritten)
 *   out: h[0..k+1] (k+2 fp64, device), stat[0] = ||M w_k||, stat[1] = breakdown
 *        flag (h[k+1] <= 1e-14 * ||M w_k||), and unless breakdown, row k+1 of W =
 *        q2 / h[k+1].  stat must hold 4 doubles. */
int ctk_cgs2_step(float* W, int64_t ld, int k, int64_t L, float* q, double* h,
                  double* stat, void* scratch, void* stream);
/* Same with passes = 2 (CGS2, reorthogonalize=True) or 1 (one classical
 * Gram-Schmidt pass, reorthogonalize=False; the reference's single pass is
 * modified Gram-Schmidt -- equal in exact arithmetic). */
int ctk_gs_step(float* W, int64_t ld, int k, int64_t L, float* q, int passes, double* h,
                double* stat, void* scratch, void* stream);

/* dst = (x0 ? x0 : 0) + sum_{j<k} y[j] W_j   (y: k fp64, device);
 * norm2_out[0] = ||dst||^2 if non-NULL. */
int ctk_combine(const float* W, int64_t ld, int k, const double* y, const float* x0,
                float* dst, int64_t L, double* norm2_out, void* scratch, void* stream);

/* ---- Native per-iteration orchestration of (hybrid) AB/BA-GMRES
 * (ctkrylov/gmres.py:186-211).  ab != 0: M = A B on sinograms (L = m);
 * ab == 0: M = B A on images (L = n).  stage_work / back_work as for
 * ctk_forward / ctk_back (one set per stream). */

/* Arnoldi step j: q = M W_j, CGS2 against rows 0..j, row j+1 written;
 * h_dev[0..hcols) receives h (j+2 values) with the 4 stats of
 * ctk_cgs2_step in its last 4 entries, copied asynchronously to h_host
 * (pinned) when non-NULL.  The intermediate goes to tmp, or is kept when
 * aux rows are given: BA: aux1[j] = A w_j; AB: aux1[j] = B w_j and
 * aux2[j] = A B w_j (before orthogonalisation).  Steps of one Arnoldi cycle
 * must be issued in order j = 0, 1, ... on the same stage_work: step j > 0
 * reuses the K1 staged copies that step j-1 (BA) or its own K2 (AB) wrote. */
int ctk_arnoldi_step(const ctk_geom_t* g, int ab, int passes, float* W, int64_t ld, int j,
                     float* q,
                     float* tmp, float* aux1, int64_t ld1, float* aux2, int64_t ld2,
                     float* stage_work, float* back_work, double* h_dev, int hcols,
                     double* h_host, void* scratch, void* stream);

/* Iterate k: y (k fp64; copied from pinned y_host when non-NULL) ->
 * x_k = x0 + W y (BA) or x0 + B (W y) (AB, z = m-length scratch);
 * r = b - A x_k; norms_dev[0] = ||r||^2, norms_dev[1] = ||x_k||^2.
 * With the aux rows kept by ctk_arnoldi_step and d0 = b - A x0, the same
 * x_k and r follow by linearity from two basis combinations and no projector
 * apply: x_k = x0 + sum y_j X_j, r = d0 - sum y_j (A X_j). */
int ctk_iterate(const ctk_geom_t* g, int ab, const float* W, int64_t ld, int k,
                const double* y_host, double* y_dev, const float* x0, float* xk, float* z,
                const float* b, float* r, double* norms_dev, const float* aux1, int64_t ld1,
                const float* aux2, int64_t ld2, const float* d0, float* stage_work,
                float* back_work, void* scratch, void* stream);

/* Batched iterate norms for nb (<= 8) consecutive iterations k0 .. k0+nb-1 of
 * one cycle (the linear iterate path of ctk_iterate): with y_b = y + b*ystride
 * (device, k0+b entries), norms[2b] = ||d0 - AX y_b||^2 and
 * norms[2b+1] = ||x0 + X y_b||^2, and the last iterate of the batch stored to
 * x / r (either may be NULL).  One pass over the basis for the whole batch.
 * scratch: ctk_reduce_scratch_bytes(nvec_cap, .) bytes, zero-filled once. */
int ctk_iterate_batch(const float* X, int64_t ldx, const float* x0, float* x, int64_t Lx,
                      const float* AX, int64_t ldax, const float* d0, float* r, int64_t Lr,
                      int k0, int nb, const double* y, int ystride, double* norms,
                      void* scratch, int nvec_cap, void* stream);

/* ---- Native (hybrid) AB-/BA-GMRES driver: the run_gmres loop
 * (ctkrylov/gmres.py:135-241) without Python per iteration.  Stopping rules
 * none / dp / rns; restarts; breakdown; degenerate-curve fallback.  All
 * buffers are caller-owned (device unless marked host/pinned). */
#define CTK_STOP_NONE 0
#define CTK_STOP_MAXITER 1
#define CTK_STOP_BREAKDOWN 2
#define CTK_STOP_DP 3
#define CTK_STOP_RNS 4

typedef struct {
    int ab;              /* 1: AB-GMRES (M = A B), 0: BA-GMRES (M = B A) */
    int hybrid;          /* 0: plain (lambda = 0) */
    int strategy;        /* 1 fixed, 2 lcurve, 3 gcv (hybrid only) */
    int max_iter;
    int restart_period;  /* 0: no restart */
    int stopping;        /* CTK_STOP_NONE / CTK_STOP_DP / CTK_STOP_RNS */
    int lookahead;       /* Arnoldi steps in flight ahead of the host (<= 0: 6) */
    double lambda_value, dp_tau, noise_norm, rns_epsilon;
    int reorthogonalize; /* 1: CGS2 (reference default), 0: single pass */
} ctk_solve_cfg;

typedef struct {
    float* W;            /* basis [rows][ld] */
    int64_t ld;
    int rows;            /* >= min(restart_period or max_iter, max_iter) + 1 */
    float *q, *tmp, *z, *r, *xk, *x_cur;   /* q: L, tmp: n (AB) / m (BA), z: m, r: m, xk/x_cur: n */
    const float* b;      /* m */
    float* aux1;         /* [rows][ld1]: A w_j (BA, ld1 >= m) or B w_j (AB, ld1 >= n); NULL = apply */
    int64_t ld1;
    float* aux2;         /* [rows][ld2]: A B w_j (AB, ld2 >= m) */
    int64_t ld2;
    float* d0;           /* m: b - A x0 of the current cycle (with aux) */
    double* hs;          /* [rows][hcols] device */
    double* h_host;      /* [rows][hcols] pinned host */
    int hcols;           /* >= rows + 5 */
    double* y_dev;       /* [max_iter][rows] */
    double* y_host;      /* [max_iter][rows] pinned host */
    double* norms;       /* [(max_iter + 1) * 2] device */
    double* norms_host;  /* same, pinned host */
    double* scal;        /* [4] device */
    double* scal_host;   /* [4] pinned host */
    float *stage_a, *back_a, *stage_b, *back_b;   /* projector workspaces per stream */
    void *scratch_a, *scratch_b;                  /* reduction scratch per stream */
    void *stream_a, *stream_b;                    /* Arnoldi / iterate streams */
    /* optional per-iteration records, NULL / 0 when unused */
    const float* x_true;  /* n: RRE / SSIM reference image */
    int img_nx, img_ny;   /* SSIM image shape (SSIM skipped when min < 8) */
    double dyn_range;     /* SSIM dynamic range L (max - min of x_true) */
    double* metrics;      /* [(max_iter + 1) * 2] device: ||x_k - x_true||^2, SSIM map sum */
    double* metrics_host; /* same, pinned host */
    void* scratch_m;      /* ctk_metrics_scratch_bytes() zero-filled */
    int snapshot_stride;  /* copy x_k to snaps[(k / stride) - 1] every stride iterations */
    float** snaps;        /* host pointers (pinned), n floats each */
    int n_snaps;
    /* angle-sharded solve (SURVEY row e): NULL = one GPU.  Otherwise g is this
     * rank's angle subset, b / d0 / r / aux rows of sinogram length hold this
     * rank's rows, images (x, BA basis) are replicated; the driver issues the
     * collectives itself (ctk_comm_*). */
    struct ctk_comm* comm;
} ctk_solve_bufs;

typedef struct {
    int n_records, stop_reason, cycles;
    int x_is_x0;         /* final iterate is x_cur (zero initial residual) else xk */
    int* k;              /* host arrays of length max_iter (+1) */
    int* warn;
    double *lambda, *residual, *data_residual, *proj_residual, *solution_norm, *elapsed;
    double *rre, *ssim;  /* with x_true (NaN when not computed) */
} ctk_solve_out;

int ctk_solve(const ctk_geom_t* g, const ctk_solve_cfg* cfg, ctk_solve_bufs* bufs,
              ctk_solve_out* out);

/* Device-side reconstruction metrics (ctkrylov/metrics.py:13-62):
 * out[0] = ||x - x_true||^2, out[1] = sum of the SSIM map over the valid
 * 8x8 Gaussian windows (divide by (nx-7)(ny-7)); SSIM skipped when nx or
 * ny < 8 or dyn_range <= 0.  scratch: ctk_metrics_scratch_bytes(), zeroed. */
size_t ctk_metrics_scratch_bytes(void);
int ctk_metrics(const float* x, const float* x_true, int nx, int ny, double dyn_range,
                double* out, void* scratch, void* stream);

/* ---- Angle-sharded B with the partial-image sum exchanged over peer memory
 * (SURVEY row e, N1; ctk_exchange.cu).  Replaces back_partial + all-reduce
 * of the sharded driver: each rank's K2 pushes its finished tiles into the
 * tile owner's receive buffer (owner = tile mod nranks; NVLink peer stores),
 * the owner sums them in rank order and delivers the tile to every rank.
 * The exchange owns its buffers (receive [nranks][n], result image [n],
 * flags); peers map them with CUDA IPC (export / connect_ipc) or, in one
 * process, connect with raw pointers (connect_ptrs).  At most 8 ranks. */
typedef struct ctk_xchg ctk_xchg_t;
int ctk_xchg_create(const ctk_geom_t* g, int rank, int nranks, ctk_xchg_t** out);
int ctk_xchg_destroy(ctk_xchg_t* x);
int ctk_xchg_local(const ctk_xchg_t* x, float** recv, float** img, unsigned** flags);
size_t ctk_xchg_handle_bytes(void);
int ctk_xchg_export(const ctk_xchg_t* x, void* handles);
int ctk_xchg_connect_ipc(ctk_xchg_t* x, const void* handles);
int ctk_xchg_connect_ptrs(ctk_xchg_t* x, float* const* recv, float* const* img,
                          unsigned* const* flags);
/* img (every rank) = sum over ranks of B_rank u_rank; g = this rank's angle
 * subset.  phases: bit 0 compute + push, bit 1 reduce owned tiles and
 * deliver, bit 2 wait for the other tiles (7 in a multi-GPU run).  epoch:
 * call counter (>= 1, equal on all ranks, increasing).  work: as ctk_back. */
int ctk_back_exchange(const ctk_geom_t* g, ctk_xchg_t* x, const float* u, unsigned epoch,
                      int phases, float* work, void* stream);
/* *timed_out = 1 when one of this rank's exchange waits gave up after ~20 s
 * (a peer never delivered); the word is cleared.  Synchronises the device. */
int ctk_xchg_status(ctk_xchg_t* x, int* timed_out);

/* ---- Communicator of the angle-sharded native solve (SURVEY row e;
 * ctk_comm.cu): libctk's own NCCL communicator (NCCL loaded at run time from
 * nccl_lib, e.g. the libnccl.so.2 torch uses; NULL: the default search),
 * optionally with a peer exchange for B's partial images.  Replaces the
 * reference's single-process loop (ctkrylov/gmres.py:186-211) across ranks:
 * A sharded by angle with a replicated image, B's partial images summed,
 * AB Krylov vectors sharded in measurement space (fp64 all-reduces of the
 * Gram-Schmidt dots and norms).  Rank 0 makes the id, every rank creates the
 * communicator with it (the caller ships the id bytes). */
typedef struct ctk_comm ctk_comm_t;
size_t ctk_comm_id_bytes(void);
int ctk_comm_unique_id(const char* nccl_lib, void* id_out);
int ctk_comm_create(const char* nccl_lib, const void* id, int nranks, int rank, int device,
                    ctk_comm_t** out);
int ctk_comm_destroy(ctk_comm_t* c);
int ctk_comm_attach_exchange(ctk_comm_t* c, ctk_xchg_t* x);
int ctk_comm_rank(const ctk_comm_t* c, int* rank, int* nranks);
/* In-place sum over ranks, stream-ordered; dtype 0 fp32, 1 fp64. */
int ctk_comm_allreduce(ctk_comm_t* c, void* buf, int64_t count, int dtype, void* stream);
/* x (every rank) = sum over ranks of B_rank u_rank, g = this rank's angles:
 * the peer exchange when attached (nranks > 1), else K2 + one all-reduce.
 * work: ctk_back_work_floats(g, 0, n_angles) floats, zero-filled once. */
int ctk_comm_back(ctk_comm_t* c, const ctk_geom_t* g, const float* u, float* x, float* work,
                  void* stream);

/* ---- On-device problem generation.
 * ctk_phantom replaces shepp_logan (ctkrylov/ct.py:115-134) and the harness's
 * random-ellipse recipe: img[iy*nx+ix] = sum over ellipses, in order, of
 * value_e where u^2 + v^2 <= 1, with (X, Y) = pixel centre / scale
 * (xc = xmin + (ix+0.5) h, yc = ymax - (iy+0.5) h, ct.py:60-66) and
 * u = ((X-x0) c + (Y-y0) s) / a, v = (-(X-x0) s + (Y-y0) c) / b -- the
 * reference's fp64 operation order, bitwise.  ellipses: HOST array of
 * n_ellipses x 7 doubles (value, a, b, x0, y0, cos phi, sin phi; at most 128);
 * img64 / img32 device outputs (either may be NULL). */
int ctk_phantom(int nx, int ny, double xmin, double ymax, double pixel_size, double scale,
                const double* ellipses, int n_ellipses, double* img64, float* img32,
                void* stream);
/* add_noise (ctkrylov/ct.py:267-283) on a device sinogram: clean data in
 * exactly one of b_clean (fp32) / b_clean64 (fp64); g = the m-sample
 * standard-normal draw (device fp64, numpy default_rng(seed) on the host);
 * noise_norm = level * ||b_clean||; b = b_clean + (noise_norm * g) / ||g||
 * into b64 / b32 (either may be NULL); noise_norm_dev[0] = noise_norm.
 * scratch: ctk_noise_scratch_bytes().  level 0 is the caller's copy. */
size_t ctk_noise_scratch_bytes(void);
int ctk_add_noise(const float* b_clean, const double* b_clean64, const double* g, int64_t m,
                  double level, double* b64, float* b32, double* noise_norm_dev, void* scratch,
                  void* stream);

/* CUDA-event profiler over library calls: kinds 0 = forward (stage + K1),
 * 1 = back (K2 + finalize), 2 = CGS2 step, 3 = basis combination.  end()
 * synchronises the recorded events and fills per-kind counts / mean / total. */
int ctk_profile_begin(void);
int ctk_profile_end(int nkinds, int64_t* counts, double* mean_ms, double* total_ms);

/* ---- Host fp64 projected problem (ctkrylov/regparam.py, arnoldi.py:95-141).
 * ctk_set_lapack registers LAPACK dgesdd and BLAS ddot (Fortran ABI, 32-bit
 * ints; ddot may be NULL).
 * ctk_projected_solve: H (k+1) x k row-major; strategy 0 none, 1 fixed,
 * 2 lcurve, 3 gcv; grid_count points (200 in the reference); on a degenerate
 * curve lambda = fallback_lambda (NaN: y left unset).  out = {lambda,
 * ||H y - beta e1||, degenerate flag, rank-deficient flag}; y: k doubles.
 * Thread-safe: no shared state beyond the registered function pointer. */
int ctk_set_lapack(void* dgesdd, void* ddot);
/* LAPACK dbdsqr for the lock-free path (bidiagonalisation in C++, singular
 * values with one rotated vector, Givens Tikhonov); without it every solve
 * uses dgesdd (serialised by OpenBLAS across threads). */
int ctk_set_lapack_extra(void* dbdsqr);
/* 0 (default): lock-free path; 1: always dgesdd, whose rounding reproduces
 * the reference's numpy SVD bit for bit (the L-curve corner is sensitive to
 * the last bits of the SVD). */
int ctk_set_svd_path(int lapack_only);
int ctk_projected_solve(const double* H, int k, double beta, int strategy, double fixed_value,
                        int grid_count, double fallback_lambda, double* out, double* y);

/* Host-side helpers to let drivers avoid a libcudart dependency. */
int ctk_device_count(int* out);
/* Total kernels this library has launched in the process (all threads). */
int64_t ctk_launch_counter(void);

#ifdef __cplusplus
}
#endif

#endif /* CTK_H_ */
