// ctk_common.cuh -- shared declarations for the B200 projector library.
//
// Layout conventions (reference: ctkrylov/ct.py:10-18):
//   image    row-major (ny, nx), row 0 = top (largest y), fp32
//   sinogram angle-major, sample a*D + j, fp32
//   Krylov basis W: [K+1][ld] fp32, ld a multiple of 4 (16-B rows)
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ctk.h"

namespace ctk {

// Per-angle forward (K1) parameters, computed once on the host in fp64.
// The ray for bin j meets walk-row boundary k at cross coordinate
//   u_k = (alpha + beta * s_j) + k * sigma      (pixel units, sigma in [0, 1])
// where a walk row is an image row (frame 0, |cos| >= |sin|) or an image
// column (frame 1), and "mirror" flips the cross axis so sigma >= 0.
struct AngleParams {
    double alpha, beta;     // u_0 = alpha + beta * s
    long long sigma_fx;     // sigma in 32.32 fixed point
    float L;                // chord per walk row  (h / |walk-axis cosine|)
    float Lx;               // chord per unit cross coordinate (h / |cross-axis cosine|)
    int frame;              // 0: walk rows of x, 1: walk columns (transposed copy)
    int mirror;             // cross axis reversed
    int degenerate;         // literal path: |sin| or |cos| < 1e-14 (ct.py:153-155,165,168) or < 1e-5 (ctk_geom.cu)
    int exact_flags;        // bit0: |dx| is a power of two, bit1: |dy| is (division == exact multiply)
    double inv_dx, inv_dy;  // 1/dx, 1/dy (used only when the matching bit is set)
    double inv_sg;          // 1 / sigma_fx (walk range estimates)
};

constexpr int CTK_MAX_DEG_LIST = 8;
constexpr int CTK_MAX_NEAR_AXIS = 16;   // near-axis (not exactly axis-aligned) angles on the literal path

struct BackParams {         // per angle for K2: g = X*cg + Y*sg + center
    double cg, sg;
};

}  // namespace ctk

struct ctk_geom {
    int device;
    int nx, ny, n_angles, det_count;
    double h, det_spacing;
    double xmin, xmax, ymin, ymax, center;
    int back_wmax;            // max staged bins per angle for one K2 tile
    int fwd_split;            // K1 row chunks per ray (small problems: more CTAs)
    int fwd_pad;              // K1 zero columns each side of P / PT (warp lockstep walk)
    int fwd_pair;             // K1 warps take 2 angles x 16 bins (CTK_FWD_PAIR=0: 1 x 32)
    int back_ppt;             // K2 pixels per thread (tile 32 x 8 ppt): 2, or 4 for >= 512^2
    int n_degenerate;
    int h_pow2;               // pixel size is a power of two: x / h == x * (1 / h) exactly
    double inv_h;
    int deg_list[ctk::CTK_MAX_DEG_LIST];   // degenerate angle indices (first CTK_MAX_DEG_LIST)
    // device tables
    ctk::AngleParams* d_ap;   // [n_angles]
    ctk::BackParams* d_bp;    // [n_angles]
    double* d_cos;            // [n_angles] bitwise np.cos (exact path)
    double* d_sin;            // [n_angles]
    double* d_offsets;        // [det_count] bitwise bin_offsets()
    // degenerate (axis-aligned) angles: literal-Siddon segment lists built once
    int* d_deg_slot;          // [n_angles] -> slot in the lists below, or -1
    long long* d_deg_ptr;     // [n_degenerate * det_count] kept segments per ray
    int* d_deg_pix;           // [n_degenerate][deg_maxseg][det_count] pixel index
    float* d_deg_len;         // same layout: exact fp64 length rounded to fp32
    long long deg_segments;
    int deg_maxseg;
    // K7 (exact adjoint): the lists above transposed to pixel -> (ray, length),
    // built on first use (ctk_adjoint.cu)
    long long* d_degt_ptr;    // [n_degenerate][n + 1]
    int* d_degt_ray;
    float* d_degt_len;
    int* d_degt_angle;        // slot -> angle index
};

// Builds the degenerate-angle segment lists (ctk_forward.cu); called by
// ctk_geom_create after the tables are on the device.
int ctk_build_degenerate_lists(ctk_geom* g);

// Kernel launches issued by the library (all threads); ctk_launch_counter().
void ctk_count_launch(int n = 1);

// CUDA-event profiler (ctk_solver.cu): kinds 0 forward, 1 back, 2 cgs2,
// 3 basis combination.  open returns -1 when profiling is off.
int ctk_prof_open(int kind, cudaStream_t st);
void ctk_prof_close(int handle, cudaStream_t st);

// error plumbing (thread-local last error string)
int ctk_fail(int code, const char* fmt, ...);
int ctk_check_cuda(cudaError_t e, const char* what);

#define CTK_CUDA(call)                                                 \
    do {                                                               \
        cudaError_t e_ = (call);                                       \
        if (e_ != cudaSuccess) return ctk_check_cuda(e_, #call);       \
    } while (0)

#define CTK_LAUNCH_CHECK(what)                                         \
    do {                                                               \
        ctk_count_launch();                                            \
        cudaError_t e_ = cudaGetLastError();                           \
        if (e_ != cudaSuccess) return ctk_check_cuda(e_, what);        \
    } while (0)

static inline cudaStream_t ctk_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// Programmatic dependent launch: kernels of the Arnoldi chain (K1, K2, K3)
// let their successor launch early (launch_dependents at entry) and the
// successor waits for its predecessor's memory only where it first reads
// it (griddepcontrol.wait), so its launch and set-up overlap the previous
// kernel's tail.  Both are no-ops without a programmatic launch.
// Last-arriver tickets (split reductions): after a __syncthreads() that
// orders every thread's partial stores before it, ONE thread releases them at
// gpu scope with the ticket increment (cumulativity covers the CTA's stores);
// the last arriver's thread acquires before its CTA reads the partials (.cg).
// Cheaper than a __threadfence() in every thread (MEMBAR.SC.GPU per warp).
__device__ __forceinline__ bool ctk_ticket_arrive(unsigned* ticket, unsigned arrivals) {
    unsigned old;
    asm volatile("atom.add.release.gpu.global.u32 %0, [%1], 1;" : "=r"(old) : "l"(ticket) : "memory");
    const bool last = old == arrivals - 1;
    if (last) asm volatile("fence.acq_rel.gpu;" ::: "memory");     // acquire the others' partials
    return last;
}

__device__ __forceinline__ unsigned ctk_ld_acquire_gpu(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void ctk_pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void ctk_pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;"); }

// cudaLaunchKernelEx with the programmatic-serialization attribute (plus an
// optional cluster shape).
template <typename... KArgs, typename... Args>
static inline cudaError_t ctk_launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                                         cudaStream_t st, dim3 cluster, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    int na = 0;
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
    if (cluster.x * cluster.y * cluster.z > 1) {
        at[na].id = cudaLaunchAttributeClusterDimension;
        at[na].val.clusterDim.x = cluster.x;
        at[na].val.clusterDim.y = cluster.y;
        at[na].val.clusterDim.z = cluster.z;
        ++na;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    return cudaLaunchKernelEx(&cfg, kern, args...);
}

// Peer exchange for angle-sharded B (SURVEY row e; ctk_exchange.cu): every
// rank's partial image is pushed tile by tile into the tile owner's receive
// buffer over peer memory, the owner sums its tiles in rank order and pushes
// the result to every rank.  Pointers are this process's mappings of each
// rank's buffers (CUDA IPC, or the same device in the single-GPU emulation).
constexpr int CTK_XCHG_MAX_RANKS = 8;
struct ctk_xchg_args {
    int rank, nranks, tiles;
    unsigned epoch;
    float* recv[CTK_XCHG_MAX_RANKS];      // rank q's receive buffer [nranks][n]
    float* x[CTK_XCHG_MAX_RANKS];         // rank q's result image [n]
    unsigned* flags[CTK_XCHG_MAX_RANKS];  // rank q's flags: arrive [nranks][tiles], done [tiles]
    unsigned* err;                         // this rank's error word: 1 = a wait timed out
};

// Bounded spin for the exchange's cross-GPU waits: a peer that never arrives
// (dead rank, mismatched call sequence) ends the wait after ~20 s with the
// error word set (reported by ctk_xchg_status / the sharded solve) instead of
// hanging every GPU of the job.
constexpr unsigned long long CTK_XCHG_TIMEOUT_NS = 20000000000ull;

// Destination of a fused K1 staging write (P / PT of an image vector).
struct ctk_stage_dst {
    float* P;
    float* PT;
    int nx, ny, pad;
};

// Internal variants used by the Arnoldi step (not part of the C ABI):
// GS step that also stages its new row for the next forward (SMEM path only),
// whether that path is taken for (L, k), forward over already-staged copies,
// back that also stages its output image.
// comm != NULL: the vectors are this rank's shard; dots and norms are summed
// over ranks between the launches (multi-kernel CGS2, stream-ordered NCCL).
int ctk_gs_step_ex(float* W, int64_t ld, int k, int64_t L, float* q, int passes, double* h,
                   double* stat, void* scratch, void* stream, const ctk_stage_dst* sd,
                   double* h_mirror, const ctk_comm* comm = nullptr);
int ctk_arnoldi_step_ex(const ctk_geom_t* g, int ab, int passes, float* W, int64_t ld, int j,
                        float* q, float* tmp, float* aux1, int64_t ld1, float* aux2, int64_t ld2,
                        float* stage_work, float* back_work, double* h_dev, int hcols,
                        double* h_host, void* scratch, void* stream, const ctk_comm* comm);
bool ctk_gs_smem_ok(int64_t L, int k);
// Streamed path (long vectors): also leaves q untouched and takes the stage /
// host-mirror outputs.  False whenever the SMEM path applies.
bool ctk_gs_stream_ok(int64_t L, int k);
int ctk_combine_pair(const float* X, int64_t ldx, const float* x0, float* x, int64_t Lx,
                     double* n_x, const float* AX, int64_t ldax, const float* d0, float* r,
                     int64_t Lr, double* n_r, int k, const double* y, void* scratch,
                     void* stream, const double* y_host);
bool ctk_iterate_batch_ok(int k0, int nb, int nvec_cap, int64_t Lx, int64_t Lr);
// K1 -> K2 chaining (BA Arnoldi step, q = B (A w)): K1 CTAs count finished
// 4-angle groups into flag words at the head of K2's work buffer (release),
// and K2 CTAs start each 32-angle chunk as soon as its groups are complete
// (acquire) instead of waiting for the whole of K1 -- K2 overlaps K1's last
// wave.  Deadlock-free: K2 is a programmatic dependent of K1, which triggers
// at entry, so every K1 CTA is resident or done before any K2 CTA can spin.
// The counters grow monotonically through a cycle (see wait_k1_groups).
#ifndef CTK_FWD_APB_N
#define CTK_FWD_APB_N 4
#endif
constexpr int CTK_FWD_APB = CTK_FWD_APB_N;     // angles per K1 CTA (one warp each)
unsigned* ctk_back_flags(const ctk_geom* g, float* work);
int ctk_forward_ex(const ctk_geom_t* g, const float* x, float* y, int a0, int a1, const float* b,
                   float* work, bool prestaged, void* stream, unsigned* done_flags = nullptr);
// k1_epoch > 0: chained after K1 (step j of an Arnoldi cycle passes j + 1;
// the caller zeroes the ctk_back_flag_count() flag words before step 0).
int ctk_back_ex(const ctk_geom_t* g, const float* u, float* x, int a0, int a1, const float* x0,
                float* work, float* stage, void* stream, unsigned k1_epoch = 0);
int ctk_back_xc(const ctk_geom_t* g, const float* u, float* x, int a0, int a1, const float* x0,
                float* work, float* stage, const ctk_xchg_args* xc, void* stream,
                unsigned k1_epoch = 0);
int64_t ctk_back_flag_count(const ctk_geom* g);
int ctk_xchg_finish(const ctk_geom* g, const ctk_xchg_args* xc, int nranks, int phases,
                    cudaStream_t st);
int64_t ctk_back_tiles(const ctk_geom* g);

// Angle-sharded solve (ctk_comm.cu): stream-ordered fp64 sums over ranks and
// B summed over ranks (peer exchange or all-reduce).
int ctk_comm_sum_f64(const ctk_comm* c, double* buf, int64_t count, cudaStream_t st);
int ctk_comm_back_sum(const ctk_comm* c, const ctk_geom* g, const float* u, float* dst,
                      float* work, cudaStream_t st);
int ctk_comm_size(const ctk_comm* c);
int ctk_comm_check(const ctk_comm* c);
int ctk_comm_rank_of(const ctk_comm* c);

// K1 workspace: zero-padded copies P, PT
// and one arrival ticket per (angle, 128-bin block) -- zero-filled once.
static inline int64_t ctk_stage_floats(const ctk_geom* g) {
    return (int64_t)g->ny * (g->nx + 2 * g->fwd_pad) + (int64_t)g->nx * (g->ny + 2 * g->fwd_pad);
}
