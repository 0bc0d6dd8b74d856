// ctk_solver.cu -- native per-iteration orchestration of hybrid GMRES and a
// CUDA-event profiler for the projector kernels.
//
// ctk_arnoldi_step / ctk_iterate enqueue, in one C call, everything one
// Arnoldi step / one iterate update of run_gmres needs (reference loop:
// ctkrylov/gmres.py:186-211, arnoldi.py:64-82), so the Python driver pays one
// FFI crossing per step instead of a dozen launches through ctypes.
#include <math.h>

#include <mutex>
#include <vector>

#include "ctk_common.cuh"

namespace {

struct ProfRec {
    int kind;
    cudaEvent_t e0, e1;
};

std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<ProfRec> g_prof;

}  // namespace

int ctk_prof_open(int kind, cudaStream_t st) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (!g_prof_on) return -1;
    ProfRec r;
    r.kind = kind;
    if (cudaEventCreate(&r.e0) != cudaSuccess) return -1;
    if (cudaEventCreate(&r.e1) != cudaSuccess) {
        cudaEventDestroy(r.e0);
        return -1;
    }
    cudaEventRecord(r.e0, st);
    g_prof.push_back(r);
    return (int)g_prof.size() - 1;
}

void ctk_prof_close(int handle, cudaStream_t st) {
    if (handle < 0) return;
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (handle < (int)g_prof.size()) cudaEventRecord(g_prof[handle].e1, st);
}

static void prof_clear() {
    for (auto& r : g_prof) {
        cudaEventDestroy(r.e0);
        cudaEventDestroy(r.e1);
    }
    g_prof.clear();
}

extern "C" int ctk_profile_begin(void) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    prof_clear();
    g_prof_on = true;
    return CTK_OK;
}

extern "C" int ctk_profile_end(int nkinds, int64_t* counts, double* mean_ms, double* total_ms) {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    g_prof_on = false;
    for (int k = 0; k < nkinds; ++k) {
        if (counts) counts[k] = 0;
        if (mean_ms) mean_ms[k] = 0.0;
        if (total_ms) total_ms[k] = 0.0;
    }
    for (auto& r : g_prof) {
        if (r.kind < 0 || r.kind >= nkinds) continue;
        if (cudaEventSynchronize(r.e1) != cudaSuccess) {
            prof_clear();
            return ctk_check_cuda(cudaGetLastError(), "ctk_profile_end");
        }
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.e0, r.e1);
        if (counts) counts[r.kind] += 1;
        if (total_ms) total_ms[r.kind] += ms;
    }
    for (int k = 0; k < nkinds; ++k)
        if (mean_ms && counts && counts[k]) mean_ms[k] = (total_ms ? total_ms[k] : 0.0) / counts[k];
    prof_clear();
    return CTK_OK;
}

extern "C" int ctk_arnoldi_step(const ctk_geom_t* g, int ab, int passes, float* W, int64_t ld,
                                int j, float* q,
                                float* tmp, float* aux1, int64_t ld1, float* aux2, int64_t ld2,
                                float* stage_work, float* back_work, double* h_dev, int hcols,
                                double* h_host, void* scratch, void* stream) {
    return ctk_arnoldi_step_ex(g, ab, passes, W, ld, j, q, tmp, aux1, ld1, aux2, ld2, stage_work,
                               back_work, h_dev, hcols, h_host, scratch, stream, nullptr);
}

// comm != NULL: angle-sharded step (g = this rank's angles).  B's partial
// images are summed over ranks (ctk_comm_back_sum) before anything reads
// them; AB's Krylov vectors are this rank's sinogram rows, so the
// Gram-Schmidt dots and norms are summed over ranks too (ctk_gs_step_ex);
// BA's are replicated images and orthogonalise locally.
int ctk_arnoldi_step_ex(const ctk_geom_t* g, int ab, int passes, float* W, int64_t ld, int j,
                        float* q, float* tmp, float* aux1, int64_t ld1, float* aux2, int64_t ld2,
                        float* stage_work, float* back_work, double* h_dev, int hcols,
                        double* h_host, void* scratch, void* stream, const ctk_comm* comm) {
    if (!g) return ctk_fail(CTK_ERR_ARG, "null geometry");
    if (hcols < j + 6) return ctk_fail(CTK_ERR_ARG, "h row too short (%d) for step %d", hcols, j);
    const int na = g->n_angles;
    const int64_t n = (int64_t)g->nx * g->ny, m = (int64_t)na * g->det_count;
    const int64_t L = ab ? m : n;
    const float* w = W + (size_t)j * ld;
    cudaStream_t st = ctk_stream(stream);
    int rc;
    // K1 staging is fused into the producer of the forward's input where it
    // can be: AB stages B w_j in K2's epilogue; BA stages w_{j+1} in the SMEM
    // Gram-Schmidt step of step j (so step j+1 skips it).  Step 0 always runs
    // the staging kernel, which also writes the zero padding.
    const float* pre_w = nullptr;                          // GS input when q is not copied
    ctk_stage_dst sd = {stage_work, stage_work + (size_t)g->ny * (g->nx + 2 * g->fwd_pad),
                        g->nx, g->ny, g->fwd_pad};
    // both single-launch Gram-Schmidt paths leave q untouched, stage w_{j+1}
    // for K1 and write the host-mapped column
    const bool gs_smem = (ctk_gs_smem_ok(L, j) || ctk_gs_stream_ok(L, j)) && !(ab && comm);
    if (ab) {   // q = A (B w); keep B w_j (aux1) and A B w_j (aux2) for the iterates
        float* bw = aux1 ? aux1 + (size_t)j * ld1 : tmp;
        float* abw = aux2 ? aux2 + (size_t)j * ld2 : q;
        // K2's epilogue stages B w_j for K1 -- not when B w_j is a partial
        // image still to be summed over ranks (k_stage then runs in K1's launch)
        const bool fuse = j > 0 && !comm;
        if (comm) {
            if ((rc = ctk_comm_back_sum(comm, g, w, bw, back_work, st))) return rc;
        } else if ((rc = ctk_back_ex(g, w, bw, 0, na, nullptr, back_work,
                                     fuse ? stage_work : nullptr, stream))) {
            return rc;
        }
        if ((rc = ctk_forward_ex(g, bw, abw, 0, na, nullptr, stage_work, fuse, stream))) return rc;
        // the SMEM Gram-Schmidt path leaves its input untouched: no copy of A B w_j
        if (aux2 && !gs_smem)
            CTK_CUDA(cudaMemcpyAsync(q, abw, sizeof(float) * m, cudaMemcpyDeviceToDevice, st));
        if (aux2 && gs_smem) pre_w = abw;
    } else {    // q = B (A w); keep A w_j (aux1)
        float* aw = aux1 ? aux1 + (size_t)j * ld1 : tmp;
        const bool pre = j > 0 && (ctk_gs_smem_ok(L, j - 1) || ctk_gs_stream_ok(L, j - 1));
        // K2 starts each angle chunk as soon as K1 has finished its rows
        // (chaining flags at the head of back_work; CTK_NO_CHAIN=1 disables)
        static const bool chain = [] {
            const char* e = getenv("CTK_NO_CHAIN");
            return !(e && e[0] == '1');
        }();
        // only where K1's last wave is a large share of it (a few waves of
        // K1 CTAs); at c5 (~35 waves) the early K2 CTAs would just spin
        const int64_t k1_ctas = (int64_t)((g->det_count + 31) / 32) *
                                ((na + CTK_FWD_APB - 1) / CTK_FWD_APB) * g->fwd_split;
        const bool ch = chain && back_work && k1_ctas <= 4 * 8 * 148 && !comm;
        // monotonic counters: zeroed (stream-ordered) before a cycle's step 0,
        // step j's K2 waits for (j + 1) K1 passes per group
        if (ch && j == 0)
            CTK_CUDA(cudaMemsetAsync(ctk_back_flags(g, back_work), 0,
                                     sizeof(unsigned) * (size_t)ctk_back_flag_count(g), st));
        if ((rc = ctk_forward_ex(g, w, aw, 0, na, nullptr, stage_work, pre, stream,
                                 ch ? ctk_back_flags(g, back_work) : nullptr)))
            return rc;
        if (comm) {
            if ((rc = ctk_comm_back_sum(comm, g, aw, q, back_work, st))) return rc;
        } else if ((rc = ctk_back_ex(g, aw, q, 0, na, nullptr, back_work, nullptr, stream,
                                     ch ? (unsigned)(j + 1) : 0u))) {
            return rc;
        }
    }
    // The SMEM Gram-Schmidt step writes the column straight into the
    // page-locked host row (mapped, UVA) -- no D2H copy on the critical stream.
    double* hm = nullptr;
    if (h_host && gs_smem && cudaHostGetDevicePointer((void**)&hm, h_host, 0) != cudaSuccess) {
        cudaGetLastError();
        hm = nullptr;
    }
    const int ph = ctk_prof_open(2, st);
    rc = ctk_gs_step_ex(W, ld, j, L, pre_w ? const_cast<float*>(pre_w) : q, passes, h_dev,
                        h_dev + hcols - 4, scratch, stream, ab ? nullptr : &sd, hm,
                        ab ? comm : nullptr);
    ctk_prof_close(ph, st);
    if (rc) return rc;
    if (h_host && !hm)
        CTK_CUDA(cudaMemcpyAsync(h_host, h_dev, sizeof(double) * hcols, cudaMemcpyDeviceToHost, st));
    return CTK_OK;
}

extern "C" int ctk_iterate(const ctk_geom_t* g, int ab, const float* W, int64_t ld, int k,
                           const double* y_host, double* y_dev, const float* x0, float* xk,
                           float* z, const float* b, float* r, double* norms_dev,
                           const float* aux1, int64_t ld1, const float* aux2, int64_t ld2,
                           const float* d0, float* stage_work, float* back_work, void* scratch,
                           void* stream) {
    if (!g || !y_dev || !xk || !b || !r || !norms_dev) return ctk_fail(CTK_ERR_ARG, "null argument");
    const int na = g->n_angles;
    const int64_t n = (int64_t)g->nx * g->ny, m = (int64_t)na * g->det_count;
    cudaStream_t st = ctk_stream(stream);
    int rc;
    const bool linear = aux1 && d0 && (!ab || aux2);
    // the linear path takes y in the kernel parameters (no H2D copy) when k is small
    if (y_host && k > 0 && !(linear && k <= 160))
        CTK_CUDA(cudaMemcpyAsync(y_dev, y_host, sizeof(double) * k, cudaMemcpyHostToDevice, st));
    const int ph = ctk_prof_open(3, st);
    if (linear) {
        // By linearity: x_k = x0 + sum y_j X_j with X_j = w_j (BA) or B w_j (AB),
        // A x_k = A x0 + sum y_j A X_j with A X_j kept by the Arnoldi steps, so
        // r = d0 - sum y_j (A X_j) needs no projector apply (d0 = b - A x0).
        const float* Xr = ab ? aux1 : W;
        const int64_t ldx = ab ? ld1 : ld;
        const float* AXr = ab ? aux2 : aux1;
        const int64_t ldax = ab ? ld2 : ld1;
        rc = ctk_combine_pair(Xr, ldx, x0, xk, n, norms_dev + 1, AXr, ldax, d0, r, m, norms_dev, k,
                              y_dev, scratch, stream, y_host);
        ctk_prof_close(ph, st);
        return rc;
    }
    if (ab) {   // x_k = x0 + B (W y)
        if (!z) return ctk_fail(CTK_ERR_ARG, "AB iterate needs z");
        if ((rc = ctk_combine(W, ld, k, y_dev, nullptr, z, m, nullptr, scratch, stream))) return rc;
        ctk_prof_close(ph, st);
        if ((rc = ctk_back(g, z, xk, 0, na, x0, back_work, stream))) return rc;
        if ((rc = ctk_norm2(xk, n, norms_dev + 1, scratch, stream))) return rc;
    } else {    // x_k = x0 + W y
        if ((rc = ctk_combine(W, ld, k, y_dev, x0, xk, n, norms_dev + 1, scratch, stream)))
            return rc;
        ctk_prof_close(ph, st);
    }
    // true residual r = b - A x_k and its norm
    if ((rc = ctk_forward(g, xk, r, 0, na, b, stage_work, stream))) return rc;
    return ctk_norm2(r, m, norms_dev, scratch, stream);
}
