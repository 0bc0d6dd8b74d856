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

extern "C" int ctk_arnoldi_step(const ctk_geom_t* g, int ab, float* W, int64_t ld, int j, float* q,
                                float* tmp, float* stage_work, float* back_work, double* h_dev,
                                int hcols, double* h_host, void* scratch, void* stream) {
    if (!g) return ctk_fail(CTK_ERR_ARG, "null geometry");
    if (hcols < j + 6) return ctk_fail(CTK_ERR_ARG, "h row too short (%d) for step %d", hcols, j);
    const int na = g->n_angles;
    const int64_t L = ab ? (int64_t)na * g->det_count : (int64_t)g->nx * g->ny;
    const float* w = W + (size_t)j * ld;
    int rc;
    if (ab) {   // q = A (B w)
        if ((rc = ctk_back(g, w, tmp, 0, na, nullptr, back_work, stream))) return rc;
        if ((rc = ctk_forward(g, tmp, q, 0, na, nullptr, stage_work, stream))) return rc;
    } else {    // q = B (A w)
        if ((rc = ctk_forward(g, w, tmp, 0, na, nullptr, stage_work, stream))) return rc;
        if ((rc = ctk_back(g, tmp, q, 0, na, nullptr, back_work, stream))) return rc;
    }
    cudaStream_t st = ctk_stream(stream);
    const int ph = ctk_prof_open(2, st);
    rc = ctk_cgs2_step(W, ld, j, L, q, h_dev, h_dev + hcols - 4, scratch, stream);
    ctk_prof_close(ph, st);
    if (rc) return rc;
    if (h_host)
        CTK_CUDA(cudaMemcpyAsync(h_host, h_dev, sizeof(double) * hcols, cudaMemcpyDeviceToHost, st));
    return CTK_OK;
}

extern "C" int ctk_iterate(const ctk_geom_t* g, int ab, const float* W, int64_t ld, int k,
                           const double* y_host, double* y_dev, const float* x0, float* xk,
                           float* z, const float* b, float* r, double* norms_dev,
                           float* stage_work, float* back_work, void* scratch, void* stream) {
    if (!g || !y_dev || !xk || !b || !r || !norms_dev) return ctk_fail(CTK_ERR_ARG, "null argument");
    const int na = g->n_angles;
    const int64_t n = (int64_t)g->nx * g->ny, m = (int64_t)na * g->det_count;
    cudaStream_t st = ctk_stream(stream);
    if (y_host && k > 0)
        CTK_CUDA(cudaMemcpyAsync(y_dev, y_host, sizeof(double) * k, cudaMemcpyHostToDevice, st));
    int rc;
    const int ph = ctk_prof_open(3, st);
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
