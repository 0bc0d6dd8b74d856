// ctk_comm.cu -- libctk's own communicator for the angle-sharded solve
// (SURVEY row e): NCCL, loaded at run time, plus the optional peer-memory
// exchange for B's partial images (ctk_exchange.cu).
//
// The sharded native driver (ctk_solve with bufs->comm) issues every
// collective itself, stream-ordered on the Arnoldi / iterate streams, so a
// sharded Arnoldi step needs no host round trip:
//   * B's partial image (n fp32, every B apply): the peer exchange fused into
//     K2 when the ranks mapped each other's buffers, else one ncclAllReduce;
//   * AB's measurement-space dots (h1 with ||q||^2, h2, ||q2||^2 of a CGS2
//     step) and the residual norms: ncclAllReduce of a few fp64 values.
// NCCL reduces every element on one rank and broadcasts it, so all ranks hold
// bitwise the same sums (the replicated Hessenberg needs that: lambda and
// the Tikhonov solve run redundantly on every rank, no broadcast).
//
// NCCL is dlopen'ed (the single-GPU library does not depend on it); pass the
// path of the libnccl.so.2 the process already uses (torch's) so that one
// NCCL instance serves both.
#include <dlfcn.h>
#include <string.h>

#include <mutex>

#include <nccl.h>

#include "ctk_common.cuh"

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    void* handle = nullptr;
};

std::mutex g_nccl_mu;
NcclApi g_nccl;

int nccl_load(const char* path) {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.handle) return CTK_OK;
    void* h = dlopen(path && path[0] ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return ctk_fail(CTK_ERR_ARG, "cannot load NCCL (%s): %s", path ? path : "libnccl.so.2",
                            dlerror());
    NcclApi a;
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(dlsym(h, "ncclAllReduce"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    if (!a.get_unique_id || !a.comm_init_rank || !a.all_reduce || !a.comm_destroy) {
        dlclose(h);
        return ctk_fail(CTK_ERR_ARG, "NCCL library lacks the expected symbols");
    }
    a.handle = h;
    g_nccl = a;
    return CTK_OK;
}

int nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return CTK_OK;
    return ctk_fail(CTK_ERR_CUDA, "%s: NCCL error %d (%s)", what, (int)r,
                    g_nccl.error_string ? g_nccl.error_string(r) : "?");
}

}  // namespace

struct ctk_comm {
    int rank, nranks, device;
    ncclComm_t nc;
    ctk_xchg_t* xchg;        // optional peer exchange for B (not owned)
    unsigned epoch;          // exchange call counter (same sequence on every rank)
};

extern "C" int ctk_comm_unique_id(const char* nccl_lib, void* id_out) {
    if (!id_out) return ctk_fail(CTK_ERR_ARG, "null id");
    int rc = nccl_load(nccl_lib);
    if (rc) return rc;
    ncclUniqueId id;
    if ((rc = nccl_check(g_nccl.get_unique_id(&id), "ncclGetUniqueId"))) return rc;
    memcpy(id_out, &id, sizeof(id));
    return CTK_OK;
}

extern "C" size_t ctk_comm_id_bytes(void) { return sizeof(ncclUniqueId); }

extern "C" int ctk_comm_create(const char* nccl_lib, const void* id, int nranks, int rank,
                               int device, ctk_comm_t** out) {
    if (!id || !out) return ctk_fail(CTK_ERR_ARG, "null argument");
    *out = nullptr;
    if (nranks < 1 || rank < 0 || rank >= nranks)
        return ctk_fail(CTK_ERR_ARG, "rank %d of %d", rank, nranks);
    int rc = nccl_load(nccl_lib);
    if (rc) return rc;
    CTK_CUDA(cudaSetDevice(device));
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t nc = nullptr;
    if ((rc = nccl_check(g_nccl.comm_init_rank(&nc, nranks, uid, rank), "ncclCommInitRank")))
        return rc;
    ctk_comm* c = new ctk_comm();
    c->rank = rank;
    c->nranks = nranks;
    c->device = device;
    c->nc = nc;
    c->xchg = nullptr;
    c->epoch = 0;
    *out = c;
    return CTK_OK;
}

extern "C" int ctk_comm_destroy(ctk_comm_t* c) {
    if (!c) return CTK_OK;
    cudaSetDevice(c->device);
    cudaDeviceSynchronize();
    if (c->nc) g_nccl.comm_destroy(c->nc);
    delete c;
    return CTK_OK;
}

extern "C" int ctk_comm_attach_exchange(ctk_comm_t* c, ctk_xchg_t* x) {
    if (!c) return ctk_fail(CTK_ERR_ARG, "null communicator");
    c->xchg = x;
    return CTK_OK;
}

extern "C" int ctk_comm_rank(const ctk_comm_t* c, int* rank, int* nranks) {
    if (!c) return ctk_fail(CTK_ERR_ARG, "null communicator");
    if (rank) *rank = c->rank;
    if (nranks) *nranks = c->nranks;
    return CTK_OK;
}

// In-place sum over ranks, stream-ordered.  dtype 0: fp32, 1: fp64.
extern "C" int ctk_comm_allreduce(ctk_comm_t* c, void* buf, int64_t count, int dtype,
                                  void* stream) {
    if (!c || (!buf && count > 0)) return ctk_fail(CTK_ERR_ARG, "null argument");
    if (count <= 0) return CTK_OK;
    return nccl_check(g_nccl.all_reduce(buf, buf, (size_t)count,
                                        dtype == 1 ? ncclFloat64 : ncclFloat32, ncclSum, c->nc,
                                        ctk_stream(stream)),
                      "ncclAllReduce");
}

int ctk_comm_sum_f64(const ctk_comm* c, double* buf, int64_t count, cudaStream_t st) {
    return ctk_comm_allreduce(const_cast<ctk_comm*>(c), buf, count, 1, st);
}

// dst = sum over ranks of B_rank u_rank (this rank's angles in g).  With the
// peer exchange: K2 pushes tiles to their owners, owners reduce in rank order
// and deliver (ctk_back_exchange), then the result image is copied to dst.
// Otherwise: K2 into dst, then one fp32 all-reduce.
int ctk_comm_back_sum(const ctk_comm* cc, const ctk_geom* g, const float* u, float* dst,
                      float* work, cudaStream_t st) {
    ctk_comm* c = const_cast<ctk_comm*>(cc);
    const int64_t n = (int64_t)g->nx * g->ny;
    int rc;
    if (c->xchg && c->nranks > 1) {
        float* img = nullptr;
        if ((rc = ctk_xchg_local(c->xchg, nullptr, &img, nullptr))) return rc;
        if ((rc = ctk_back_exchange(g, c->xchg, u, ++c->epoch, 7, work, st))) return rc;
        CTK_CUDA(cudaMemcpyAsync(dst, img, sizeof(float) * n, cudaMemcpyDeviceToDevice, st));
        return CTK_OK;
    }
    if ((rc = ctk_back_ex(g, u, dst, 0, g->n_angles, nullptr, work, nullptr, st))) return rc;
    return ctk_comm_allreduce(c, dst, n, 0, st);        // (a no-op copy at one rank)
}

// After a sharded solve: did any bounded exchange wait give up?
int ctk_comm_check(const ctk_comm* c) {
    if (!c || !c->xchg) return CTK_OK;
    int timed_out = 0;
    int rc = ctk_xchg_status(c->xchg, &timed_out);
    if (rc) return rc;
    if (timed_out)
        return ctk_fail(CTK_ERR_CUDA, "peer exchange: a rank's partial image never arrived "
                                      "(wait timed out; ranks out of step or a peer died)");
    return CTK_OK;
}

extern "C" int ctk_comm_back(ctk_comm_t* c, const ctk_geom_t* g, const float* u, float* x,
                             float* work, void* stream) {
    if (!c || !g || !u || !x) return ctk_fail(CTK_ERR_ARG, "null argument");
    CTK_CUDA(cudaSetDevice(g->device));
    return ctk_comm_back_sum(c, g, u, x, work, ctk_stream(stream));
}

int ctk_comm_size(const ctk_comm* c) { return c ? c->nranks : 1; }
int ctk_comm_rank_of(const ctk_comm* c) { return c ? c->rank : 0; }
