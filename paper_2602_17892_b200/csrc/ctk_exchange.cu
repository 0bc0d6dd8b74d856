// ctk_exchange.cu -- angle-sharded B with the partial-image reduction done
// over peer memory instead of an all-reduce (SURVEY.md row e, N1).
//
// The reference applies B over all angles on one CPU (ctkrylov/ct.py:234-245).
// Sharded by angle over p GPUs, every rank back-projects its own angles into
// a full-size partial image that must be summed over ranks.  Here:
//   phase 1  K2 (k_back) with an exchange epilogue: each finished tile is
//            stored straight into the receive buffer of the tile's owner
//            (owner = tile mod p) -- a peer-memory store over NVLink when the
//            owner is another GPU -- followed by one system-scope release of
//            the tile's arrival flag.  Tiles leave while the rest compute.
//   phase 2  k_xchg_reduce: the owner waits (acquire) for the p partials of
//            each of its tiles, sums them in rank order in fp64 (so every
//            rank ends with bitwise the same image) and stores the tile into
//            every rank's result image, then releases their "done" flags.
//   phase 3  k_xchg_wait: a rank waits for the tiles it does not own.
// No kernel waits on work that could itself be waiting (phase 1 never
// waits; phase 2 waits only on phase 1, phase 3 only on phase 2), so there
// is no cross-GPU deadlock whatever the CTA scheduling.  Traffic per rank is
// that of a ring all-reduce, 2 (p-1)/p n floats, without a separate
// collective launch or its staging copies.  Flags carry the call's epoch, so
// nothing is reset between calls.
//
// Buffers are owned by the exchange object and shared across processes with
// CUDA IPC (ctk_xchg_export / ctk_xchg_connect_ipc); in one process (the
// single-GPU emulation used by the tests) peers connect with raw pointers.
#include <string.h>

#include "ctk_common.cuh"

struct ctk_xchg {
    int device, rank, nranks;
    int64_t n, tiles;
    float* recv;            // [nranks][n] partials received for the tiles this rank owns
    float* x;               // [n] result image
    unsigned* flags;        // arrive [nranks][tiles], done [tiles], error word
    ctk_xchg_args host;     // peer mappings
    ctk_xchg_args* dev;     // device copy for the kernels
    bool ipc_open[CTK_XCHG_MAX_RANKS][3];
};

namespace {

size_t flags_bytes(const ctk_xchg* x) {
    return sizeof(unsigned) * ((size_t)(x->nranks + 1) * (size_t)x->tiles + 1);
}

unsigned* err_word(const ctk_xchg* x) { return x->flags + (size_t)(x->nranks + 1) * x->tiles; }

int push_args(ctk_xchg* x) {
    CTK_CUDA(cudaMemcpy(x->dev, &x->host, sizeof(ctk_xchg_args), cudaMemcpyHostToDevice));
    return CTK_OK;
}

void close_ipc(ctk_xchg* x) {
    for (int q = 0; q < x->nranks; ++q) {
        void* p[3] = {x->host.recv[q], x->host.x[q], x->host.flags[q]};
        for (int b = 0; b < 3; ++b)
            if (x->ipc_open[q][b] && p[b]) cudaIpcCloseMemHandle(p[b]);
        for (int b = 0; b < 3; ++b) x->ipc_open[q][b] = false;
    }
}

}  // namespace

extern "C" int ctk_xchg_create(const ctk_geom_t* g, int rank, int nranks, ctk_xchg_t** out) {
    if (!g || !out) return ctk_fail(CTK_ERR_ARG, "null argument");
    *out = nullptr;
    if (nranks < 1 || nranks > CTK_XCHG_MAX_RANKS || rank < 0 || rank >= nranks)
        return ctk_fail(CTK_ERR_ARG, "rank %d of %d (at most %d ranks)", rank, nranks,
                        CTK_XCHG_MAX_RANKS);
    CTK_CUDA(cudaSetDevice(g->device));
    ctk_xchg* x = new ctk_xchg();
    memset(x, 0, sizeof(*x));
    x->device = g->device;
    x->rank = rank;
    x->nranks = nranks;
    x->n = (int64_t)g->nx * g->ny;
    x->tiles = ctk_back_tiles(g);
    cudaError_t e = cudaMalloc(&x->recv, sizeof(float) * (size_t)nranks * x->n);
    if (e == cudaSuccess) e = cudaMalloc(&x->x, sizeof(float) * (size_t)x->n);
    if (e == cudaSuccess) e = cudaMalloc(&x->flags, flags_bytes(x));
    if (e == cudaSuccess) e = cudaMemset(x->flags, 0, flags_bytes(x));
    if (e == cudaSuccess) e = cudaMalloc(&x->dev, sizeof(ctk_xchg_args));
    if (e != cudaSuccess) {
        cudaFree(x->recv);
        cudaFree(x->x);
        cudaFree(x->flags);
        cudaFree(x->dev);
        delete x;
        return ctk_check_cuda(e, "ctk_xchg_create");
    }
    x->host.rank = rank;
    x->host.nranks = nranks;
    x->host.tiles = (int)x->tiles;
    x->host.recv[rank] = x->recv;
    x->host.x[rank] = x->x;
    x->host.flags[rank] = x->flags;
    x->host.err = err_word(x);
    *out = x;
    return CTK_OK;
}

extern "C" int ctk_xchg_destroy(ctk_xchg_t* x) {
    if (!x) return CTK_OK;
    cudaSetDevice(x->device);
    cudaDeviceSynchronize();
    close_ipc(x);
    cudaFree(x->recv);
    cudaFree(x->x);
    cudaFree(x->flags);
    cudaFree(x->dev);
    delete x;
    return CTK_OK;
}

extern "C" int ctk_xchg_local(const ctk_xchg_t* x, float** recv, float** img, unsigned** flags) {
    if (!x) return ctk_fail(CTK_ERR_ARG, "null exchange");
    if (recv) *recv = x->recv;
    if (img) *img = x->x;
    if (flags) *flags = x->flags;
    return CTK_OK;
}

// *timed_out = 1 when a wait of this rank's exchange kernels gave up (the
// peers never delivered); clears the word.  Synchronises the device.
extern "C" int ctk_xchg_status(ctk_xchg_t* x, int* timed_out) {
    if (!x || !timed_out) return ctk_fail(CTK_ERR_ARG, "null argument");
    CTK_CUDA(cudaSetDevice(x->device));
    unsigned v = 0;
    CTK_CUDA(cudaMemcpy(&v, err_word(x), sizeof(v), cudaMemcpyDeviceToHost));
    *timed_out = v != 0;
    if (v) CTK_CUDA(cudaMemset(err_word(x), 0, sizeof(v)));
    return CTK_OK;
}

extern "C" size_t ctk_xchg_handle_bytes(void) { return 3 * sizeof(cudaIpcMemHandle_t); }

// handles: receive buffer, result image, flags (3 cudaIpcMemHandle_t).
extern "C" int ctk_xchg_export(const ctk_xchg_t* x, void* handles) {
    if (!x || !handles) return ctk_fail(CTK_ERR_ARG, "null argument");
    CTK_CUDA(cudaSetDevice(x->device));
    cudaIpcMemHandle_t* h = static_cast<cudaIpcMemHandle_t*>(handles);
    CTK_CUDA(cudaIpcGetMemHandle(&h[0], x->recv));
    CTK_CUDA(cudaIpcGetMemHandle(&h[1], x->x));
    CTK_CUDA(cudaIpcGetMemHandle(&h[2], x->flags));
    return CTK_OK;
}

// handles: nranks x 3 handles in rank order (this rank's own entry ignored).
extern "C" int ctk_xchg_connect_ipc(ctk_xchg_t* x, const void* handles) {
    if (!x || !handles) return ctk_fail(CTK_ERR_ARG, "null argument");
    CTK_CUDA(cudaSetDevice(x->device));
    close_ipc(x);
    const cudaIpcMemHandle_t* h = static_cast<const cudaIpcMemHandle_t*>(handles);
    for (int q = 0; q < x->nranks; ++q) {
        if (q == x->rank) continue;
        void* p[3] = {nullptr, nullptr, nullptr};
        for (int b = 0; b < 3; ++b) {
            CTK_CUDA(cudaIpcOpenMemHandle(&p[b], h[3 * q + b], cudaIpcMemLazyEnablePeerAccess));
            x->ipc_open[q][b] = true;
        }
        x->host.recv[q] = static_cast<float*>(p[0]);
        x->host.x[q] = static_cast<float*>(p[1]);
        x->host.flags[q] = static_cast<unsigned*>(p[2]);
    }
    return push_args(x);
}

// Same-process peers (single-GPU emulation): raw device pointers per rank.
extern "C" int ctk_xchg_connect_ptrs(ctk_xchg_t* x, float* const* recv, float* const* img,
                                     unsigned* const* flags) {
    if (!x || !recv || !img || !flags) return ctk_fail(CTK_ERR_ARG, "null argument");
    close_ipc(x);
    for (int q = 0; q < x->nranks; ++q) {
        x->host.recv[q] = recv[q];
        x->host.x[q] = img[q];
        x->host.flags[q] = flags[q];
    }
    return push_args(x);
}

// x(every rank) = sum over ranks of B_rank u_rank.  g: this rank's geometry
// (its own angles; the image is the same on every rank).  phases: bit 0
// compute + push, bit 1 reduce owned tiles + deliver, bit 2 wait for the
// rest (7 for a real multi-GPU call).  epoch: call counter, >= 1, equal on
// all ranks and increasing.
extern "C" int ctk_back_exchange(const ctk_geom_t* g, ctk_xchg_t* x, const float* u,
                                 unsigned epoch, int phases, float* work, void* stream) {
    if (!g || !x) return ctk_fail(CTK_ERR_ARG, "null argument");
    if (epoch == 0) return ctk_fail(CTK_ERR_ARG, "epoch must be >= 1");
    if ((int64_t)g->nx * g->ny != x->n || ctk_back_tiles(g) != x->tiles)
        return ctk_fail(CTK_ERR_SHAPE, "exchange built for another image size");
    for (int q = 0; q < x->nranks; ++q)
        if (!x->host.recv[q] || !x->host.x[q] || !x->host.flags[q])
            return ctk_fail(CTK_ERR_ARG, "exchange not connected to rank %d", q);
    CTK_CUDA(cudaSetDevice(g->device));
    cudaStream_t st = ctk_stream(stream);
    if (x->host.epoch != epoch) {
        x->host.epoch = epoch;
        CTK_CUDA(cudaMemcpyAsync(&x->dev->epoch, &x->host.epoch, sizeof(unsigned),
                                 cudaMemcpyHostToDevice, st));
    }
    int rc;
    if ((phases & 1) &&
        (rc = ctk_back_xc(g, u, x->x, 0, g->n_angles, nullptr, work, nullptr, x->dev, stream)))
        return rc;
    return ctk_xchg_finish(g, x->dev, x->nranks, phases, st);
}
