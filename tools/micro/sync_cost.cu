// Launch / grid-barrier cost microbenchmark (tools only, not the product).
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void k_empty(int* p) { if (p && threadIdx.x == 9999) *p = 1; }

template <int NS>
__global__ void k_coop(int* p) {
    cg::grid_group g = cg::this_grid();
#pragma unroll 1
    for (int i = 0; i < NS; ++i) g.sync();
    if (p && threadIdx.x == 9999) *p = 1;
}

// hand-rolled sense-free barrier: monotonically increasing counter
__device__ __forceinline__ void bar(unsigned* ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        atomicAdd(ctr, 1u);
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(v) : "l"(ctr));
        } while (v < target);
    }
    __syncthreads();
}

template <int NS>
__global__ void k_hand(unsigned* ctr, unsigned base) {
#pragma unroll 1
    for (int i = 0; i < NS; ++i) bar(ctr, base + (i + 1) * gridDim.x);
}

int main() {
    int* d; cudaMalloc(&d, 4);
    unsigned* ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int R = 200;
    auto time = [&](const char* name, auto fn) {
        for (int i = 0; i < 20; ++i) fn();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int i = 0; i < R; ++i) fn();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-40s %8.2f us/launch  (%s)\n", name, ms * 1e3 / R, cudaGetErrorString(cudaGetLastError()));
    };
    for (int G : {64, 148, 296}) {
        char nm[64];
        snprintf(nm, 64, "empty G=%d", G);
        time(nm, [&] { k_empty<<<G, 256>>>(nullptr); });
        int* np = nullptr;
        void* args[] = {&np};
        snprintf(nm, 64, "coop 0 sync G=%d", G);
        time(nm, [&] { cudaLaunchCooperativeKernel((void*)k_coop<0>, G, 256, args, 0, 0); });
        snprintf(nm, 64, "coop 1 sync G=%d", G);
        time(nm, [&] { cudaLaunchCooperativeKernel((void*)k_coop<1>, G, 256, args, 0, 0); });
        snprintf(nm, 64, "coop 5 sync G=%d", G);
        time(nm, [&] { cudaLaunchCooperativeKernel((void*)k_coop<5>, G, 256, args, 0, 0); });
        unsigned base = 0;
        cudaMemset(ctr, 0, 4);
        snprintf(nm, 64, "hand 5 bar G=%d", G);
        time(nm, [&] { k_hand<5><<<G, 256>>>(ctr, base); base += 5 * G; });
        cudaMemset(ctr, 0, 4); base = 0;
        snprintf(nm, 64, "hand 1 bar G=%d", G);
        time(nm, [&] { k_hand<1><<<G, 256>>>(ctr, base); base += G; });
    }
    return 0;
}
