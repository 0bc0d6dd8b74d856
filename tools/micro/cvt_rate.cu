// Throughput of fp32 -> fp64 widening (F2F.F64.F32) and DFMA on one SM set,
// in results per clock per SM.  nvcc -arch=sm_100a -o cvt_rate cvt_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>   // 0: F2F + DADD chain-free, 1: DFMA only, 2: integer widening + DADD
__global__ void k(const float* in, double* out, int iters) {
    float x[8];
    for (int i = 0; i < 8; ++i) x[i] = in[threadIdx.x + 32 * i];
    double a[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) {
                double d;
                asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(x[i]));
                a[i] += d;
            } else if (MODE == 1) {
                a[i] = fma(a[i], 1.0000001, 0.5);
            } else {
                const unsigned b = __float_as_uint(x[i]);
                const unsigned hi = (b & 0x80000000u) | (((b & 0x7fffffffu) >> 3) + 0x38000000u);
                const unsigned lo = b << 29;
                a[i] += __hiloint2double((int)hi, (int)lo);
                x[i] = __uint_as_float(b + 1);
            }
        }
    }
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MODE>
void run(const char* name, int threads) {
    float* in; double* out;
    cudaMalloc(&in, 4096 * 4); cudaMemset(in, 0x3f, 4096 * 4);
    cudaMalloc(&out, 148 * 1024 * 8);
    const int iters = 20000;
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    k<MODE><<<148, threads>>>(in, out, 10);
    cudaEventRecord(e0);
    k<MODE><<<148, threads>>>(in, out, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    int mhz; cudaDeviceGetAttribute(&mhz, cudaDevAttrClockRate, 0);
    const double ops = (double)iters * 8 * threads;            // per SM
    printf("%s threads=%d: %.2f results/clk/SM (at %d MHz nominal), %.3f ms\n", name, threads,
           ops / (ms * 1e-3 * mhz * 1e3), mhz / 1000, ms);
}

int main() {
    for (int t : {128, 512, 1024}) {
        if (t == 128) { run<0>("F2F.F64.F32+DADD", 128); run<1>("DFMA", 128); run<2>("int widen+DADD", 128); }
        if (t == 512) { run<0>("F2F.F64.F32+DADD", 512); run<1>("DFMA", 512); run<2>("int widen+DADD", 512); }
        if (t == 1024) { run<0>("F2F.F64.F32+DADD", 1024); run<1>("DFMA", 1024); run<2>("int widen+DADD", 1024); }
    }
    return 0;
}
