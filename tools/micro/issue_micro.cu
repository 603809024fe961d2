// Do non-FP64 instructions co-issue with the 2-cycle FP64 dispatch on B200?
// The Euler substep (14 FP64 ops) plus NX integer ops per substep.
#include <cstdio>
#include <cuda_runtime.h>

template <int NX>
__global__ void substep_x(double* out, int* iout, int n, double bp, double g, double mu, double h) {
    double S = 1e6 - threadIdx.x, I = 100.0 + blockIdx.x, R = 0.0, D = 0.0;
    unsigned a = threadIdx.x, b = blockIdx.x * 7 + 1;
    for (int k = 0; k < n; ++k) {
#pragma unroll
        for (int u = 0; u < 24; ++u) {
            const double inf = __dmul_rn(__dmul_rn(bp, S), I);
            const double gI = __dmul_rn(g, I);
            const double mI = __dmul_rn(mu, I);
            const double dI = __dsub_rn(__dsub_rn(inf, gI), mI);
            S = __dsub_rn(S, __dmul_rn(h, inf));
            I = __dadd_rn(I, __dmul_rn(h, dI));
            R = __dadd_rn(R, __dmul_rn(h, gI));
            D = __dadd_rn(D, __dmul_rn(h, mI));
#pragma unroll
            for (int x = 0; x < NX; ++x) {
                asm volatile("xor.b32 %0, %0, %1;" : "+r"(a) : "r"(b));
                asm volatile("add.u32 %0, %0, %1;" : "+r"(b) : "r"(a));
            }
        }
    }
    if (S + I + R + D == 1.2345) out[0] = S;
    if (a == 12345u) iout[0] = b;
}

template <int NX>
void run(double* d, int* di, int sms) {
    const int threads = 128, warps_per_sm = 32;
    const int blocks = sms * warps_per_sm * 32 / threads;
    const int iters = 200;
    substep_x<NX><<<blocks, threads>>>(d, di, 10, 1e-8, 0.1, 0.01, 1.0 / 24);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    substep_x<NX><<<blocks, threads>>>(d, di, iters, 1e-8, 0.1, 0.01, 1.0 / 24);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double ops = (double)blocks * threads * iters * 24 * 14;
    printf("14 FP64 + %2d int ops per substep: %.2f T fp64 lane-ops/s\n", 2 * NX, ops / (ms * 1e-3) / 1e12);
}

int main() {
    double* d; int* di;
    cudaMalloc(&d, 8); cudaMalloc(&di, 4);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0>(d, di, sms); run<1>(d, di, sms); run<2>(d, di, sms); run<3>(d, di, sms); run<4>(d, di, sms);
    run<5>(d, di, sms); run<7>(d, di, sms); run<10>(d, di, sms);
    return 0;
}
