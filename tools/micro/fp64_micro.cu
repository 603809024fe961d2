// FP64 microbenchmarks on B200 (tools only): dependent-op latency and the
// throughput of the Euler substep's dependency structure vs warps per SM.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_dadd(double* out, long long* cyc, int n, double a) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}
__global__ void lat_dmul(double* out, long long* cyc, int n, double a) {
    double x = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) x = __dmul_rn(x, a);
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; cyc[0] = t1 - t0; }
}

// The exact operation structure of euler_substep (14 ops, 6-deep chain).
__global__ void substep_tp(double* out, int n, double bp, double g, double mu, double h) {
    double S = 1e6 - threadIdx.x, I = 100.0 + blockIdx.x, R = 0.0, D = 0.0;
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
        }
    }
    if (S + I + R + D == 1.2345) out[0] = S;
}

int main() {
    double* d; long long* c;
    cudaMalloc(&d, 8); cudaMalloc(&c, 8);
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    const int n = 1 << 16;
    long long cyc;
    lat_dadd<<<1, 32>>>(d, c, n, 1.0000001); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.2f cycles\n", (double)cyc / n);
    lat_dmul<<<1, 32>>>(d, c, n, 0.9999999); cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.2f cycles\n", (double)cyc / n);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps_per_sm : {4, 8, 12, 16, 20, 24, 32, 48, 64}) {
        const int threads = 128;
        const int blocks = sms * warps_per_sm * 32 / threads;
        const int iters = 200;
        substep_tp<<<blocks, threads>>>(d, 10, 1e-8, 0.1, 0.01, 1.0 / 24);
        cudaEventRecord(e0);
        substep_tp<<<blocks, threads>>>(d, iters, 1e-8, 0.1, 0.01, 1.0 / 24);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        const double ops = (double)blocks * threads * iters * 24 * 14;
        printf("substep structure, %2d warps/SM: %.2f T lane-ops/s\n", warps_per_sm, ops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
