// Microbenchmark: DMMA m8n8k4 rate vs independent accumulator chains per warp
// and warps per SM (how much parallelism the fp64 tensor pipe needs), the
// dependent-chain latency, and DMMA + DFMA issued by different warps at once
// (do they share a pipe?).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_kernel(double* out, int iters) {
    double d[CHAINS][2];
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = 0;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// warps with even index issue DMMA chains, odd ones DFMA chains
__global__ void mixed_kernel(double* out, int iters) {
    const int warp = threadIdx.x >> 5;
    double s = 0;
    if (warp & 1) {
        double acc[8];
        double x = 1.0 + threadIdx.x * 1e-9, y = 0.999999;
#pragma unroll
        for (int c = 0; c < 8; ++c) acc[c] = c;
        for (int i = 0; i < iters * 4; ++i)
#pragma unroll
            for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], y, x);
#pragma unroll
        for (int c = 0; c < 8; ++c) s += acc[c];
    } else {
        double d[4][2] = {};
        double a = 1.0 + threadIdx.x * 1e-9, b = 0.5;
        for (int i = 0; i < iters; ++i)
#pragma unroll
            for (int c = 0; c < 4; ++c)
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                             : "+d"(d[c][0]), "+d"(d[c][1]) : "d"(a), "d"(b));
#pragma unroll
        for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int CHAINS>
float run(double* out, int warps_per_sm, int sms, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int threads = warps_per_sm * 32 > 1024 ? 1024 : warps_per_sm * 32;
    const int blocks = sms * (warps_per_sm * 32 / threads);
    dmma_kernel<CHAINS><<<blocks, threads>>>(out, 16);
    cudaEventRecord(e0);
    dmma_kernel<CHAINS><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * CHAINS * iters * (double)(threads / 32) * blocks;
    return (float)(flops / ms / 1e9);
}

int main() {
    int sms = 0, clk = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 2048);
    const int iters = 8192;
    const int ws[] = {4, 8, 12, 16, 24, 32, 64};
    printf("DMMA m8n8k4 TFLOP/s: rows = warps per SM, cols = independent chains per warp 1 2 4 8\n");
    for (int w : ws) {
        printf("%3d:", w);
        printf(" %6.2f", run<1>(out, w, sms, iters));
        printf(" %6.2f", run<2>(out, w, sms, iters));
        printf(" %6.2f", run<4>(out, w, sms, iters));
        printf(" %6.2f", run<8>(out, w, sms, iters));
        printf("\n");
    }
    {  // latency: one warp, one dependent chain
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        dmma_kernel<1><<<1, 32>>>(out, 16);
        cudaEventRecord(e0);
        dmma_kernel<1><<<1, 32>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        printf("dependent DMMA chain: %.1f ns per DMMA (%.0f cycles at %.0f MHz max clock)\n", ms * 1e6 / iters,
               ms * 1e-3 / iters * clk * 1e3, clk / 1e3);
    }
    {  // DMMA and DFMA warps side by side
        cudaEvent_t e0, e1;
        cudaEventCreate(&e0);
        cudaEventCreate(&e1);
        mixed_kernel<<<sms * 2, 512>>>(out, 16);
        cudaEventRecord(e0);
        mixed_kernel<<<sms * 2, 512>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double dmma = 2.0 * 256 * 4 * iters * 8.0 * sms * 2, dfma = 2.0 * 8 * iters * 4 * 256.0 * sms * 2;
        printf("mixed: DMMA %.2f + DFMA %.2f = %.2f TFLOP/s\n", dmma / ms / 1e9, dfma / ms / 1e9,
               (dmma + dfma) / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
