// Microbenchmark: fp64 FMA (DFMA) vs fp64 tensor-core MMA (DMMA m8n8k4) throughput
// on the current GPU.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_rates fp64_rates.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters) {
    double acc[CHAINS];
    double x = 1.0 + threadIdx.x * 1e-9, y = 0.999999;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], y, x);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s += acc[c];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

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

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * 148 * 8 * 1024);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096, threads = 512, blocks = sms * 4;
    for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        dfma_kernel<8><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * iters * (double)threads * blocks;
        printf("DFMA: %.2f TFLOP/s\n", flops / ms / 1e9);
        cudaEventRecord(e0);
        dmma_kernel<4><<<blocks, threads>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        flops = 2.0 * 256 * 4 * iters * (double)(threads / 32) * blocks;
        printf("DMMA m8n8k4: %.2f TFLOP/s\n", flops / ms / 1e9);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
