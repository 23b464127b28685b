// Microbenchmark: the dense block kernel's consumer loop without global memory.
// Each warp repeatedly loads a stage's DMMA fragments (2 k-steps x (MT A + NT B))
// from shared memory and issues MT x NT x 2 DMMA m8n8k4, optionally waiting on an
// already-completed mbarrier per stage.  Reports TFLOP/s for warps/SM and MT/NT
// shapes: the in-SM ceiling of the fg_block_tma_kernel consumer structure.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 dense_consumer.cu -o dense_consumer
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}
__device__ __forceinline__ double lds(uint32_t a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}

template <int MT, int NT, bool BAR>
__global__ void __launch_bounds__(256, 2) consumer(double* out, int stages) {
    __shared__ __align__(16) double buf[8 * 260 + 8 * 40];
    __shared__ uint64_t bar;
    for (int i = threadIdx.x; i < 8 * 260 + 8 * 40; i += blockDim.x) buf[i] = 1.0 + i * 1e-6;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(1));
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int fr = lane >> 2, fk = lane & 3;
    const uint32_t rs = (uint32_t)__cvta_generic_to_shared(buf) + (uint32_t)((fk * 260 + (warp % 7) * 32 + fr) * 8);
    const uint32_t cs = (uint32_t)__cvta_generic_to_shared(buf + 8 * 260) + (uint32_t)((fk * 36 + fr) * 8);
    const uint32_t barp = (uint32_t)__cvta_generic_to_shared(&bar);
    double d[MT][NT][2] = {};
    for (int g = 0; g < stages; ++g) {
        if (BAR) {
            asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}"
                         ::"r"(barp), "r"(0) : "memory");
        }
        double af[2][MT], bf[2][NT];
#pragma unroll
        for (int ks = 0; ks < 2; ++ks) {
#pragma unroll
            for (int i = 0; i < MT; ++i) af[ks][i] = lds(cs + (uint32_t)((ks * 4 * 36 + 8 * i) * 8));
#pragma unroll
            for (int j = 0; j < NT; ++j) bf[ks][j] = lds(rs + (uint32_t)((ks * 4 * 260 + 8 * j) * 8));
        }
#pragma unroll
        for (int ks = 0; ks < 2; ++ks)
#pragma unroll
            for (int i = 0; i < MT; ++i)
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma(d[i][j][0], d[i][j][1], af[ks][i], bf[ks][j]);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) s += d[i][j][0] + d[i][j][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int MT, int NT, bool BAR>
void run(double* out, int sms, int threads, int ctas_per_sm, const char* name) {
    const int stages = 4000;
    const int blocks = sms * ctas_per_sm;
    consumer<MT, NT, BAR><<<blocks, threads>>>(out, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    consumer<MT, NT, BAR><<<blocks, threads>>>(out, stages);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 256 * MT * NT * 2 * (double)stages * (threads / 32) * blocks;
    printf("%-28s warps/SM %2d: %6.2f TFLOP/s  (%s)\n", name, threads / 32 * ctas_per_sm, flops / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, sizeof(double) * sms * 2048);
    run<4, 4, false>(out, sms, 224, 2, "MT4 NT4 (dense kernel)");
    run<4, 4, true>(out, sms, 224, 2, "MT4 NT4 + mbarrier wait");
    run<4, 4, false>(out, sms, 256, 2, "MT4 NT4 8 warps/CTA");
    run<4, 2, false>(out, sms, 224, 2, "MT4 NT2");
    run<4, 2, false>(out, sms, 224, 4, "MT4 NT2 4 CTAs");
    run<2, 4, false>(out, sms, 224, 2, "MT2 NT4");
    run<4, 4, false>(out, sms, 224, 1, "MT4 NT4 1 CTA");
    return 0;
}
