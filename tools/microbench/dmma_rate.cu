// fp64 tensor-core (mma.sync m8n8k4 f64) throughput on the B200 against the
// SIMT DFMA rate (dfma_rate.cu): register operands, 4 independent accumulator
// fragments per warp, all SMs. Decides whether the bounded pricing's screen
// (any-order fp64 GEMM, error-bounded) belongs on DMMA.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a dmma_rate.cu -o dmma_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}

template <int NACC>
__global__ void __launch_bounds__(256) k(double* out, int iters, double a0, double b0) {
    double c[NACC][2];
#pragma unroll
    for (int q = 0; q < NACC; ++q) c[q][0] = c[q][1] = 0.0;
    double a = a0 + threadIdx.x * 1e-9, b = b0 - threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int q = 0; q < NACC; ++q) dmma(c[q], a, b);
    double s = 0;
#pragma unroll
    for (int q = 0; q < NACC; ++q) s += c[q][0] + c[q][1];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
void run(double* out, int ctas_per_sm) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, blocks = 148 * ctas_per_sm;
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k<NACC><<<blocks, 256>>>(out, iters, 1.0, 0.999999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    // one m8n8k4 = 256 multiply-adds = 512 flops per warp
    const double flops = 512.0 * (blocks * 256 / 32) * (double)iters * NACC;
    printf("DMMA m8n8k4, %d accumulators/warp, %d CTAs/SM: %.2f TFLOP/s (%s)\n", NACC, ctas_per_sm,
           flops / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
    run<1>(out, 8);
    run<4>(out, 2);
    run<4>(out, 4);
    run<8>(out, 4);
    run<8>(out, 8);
    return 0;
}
