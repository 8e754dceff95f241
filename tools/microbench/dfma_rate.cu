// fp64 pipe throughput on the B200 for DFMA vs DMUL+DADD (independent chains,
// all SMs): does a DFMA issue at the DMUL/DADD rate (the reinversion DGEMM's
// peak) ?  nvcc -O3 -gencode arch=compute_100a,code=sm_100a dfma_rate.cu -o dfma_rate
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) k(double* out, int iters, double a, double b) {
    double acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = a + u + threadIdx.x;
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (OP == 0) acc[u] = __fma_rn(acc[u], b, a);
            if (OP == 1) acc[u] = __dmul_rn(acc[u], b);
            if (OP == 2) acc[u] = __dadd_rn(acc[u], b);
        }
    double s = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) s += acc[u];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000, blocks = 148 * 8;
    const char* names[] = {"DFMA", "DMUL", "DADD"};
    for (int op = 0; op < 3; ++op) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(e0);
            if (op == 0) k<0><<<blocks, 256>>>(out, iters, 1.0, 0.999999);
            if (op == 1) k<1><<<blocks, 256>>>(out, iters, 1.0, 0.999999);
            if (op == 2) k<2><<<blocks, 256>>>(out, iters, 1.0, 1e-9);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double inst = (double)blocks * 256 * iters * 8;
            if (rep) printf("%s: %.2f T instructions/s\n", names[op], inst / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
