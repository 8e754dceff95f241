// fp64 issue ceiling of the lookahead GEMMs' inner step on the B200: a U x V
// outer product of sequential DMUL -> DADD chains per thread (the k_la_gemm_*
// form, bit-pinned so no DFMA), fed either from registers only or from a
// shared-memory tile (broadcast LDS.128 for the U side, LDS.64 for the V side,
// as k_la_gemm_price does), at several CTAs per SM. Prints fp64 instructions/s
// against the DFMA-probe peak (18.5 T/s, dfma_rate.cu). Measured: the smem-fed
// 8 x 4 loop with no global loads runs at 0.95 of it, so the 0.72-0.79 the
// cp.async-fed lookahead kernels reached was their staging (la_price_rate.cu).
// The register-only rows are NOT a rate: ptxas hoists their loop-invariant
// DMULs out of the loop (they print ~1.9 of peak), kept only as that warning.
// nvcc -O3 --fmad=false -gencode arch=compute_100a,code=sm_100a outer_rate.cu -o outer_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double vmul(double a, double b) {
    double r;
    asm volatile("mul.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
    return r;
}
__device__ __forceinline__ double vadd(double a, double b) {
    double r;
    asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
    return r;
}

constexpr int kSteps = 16;  // chunk depth (rows of the shared tile)

template <int U, int V, bool SMEM, int MINB>
__global__ void __launch_bounds__(256, MINB) k_outer(double* out, int iters) {
    __shared__ __align__(16) double Ws[kSteps][64];
    __shared__ __align__(16) double As[kSteps][128];
    const int t = threadIdx.x, tk = t >> 5, ts = t & 31;
    for (int e = t; e < kSteps * 64; e += 256) Ws[e / 64][e % 64] = 1.0 + 1e-9 * e;
    for (int e = t; e < kSteps * 128; e += 256) As[e / 128][e % 128] = 1.0 - 1e-9 * e;
    __syncthreads();
    double acc[U][V];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < V; ++v) acc[u][v] = 0.0;
    double wr[U], ar[V];
#pragma unroll
    for (int u = 0; u < U; ++u) wr[u] = 1.0 + 1e-7 * (u + t);
#pragma unroll
    for (int v = 0; v < V; ++v) ar[v] = 1.0 - 1e-7 * (v + t);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int ii = 0; ii < kSteps; ++ii) {
            double w[U], a[V];
            if (SMEM) {
#pragma unroll
                for (int u = 0; u < U; u += 2) {
                    const double2 v2 = *reinterpret_cast<const double2*>(&Ws[ii][(tk * U + u) & 63]);
                    w[u] = v2.x;
                    w[u + 1] = v2.y;
                }
#pragma unroll
                for (int v = 0; v < V; ++v) a[v] = As[ii][(ts + 32 * v) & 127];
            } else {
#pragma unroll
                for (int u = 0; u < U; ++u) w[u] = wr[u];
#pragma unroll
                for (int v = 0; v < V; ++v) a[v] = ar[v];
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int v = 0; v < V; ++v) acc[u][v] = vadd(acc[u][v], vmul(w[u], a[v]));
        }
        if (SMEM) __syncthreads();  // the chunk barrier of the real kernels
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int v = 0; v < V; ++v) s += acc[u][v];
    out[blockIdx.x * blockDim.x + t] = s;
}

template <int U, int V, bool SMEM, int MINB>
void run(const char* name, double* out, int ctas_per_sm) {
    const int blocks = 148 * ctas_per_sm, iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0);
        k_outer<U, V, SMEM, MINB><<<blocks, 256>>>(out, iters);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    cudaFuncAttributes fa;
    cudaFuncGetAttributes(&fa, k_outer<U, V, SMEM, MINB>);
    int occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_outer<U, V, SMEM, MINB>, 256, 0);
    const double inst = 2.0 * U * V * kSteps * (double)iters * blocks * 256;
    printf("%-28s ctas/SM %d (occ %d, regs %d): %.2f T fp64 instr/s = %.3f of 18.5\n", name, ctas_per_sm, occ,
           fa.numRegs, inst / (best * 1e-3) / 1e12, inst / (best * 1e-3) / 18.5e12);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

int main() {
    double* out;
    cudaMalloc(&out, 148 * 8 * 256 * sizeof(double));
    run<8, 4, false, 2>("8x4 registers", out, 2);
    run<8, 4, true, 2>("8x4 smem (la_price)", out, 2);
    run<4, 4, false, 2>("4x4 registers", out, 2);
    run<4, 4, true, 2>("4x4 smem", out, 2);
    run<4, 4, false, 3>("4x4 registers", out, 3);
    run<4, 4, true, 3>("4x4 smem", out, 3);
    run<4, 4, false, 4>("4x4 registers", out, 4);
    run<4, 4, true, 4>("4x4 smem", out, 4);
    run<4, 2, false, 4>("4x2 registers", out, 4);
    run<2, 2, false, 8>("2x2 registers", out, 8);
    return 0;
}
