// Read+write bandwidth of the update's access pattern (T column-major, C3:
// 8001 columns x 8000 rows, CTA b owns rows [56b, 56b+56)): in place (T -> T)
// versus out of place (T -> T2), with a trivial per-element op.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a inplace_bw.cu -o inplace_bw
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(448) k_upd(const double* __restrict__ src, double* __restrict__ dst, int ncol,
                                             int ld, int h, int mrows) {
    const int r0 = blockIdx.x * h;
    const int rows = min(h, mrows - r0);
    // thread -> (column phase, row): 448 threads = 8 columns x 56 rows
    const int r = threadIdx.x % h, cph = threadIdx.x / h, cst = blockDim.x / h;
    if (r >= rows) return;
    int j = cph;
    for (; j + 7 * cst < ncol; j += 8 * cst) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + (size_t)(j + u * cst) * ld + r0 + r);
#pragma unroll
        for (int u = 0; u < 8; ++u) __stcs(dst + (size_t)(j + u * cst) * ld + r0 + r, v[u] * 1.0000001);
    }
    for (; j < ncol; j += cst) dst[(size_t)j * ld + r0 + r] = src[(size_t)j * ld + r0 + r] * 1.0000001;
}

int main() {
    const int m = 8000, ncol = 8001, ld = 8000, h = 56;
    const int grid = (m + h - 1) / h;
    double *a, *b;
    cudaMalloc(&a, sizeof(double) * (size_t)ncol * ld);
    cudaMalloc(&b, sizeof(double) * (size_t)ncol * ld);
    cudaMemset(a, 0, sizeof(double) * (size_t)ncol * ld);
    cudaMemset(b, 0, sizeof(double) * (size_t)ncol * ld);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 16.0 * m * ncol;
    for (int mode = 0; mode < 2; ++mode) {
        float best = 1e9f, sum = 0.f;
        int n = 0;
        for (int r = 0; r < 30; ++r) {
            const double* src = (mode == 0 || r % 2 == 0) ? a : b;
            double* dst = mode == 0 ? a : (r % 2 == 0 ? b : a);
            cudaEventRecord(e0);
            k_upd<<<grid, 448>>>(src, dst, ncol, ld, h, m);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 2) { best = ms < best ? ms : best; sum += ms; ++n; }
        }
        printf("%-12s best %.1f us (%.0f GB/s)  mean %.1f us (%.0f GB/s)\n", mode == 0 ? "in-place" : "ping-pong",
               best * 1e3, bytes / (best * 1e-3) / 1e9, sum / n * 1e3, bytes / (sum / n * 1e-3) / 1e9);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
