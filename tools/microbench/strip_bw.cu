// Read bandwidth of the pricing access pattern (A_nb, C3 shape): 148 CTAs, each
// streaming its own slot range over all m rows.
//   mode 0 "strip":   row-major A_nb, CTA reads w doubles per row, row pitch ld
//   mode 1 "blocked": 16-row blocks, slot-major inside a block: per block the
//                     CTA's w slots are one contiguous w*16-double run
//   mode 2 "contig":  each CTA reads one contiguous region (upper bound)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a strip_bw.cu -o strip_bw
#include <cstdio>
#include <cuda_runtime.h>

// grid = 148 strips x P row parts; 8 independent loads in flight per thread
constexpr int P = 4;
__global__ void __launch_bounds__(512) k_read(const double2* __restrict__ a, int mode, int m, int ld, int w,
                                              double* out) {
    const int c = blockIdx.x / P, part = blockIdx.x % P;
    const int mp = m / P, i0 = part * mp;
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const int w2 = w / 2;
    if (mode == 0) {
        const int rows_per = blockDim.x / w2;
        const int s = threadIdx.x % w2, r0 = threadIdx.x / w2;
        if (r0 < rows_per) {
            const double2* base = a + ((size_t)c * w) / 2 + s;
            int i = i0 + r0;
            for (; i + 7 * rows_per < i0 + mp; i += 8 * rows_per) {
                double2 v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldcs(base + (size_t)(i + u * rows_per) * (ld / 2));
#pragma unroll
                for (int u = 0; u < 8; ++u) acc[u] += v[u].x + v[u].y;
            }
            for (; i < i0 + mp; i += rows_per) acc[0] += __ldcs(base + (size_t)i * (ld / 2)).x;
        }
    } else if (mode == 1) {
        const int run2 = w * 8;  // double2 per 16-row block run
        const int nb = mp / 16, b0 = i0 / 16;
        const long n = (long)nb * run2;
        for (long e = threadIdx.x; e + 7 * 512 < n; e += 8 * 512) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const long f = e + u * 512;
                const int b = (int)(f / run2), o = (int)(f - (long)b * run2);
                v[u] = __ldcs(a + ((size_t)(b0 + b) * 16 * ld + (size_t)c * w * 16) / 2 + o);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += v[u].x + v[u].y;
        }
    } else {
        const long n = (long)mp * w2;
        const double2* base = a + (size_t)c * m * w2 + (size_t)part * n;
        for (long e = threadIdx.x; e + 7 * 512 < n; e += 8 * 512) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(base + e + u * 512);
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] += v[u].x + v[u].y;
        }
    }
    double t = 0;
    for (int u = 0; u < 8; ++u) t += acc[u];
    if (t == 1234.5) out[0] = t;
}

int main() {
    const int m = 8000, ld = 16000, ctas = 148;
    const int w = 108;  // 148*108 = 15984 slots
    double* a;
    cudaMalloc(&a, sizeof(double) * (size_t)m * ld + 4096);
    cudaMemset(a, 0, sizeof(double) * (size_t)m * ld);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double bytes = 8.0 * m * w * ctas;
    const char* names[] = {"strip", "blocked16", "contig"};
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9f;
        for (int r = 0; r < 20; ++r) {
            cudaEventRecord(e0);
            k_read<<<ctas * P, 512>>>(reinterpret_cast<const double2*>(a), mode, m, ld, w, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (r > 1 && ms < best) best = ms;
        }
        printf("%-10s %.1f us  %.0f GB/s\n", names[mode], best * 1e3, bytes / (best * 1e-3) / 1e9);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
