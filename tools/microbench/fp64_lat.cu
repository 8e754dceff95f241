// FP64 dependent-chain latency and throughput on the B200 (sm_100a).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false fp64_lat.cu -o fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void chain(double* out, double a, double b, int n, long long* cyc) {
    double acc = a + threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) acc = __dadd_rn(acc, b);
            if (OP == 1) acc = __dmul_rn(acc, b);
            if (OP == 2) acc = __fma_rn(acc, 1.0, b);
            if (OP == 3) acc = __dadd_rn(acc, __dmul_rn(b, a));
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) *cyc = t1 - t0;
    out[threadIdx.x + blockIdx.x * blockDim.x] = acc;
}

// throughput: K independent chains per thread
template <int K>
__global__ void thr(double* out, double a, double b, int n) {
    double acc[K];
#pragma unroll
    for (int k = 0; k < K; ++k) acc[k] = a + k + threadIdx.x;
    for (int i = 0; i < n; ++i)
#pragma unroll
        for (int k = 0; k < K; ++k) acc[k] = __dadd_rn(acc[k], __dmul_rn(b, acc[k]));
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += acc[k];
    out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 1 << 24);
    cudaMalloc(&cyc, 8);
    const int n = 4096;
    const char* names[] = {"DADD", "DMUL", "DFMA(x,1,b)", "DADD(acc, DMUL)"};
    for (int op = 0; op < 4; ++op) {
        for (int threads : {32, 128}) {
            if (op == 0) chain<0><<<1, threads>>>(out, 1.0, 1e-9, n, cyc);
            if (op == 1) chain<1><<<1, threads>>>(out, 1.0, 1.0000001, n, cyc);
            if (op == 2) chain<2><<<1, threads>>>(out, 1.0, 1e-9, n, cyc);
            if (op == 3) chain<3><<<1, threads>>>(out, 1.0, 1e-9, n, cyc);
            long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("%-18s threads %4d: %.2f cycles per dependent op\n", names[op], threads, (double)c / (n * 16.0));
        }
    }
    // throughput over the whole GPU
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int bs : {128, 256, 512, 1024}) {
        const int nn = 2048;
        thr<8><<<sms * 2, bs>>>(out, 1.0, 1e-9, nn);
        cudaEventRecord(e0);
        thr<8><<<sms * 2, bs>>>(out, 1.0, 1e-9, nn);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        double pairs = (double)sms * 2 * bs * nn * 8;
        printf("throughput blocks %d x %d: %.2f T (DMUL+DADD pairs)/s = %.1f TFLOP/s-equivalent\n", sms * 2, bs,
               pairs / ms / 1e9, 2 * pairs / ms / 1e9);
    }
    return 0;
}
