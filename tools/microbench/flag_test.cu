// Two kernels on two streams exchange a flag through global memory (the P2P
// transport's signal/wait primitive), same device.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void st_flag(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_flag(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__global__ void k(unsigned long long* mine, unsigned long long* other, int rank, unsigned long long seq, long long* cyc) {
    long long t0 = clock64();
    __threadfence_system();
    if (threadIdx.x == 0) st_flag(other + rank, seq);
    if (threadIdx.x == 0) while (ld_flag(mine + (1 - rank)) < seq) {}
    __syncthreads();
    if (threadIdx.x == 0) cyc[rank] = clock64() - t0;
}
int main() {
    unsigned long long *f0, *f1;
    long long* cyc;
    cudaMalloc(&f0, 64); cudaMalloc(&f1, 64); cudaMalloc(&cyc, 16);
    cudaMemset(f0, 0, 64); cudaMemset(f1, 0, 64);
    cudaStream_t s0, s1;
    cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
    cudaDeviceSynchronize();
    for (int it = 1; it <= 1000; ++it) {
        k<<<1, 512, 0, s0>>>(f0, f1, 0, it, cyc);
        k<<<1, 512, 0, s1>>>(f1, f0, 1, it, cyc);
    }
    cudaError_t e = cudaDeviceSynchronize();
    long long c[2];
    cudaMemcpy(c, cyc, 16, cudaMemcpyDeviceToHost);
    printf("1000 rounds done: %s, last cycles %lld %lld\n", cudaGetErrorString(e), c[0], c[1]);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a, s0);
    for (int it = 1001; it <= 2000; ++it) {
        k<<<1, 512, 0, s0>>>(f0, f1, 0, it, cyc);
        k<<<1, 512, 0, s1>>>(f1, f0, 1, it, cyc);
    }
    cudaEventRecord(b, s0); cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("per round %.2f us\n", ms * 1e3 / 1000);
    return 0;
}
