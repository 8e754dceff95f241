// Stream A: 1-CTA kernel spinning on a flag. Stream B: a 148-CTA kernel with
// ~190 KB dynamic smem per CTA, then a kernel that raises the flag.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
__global__ void spin(volatile unsigned long long* f, unsigned long long v) {
    if (threadIdx.x == 0) while (*f < v) {}
    __syncthreads();
}
__global__ void big(float* out) {
    extern __shared__ float sm[];
    sm[threadIdx.x] = threadIdx.x;
    __syncthreads();
    out[blockIdx.x * blockDim.x + threadIdx.x] = sm[(threadIdx.x + 1) % blockDim.x];
}
__global__ void raise(unsigned long long* f, unsigned long long v) { *f = v; }
int main(int argc, char** argv) {
    const int nb = argc > 1 ? atoi(argv[1]) : 148;
    unsigned long long* f;
    float* out;
    cudaMalloc(&f, 8); cudaMemset(f, 0, 8);
    cudaMalloc(&out, 148 * 256 * 4 * 4);
    int smem = 190 * 1024;
    cudaFuncSetAttribute(big, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (argc > 2) {
        cudaFuncSetAttribute(spin, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(raise, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        cudaFuncSetAttribute(big, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    }
    cudaStream_t a, b;
    cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking);
    cudaStreamCreateWithFlags(&b, cudaStreamNonBlocking);
    cudaDeviceSynchronize();
    for (int it = 1; it <= 50; ++it) {
        spin<<<1, 512, 0, a>>>(f, it);
        big<<<nb, 256, smem, b>>>(out);
        raise<<<1, 1, 0, b>>>(f, it);
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("done: %s\n", cudaGetErrorString(e));
    return 0;
}
