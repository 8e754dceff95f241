// Cycles per row of k_price's consumer inner loop (two sequential DMUL+DADD
// chains per thread over an smem tile, 8-row load groups software-pipelined),
// without TMA or mbarriers: is the ~33 cycles/row seen in k_price's compute-only
// experiment the chain code itself or the stage handshakes around it?
// nvcc -O3 --fmad=false -gencode arch=compute_100a,code=sm_100a chain_rate.cu -o chain_rate
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ void lds_group(const double2* col, int pitch, const double* ws, double2 (&a)[8],
                                          double2 (&w)[4]) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a[u].x), "=d"(a[u].y) : "r"(su32(col + u * pitch)));
#pragma unroll
    for (int u = 0; u < 4; ++u)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w[u].x), "=d"(w[u].y) : "r"(su32(ws + 2 * u)));
}
__device__ __forceinline__ void pin(double& a, double& b) { asm volatile("" : "+d"(a), "+d"(b)); }
__device__ __forceinline__ void chain_group(double& acc0, double& acc1, const double2 (&a)[8], const double2 (&w)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        acc0 = xadd(acc0, xmul(w[u].x, a[2 * u].x));
        acc1 = xadd(acc1, xmul(w[u].x, a[2 * u].y));
        acc0 = xadd(acc0, xmul(w[u].y, a[2 * u + 1].x));
        acc1 = xadd(acc1, xmul(w[u].y, a[2 * u + 1].y));
    }
}

template <int R>
__global__ void k_chain(int stages, int wbx, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* ws = sm + R * wbx;
    for (int e = threadIdx.x; e < R * wbx + R; e += blockDim.x) sm[e] = 1.0 + 1e-9 * e;
    __syncthreads();
    const int t = threadIdx.x;
    const int s2 = 2 * t;
    const double2* col = reinterpret_cast<const double2*>(sm + s2);
    const int pitch = wbx / 2;
    double acc0 = 0.0, acc1 = 0.0;
    const long long c0 = clock64();
    for (int k = 0; k < stages; ++k) {
        if (s2 < wbx) {
            const int ng = R >> 3;
            double2 a0[8], w0[4], a1[8], w1[4];
            lds_group(col, pitch, ws, a0, w0);
            int gi = 0;
            for (; gi + 2 <= ng; gi += 2) {
                lds_group(col + (gi + 1) * 8 * pitch, pitch, ws + (gi + 1) * 8, a1, w1);
                pin(acc0, acc1);
                chain_group(acc0, acc1, a0, w0);
                if (gi + 2 < ng) lds_group(col + (gi + 2) * 8 * pitch, pitch, ws + (gi + 2) * 8, a0, w0);
                pin(acc0, acc1);
                chain_group(acc0, acc1, a1, w1);
            }
            if (gi < ng) chain_group(acc0, acc1, a0, w0);
        }
        __syncwarp();
    }
    const long long c1 = clock64();
    if (t == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc0 + acc1 == 12345.0) out[0] = acc0;
}


template <int NC>
__global__ void k_simple(int rows, double* out, long long* cyc) {
    __shared__ double a[1024];
    for (int e = threadIdx.x; e < 1024; e += blockDim.x) a[e] = 1.0 + 1e-9 * e;
    __syncthreads();
    double acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = 0.0;
    const long long c0 = clock64();
    for (int i = 0; i < rows; i += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = a[(i + u) & 1023];
#pragma unroll
        for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int c = 0; c < NC; ++c) acc[c] = xadd(acc[c], xmul(v[u], v[(u + c + 1) & 7]));
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    double s = 0;
#pragma unroll
    for (int c = 0; c < NC; ++c) s += acc[c];
    if (s == 12345.0) out[0] = s;
}

__device__ __forceinline__ void lds_group1(const double* col, int pitch, const double* ws, double (&a)[8],
                                           double2 (&w)[4]) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(a[u]) : "r"(su32(col + u * pitch)));
#pragma unroll
    for (int u = 0; u < 4; ++u)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w[u].x), "=d"(w[u].y) : "r"(su32(ws + 2 * u)));
}
__device__ __forceinline__ void mul_group1(double (&p)[8], const double (&a)[8], const double2 (&w)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        p[2 * u] = xmul(w[u].x, a[2 * u]);
        p[2 * u + 1] = xmul(w[u].y, a[2 * u + 1]);
    }
}
__device__ __forceinline__ void add_group1(double& acc, const double (&p)[8]) {
#pragma unroll
    for (int u = 0; u < 8; ++u) acc = xadd(acc, p[u]);
}
__device__ __forceinline__ void pin1(double& a) { asm volatile("" : "+d"(a)); }
__device__ __forceinline__ void pin8(double (&p)[8]) {
    asm volatile("" : "+d"(p[0]), "+d"(p[1]), "+d"(p[2]), "+d"(p[3]), "+d"(p[4]), "+d"(p[5]), "+d"(p[6]),
                 "+d"(p[7]));
}

// k_price's narrow consumer loop (one chain per lane), volatile loads or plain loads
template <bool VOL>
__global__ void k_one(int stages, int R, int wbx, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* ws = sm + R * wbx;
    for (int e = threadIdx.x; e < R * wbx + R; e += blockDim.x) sm[e] = 1.0 + 1e-9 * e;
    __syncthreads();
    const int s = threadIdx.x & 31;
    const double* col = sm + (s % wbx);
    double acc = 0.0;
    const long long c0 = clock64();
    for (int k = 0; k < stages; ++k) {
        const int ng = R >> 3;
        double a0[8], a1[8], p0[8], p1[8];
        double2 w0[4], w1[4];
        if (VOL) {
            lds_group1(col, wbx, ws, a0, w0);
            mul_group1(p0, a0, w0);
            int gi = 0;
            for (; gi + 2 <= ng; gi += 2) {
                lds_group1(col + (gi + 1) * 8 * wbx, wbx, ws + (gi + 1) * 8, a1, w1);
                mul_group1(p1, a1, w1);
                pin8(p1);
                add_group1(acc, p0);
                pin1(acc);
                if (gi + 2 < ng) {
                    lds_group1(col + (gi + 2) * 8 * wbx, wbx, ws + (gi + 2) * 8, a0, w0);
                    mul_group1(p0, a0, w0);
                    pin8(p0);
                }
                add_group1(acc, p1);
                pin1(acc);
            }
        } else {
            for (int r = 0; r < R; r += 8) {
                double v[8], w[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) { v[u] = col[(r + u) * wbx]; w[u] = ws[r + u]; }
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = xadd(acc, xmul(w[u], v[u]));
            }
        }
        __syncwarp();
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc == 12345.0) out[0] = acc;
}

// plain-load variants: G rows per group, loads for group g+1 issued in source
// order before group g's chain (compiler free to schedule)
template <int G>
__global__ void k_plain(int stages, int R, int wbx, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* ws = sm + R * wbx;
    for (int e = threadIdx.x; e < R * wbx + R; e += blockDim.x) sm[e] = 1.0 + 1e-9 * e;
    __syncthreads();
    const int s = threadIdx.x & 31;
    const double* col = sm + (s % wbx);
    double acc = 0.0;
    const long long c0 = clock64();
    for (int k = 0; k < stages; ++k) {
        double v[G], w[G];
#pragma unroll
        for (int u = 0; u < G; ++u) { v[u] = col[u * wbx]; w[u] = ws[u]; }
        for (int r = 0; r < R; r += G) {
            double p[G];
#pragma unroll
            for (int u = 0; u < G; ++u) p[u] = xmul(w[u], v[u]);
            if (r + G < R) {
#pragma unroll
                for (int u = 0; u < G; ++u) { v[u] = col[(r + G + u) * wbx]; w[u] = ws[r + G + u]; }
            }
#pragma unroll
            for (int u = 0; u < G; ++u) acc = xadd(acc, p[u]);
        }
        __syncwarp();
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc == 12345.0) out[0] = acc;
}

// plain single-chain loop with G rows per group (loads then chain)
template <int G>
__global__ void k_plainG(int stages, int R, int wbx, double* out, long long* cyc) {
    extern __shared__ double sm[];
    double* ws = sm + R * wbx;
    for (int e = threadIdx.x; e < R * wbx + R; e += blockDim.x) sm[e] = 1.0 + 1e-9 * e;
    __syncthreads();
    const int s = threadIdx.x & 31;
    const double* col = sm + (s % wbx);
    double acc = 0.0;
    const long long c0 = clock64();
    for (int k = 0; k < stages; ++k) {
        for (int r = 0; r + G <= R; r += G) {
            double v[G], w[G];
#pragma unroll
            for (int u = 0; u < G; ++u) { v[u] = col[(r + u) * wbx]; w[u] = ws[r + u]; }
#pragma unroll
            for (int u = 0; u < G; ++u) acc = xadd(acc, xmul(w[u], v[u]));
        }
        __syncwarp();
    }
    const long long c1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = c1 - c0;
    if (acc == 12345.0) out[0] = acc;
}

int main() {
    double* out;
    long long* cyc;
    cudaMalloc(&out, 8);
    cudaMalloc(&cyc, 8 * 148);
    const int wbx = 112;
    for (int variant = 0; variant < 2; ++variant) {
        const int stages = variant == 0 ? 167 : 42;
        long long h[148];
        if (variant == 0) {
            const int R = 48;
            const int smem = (R * wbx + R) * 8;
            k_chain<48><<<148, 64, smem>>>(stages, wbx, out, cyc);
        } else {
            const int R = 192;
            const int smem = (R * wbx + R) * 8;
            cudaFuncSetAttribute(k_chain<192>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_chain<192><<<148, 64, smem>>>(stages, wbx, out, cyc);
        }
        cudaMemcpy(h, cyc, 8 * 148, cudaMemcpyDeviceToHost);
        const int R = variant == 0 ? 48 : 192;
        printf("R=%d stages=%d: %.1f cycles/row (block 0: %lld cycles)  err=%s\n", R, stages,
               (double)h[0] / (stages * R), h[0], cudaGetErrorString(cudaGetLastError()));
    }
    {
        long long h[148];
        const int rows = 8000;
        k_simple<1><<<148, 32>>>(rows, out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("simple 1 chain : %.1f cycles/row\n", (double)h[0] / rows);
        k_simple<2><<<148, 32>>>(rows, out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("simple 2 chains: %.1f cycles/row\n", (double)h[0] / rows);
        k_simple<4><<<148, 32>>>(rows, out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("simple 4 chains: %.1f cycles/row\n", (double)h[0] / rows);
        k_simple<8><<<148, 32>>>(rows, out, cyc); cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("simple 8 chains: %.1f cycles/row\n", (double)h[0] / rows);
    }
    {
        long long h[148];
        const int R = 256, wbx = 16, stages = 32;
        const int smem = (R * wbx + R) * 8;
        cudaFuncSetAttribute(k_one<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        cudaFuncSetAttribute(k_one<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int warps : {1, 4}) {
            k_one<true><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("narrow consumer (volatile, pipelined), %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
            k_one<false><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("narrow consumer (plain loads), %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
            cudaFuncSetAttribute(k_plain<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaFuncSetAttribute(k_plain<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_plain<8><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("plain prefetch G=8, %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
            k_plain<16><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("plain prefetch G=16, %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
            cudaFuncSetAttribute(k_plainG<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaFuncSetAttribute(k_plainG<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            cudaFuncSetAttribute(k_plainG<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            k_plainG<4><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("plainG G=4, %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
            k_plainG<16><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("plainG G=16, %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
            k_plainG<32><<<148, 32 * warps, smem>>>(stages, R, wbx, out, cyc);
            cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
            printf("plainG G=32, %d warps: %.1f cycles/row\n", warps, (double)h[0] / (stages * R));
        }
    }
    return 0;
}
