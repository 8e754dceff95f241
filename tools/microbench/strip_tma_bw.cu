// Read-only HBM rate of k_price's access pattern on the B200: 148 CTAs, each
// streaming its own column strip (w doubles wide) of a row-major [rows][148 w]
// matrix through 2D TMA boxes of w x R (R = 48 KB / (8 w), as price_rows) into
// a 4-stage mbarrier ring, with no compute. Does the strip width (the
// contiguous run per row: 8 w bytes) explain C3 pricing (w ~ 112: 6.4 TB/s)
// streaming slower than C5 (w ~ 324: 7.3 TB/s)?
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a strip_tma_bw.cu -o strip_tma_bw
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                     : "=r"(ok) : "r"(su32(b)), "r"(parity) : "memory");
    } while (!ok);
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(su32(dst)), "l"(map), "r"(x), "r"(y), "r"(su32(b)) : "memory");
}

constexpr int S = 4;
__global__ void k_stream(const __grid_constant__ CUtensorMap tm, int rows, int w, int R, int nbox, int wbx, double* out) {
    extern __shared__ __align__(1024) unsigned char smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * R * w * 8);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) mbar_init(&full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int s0 = blockIdx.x * w;
    const int nst = (rows + R - 1) / R;
    double acc = 0.0;
    if (threadIdx.x == 0) {
        auto issue = [&](int k) {
            const int st = k % S;
            mbar_expect_tx(&full[st], (uint32_t)(R * w * 8));
            for (int q = 0; q < nbox; ++q)
                tma_load_2d(smem + (size_t)st * R * w * 8 + (size_t)q * wbx * R * 8, &tm, s0 + q * wbx, k * R, &full[st]);
        };
        for (int k = 0; k < S - 1 && k < nst; ++k) issue(k);
        for (int k = 0; k < nst; ++k) {
            if (k + S - 1 < nst) issue(k + S - 1);  // stage (k-1) % S was consumed by this thread
            mbar_wait(&full[k % S], (k / S) & 1);
            acc += reinterpret_cast<const double*>(smem + (size_t)(k % S) * R * w * 8)[0];
        }
        out[blockIdx.x] = acc;
    }
}

static bool encode_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
                      uint32_t box_inner, uint32_t box_outer) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess || !p) return false;
    auto fn = reinterpret_cast<CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                            const cuuint64_t*, const cuuint32_t*, const cuuint32_t*,
                                            CUtensorMapInterleave, CUtensorMapSwizzle, CUtensorMapL2promotion,
                                            CUtensorMapFloatOOBfill)>(p);
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {pitch_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int main() {
    const size_t cap = (size_t)9 << 30;  // 9 GB buffer
    double* A;
    double* out;
    if (cudaMalloc(&A, cap) != cudaSuccess) return 1;
    cudaMalloc(&out, 4096);
    cudaMemset(A, 0, cap);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int widths[] = {56, 112, 168, 224, 256, 328, 512};
    for (int w : widths) {
        const int wbx = w <= 256 ? w : w / 2;  // box width <= 256
        const int nbox = w / wbx;
        int R = (48 * 1024) / (8 * w);
        R &= ~15;
        if (R < 16) R = 16;
        if (R > 256) R = 256;
        const size_t cols = (size_t)148 * w;
        const int rows = (int)std::min<size_t>(cap / 8 / cols, 24000);
        CUtensorMap tm;
        if (!encode_2d(&tm, A, cols, rows, cols * 8, wbx, R)) { printf("encode failed w=%d\n", w); continue; }
        const size_t smem = (size_t)S * R * w * 8 + 64;
        cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            k_stream<<<148, 32, smem>>>(tm, rows, w, R, nbox, wbx, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double bytes = (double)rows * cols * 8;
        printf("w %4d (run %5d B, box %3d x %3d, %d box/stage): rows %5d, %.2f GB in %.3f ms = %.2f TB/s (%s)\n", w, w * 8,
               wbx, R, nbox, rows, bytes / 1e9, best, bytes / (best * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
