// Standalone copy of k_la_gemm_price's main loop (64-candidate x 128-slot CTA
// tiles, 8 x 4 chains per thread, 16-deep chunks through a 3-stage cp.async
// ring) over synthetic operands, to separate the steady-state fp64 rate from
// the wave tail: a grid of exactly 3 waves (888 tiles at 2 CTAs/SM) against
// C4's 1008 tiles (3.41 waves), and the single-CTA-per-SM rate of the tail.
// nvcc -O3 --fmad=false -gencode arch=compute_100a,code=sm_100a la_price_rate.cu -o la_price_rate
#include <cstdio>
#include <cuda.h>
#include <cuda_runtime.h>

#ifndef XLS
#define XLS 3
#endif
constexpr int kLK = 64, kLN = 128, kLC = 16, kLS = XLS, kLThreads = 256;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ double xmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double xadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool ok) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(su32(dst)), "l"(src), "r"(ok ? 8 : 0)
                 : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(su32(dst)), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

struct Smem {
    double W[kLS][kLC][kLK];
    double A[kLS][kLC][kLN];
};

// MODE 0: as k_la_gemm_price; 1: no global loads (ring, waits and barriers kept);
// 2: W chunk as 16-byte copies (same bytes, wrong layout: the copy-width cost);
// 3: W chunk skipped (A only); 4: A chunk skipped (W only)
template <int MODE>
__global__ void __launch_bounds__(kLThreads, 2)
k_price(const double* __restrict__ Wp, long long ldx, int K, const double* __restrict__ A_nb, long long ld_nb,
        int m, int n_scan, double* out) {
    extern __shared__ __align__(16) unsigned char smem[];
    Smem& sm = *reinterpret_cast<Smem*>(smem);
    const int s0 = blockIdx.x * kLN, k0 = blockIdx.y * kLK;
    const int t = threadIdx.x, tk = t >> 5, ts = t & 31;
    double acc[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    auto issue = [&](int stage, int i0) {
        if (MODE == 1) return;
        if (MODE == 2) {
#pragma unroll
            for (int q = 0; q < kLC * kLK / (2 * kLThreads); ++q) {
                const int e = t + kLThreads * q;
                const int kk = e % (kLK / 2), ii = e / (kLK / 2);
                const int k = k0 + 2 * kk, i = i0 + ii;
                const bool ok = k < K && i < m;
                cp_async16(&sm.W[stage][ii][2 * kk], ok ? Wp + (size_t)k * ldx + (i & ~1) : Wp, ok ? 16 : 0);
            }
        }
#pragma unroll
        for (int q = 0; q < kLC * kLK / kLThreads; ++q) {
            if (MODE == 2 || MODE == 3) break;
            const int e = t + kLThreads * q;
            const int kk = e % kLK, ii = e / kLK;
            const int k = k0 + kk, i = i0 + ii;
            const bool ok = k < K && i < m;
            cp_async8(&sm.W[stage][ii][kk], ok ? Wp + (size_t)k * ldx + i : Wp, ok);
        }
#pragma unroll
        for (int q = 0; q < kLC * kLN / (2 * kLThreads); ++q) {
            if (MODE == 4) break;
            const int e = t + kLThreads * q;
            const int sp = e % (kLN / 2), ii = e / (kLN / 2);
            const int sl = s0 + 2 * sp, i = i0 + ii;
            const int nb = (i < m) ? 8 * max(0, min(2, n_scan - sl)) : 0;
            cp_async16(&sm.A[stage][ii][2 * sp], nb ? A_nb + (size_t)i * ld_nb + sl : A_nb, nb);
        }
    };
    const int nch = (m + kLC - 1) / kLC;
#pragma unroll
    for (int st = 0; st < kLS - 1; ++st) {
        if (st < nch) issue(st, st * kLC);
        cp_async_commit();
    }
    for (int ch = 0; ch < nch; ++ch) {
        cp_async_wait<kLS - 2>();
        __syncthreads();
        if (ch + kLS - 1 < nch) issue((ch + kLS - 1) % kLS, (ch + kLS - 1) * kLC);
        cp_async_commit();
        const int stg = ch % kLS;
        const int lim = min(kLC, m - ch * kLC);
        auto step = [&](int ii) {
            double w[8], a[4];
#pragma unroll
            for (int u = 0; u < 8; u += 2) {
                const double2 v2 = *reinterpret_cast<const double2*>(&sm.W[stg][ii][tk * 8 + u]);
                w[u] = v2.x;
                w[u + 1] = v2.y;
            }
#pragma unroll
            for (int v = 0; v < 4; ++v) a[v] = sm.A[stg][ii][ts + 32 * v];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = xadd(acc[u][v], xmul(w[u], a[v]));
        };
        if (lim == kLC) {
#pragma unroll
            for (int ii = 0; ii < kLC; ++ii) step(ii);
        } else {
            for (int ii = 0; ii < lim; ++ii) step(ii);
        }
    }
    cp_async_wait<0>();
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) s = xadd(s, acc[u][v]);
    out[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * kLThreads + t] = s;
}

// ---- TMA-fed form: one thread issues two 2D tensor copies per chunk (W' as a
// [64 k][16 i] box, A_nb as [16 i][128 s]); full[] mbarriers carry the bytes.
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
struct SmemT {
    double W[kLS][kLK][kLC];  // [k][i]
    double A[kLS][kLC][kLN];  // [i][s]
    uint64_t full[kLS];
};
template <int PAIR, bool FMA = false, bool VOUT = false>
__global__ void __launch_bounds__(kLThreads, 2)
k_price_tma(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA, int K, int m, double* out) {
    extern __shared__ __align__(128) unsigned char smem[];
    SmemT& sm = *reinterpret_cast<SmemT*>(smem);
    const int s0 = blockIdx.x * kLN, k0 = blockIdx.y * kLK;
    const int t = threadIdx.x, tk = t >> 5, ts = t & 31;
    if (t == 0) {
        for (int s = 0; s < kLS; ++s) mbar_init(&sm.full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc[8][4];
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    constexpr uint32_t kBytes = (kLK * kLC + kLC * kLN) * 8;
    auto issue = [&](int stage, int i0) {
        mbar_expect_tx(&sm.full[stage], kBytes);
        tma_load_2d(&sm.W[stage][0][0], &tmW, i0, k0, &sm.full[stage]);
        tma_load_2d(&sm.A[stage][0][0], &tmA, s0, i0, &sm.full[stage]);
    };
    const int nch = (m + kLC - 1) / kLC;
    if (t == 0)
        for (int st = 0; st < kLS - 1 && st < nch; ++st) issue(st, st * kLC);
    for (int ch = 0; ch < nch; ++ch) {
        __syncthreads();  // every thread is done with chunk ch-1: its stage is free
        if (t == 0 && ch + kLS - 1 < nch) issue((ch + kLS - 1) % kLS, (ch + kLS - 1) * kLC);
        const int stg = ch % kLS;
        mbar_wait(&sm.full[stg], (ch / kLS) & 1);
        const int lim = min(kLC, m - ch * kLC);
        if (PAIR) {
            auto step2 = [&](int ii) {
                double w0[8], w1[8], a0[4], a1[4];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const double2 v2 = *reinterpret_cast<const double2*>(&sm.W[stg][tk * 8 + u][ii]);
                    w0[u] = v2.x;
                    w1[u] = v2.y;
                }
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    a0[v] = sm.A[stg][ii][ts + 32 * v];
                    a1[v] = sm.A[stg][ii + 1][ts + 32 * v];
                }
                if (VOUT) {
#pragma unroll
                    for (int v = 0; v < 4; ++v)
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[u][v] = __fma_rn(w0[u], a0[v], acc[u][v]);
#pragma unroll
                    for (int v = 0; v < 4; ++v)
#pragma unroll
                        for (int u = 0; u < 8; ++u) acc[u][v] = __fma_rn(w1[u], a1[v], acc[u][v]);
                } else {
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        acc[u][v] = FMA ? __fma_rn(w0[u], a0[v], acc[u][v]) : xadd(acc[u][v], xmul(w0[u], a0[v]));
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v)
                        acc[u][v] = FMA ? __fma_rn(w1[u], a1[v], acc[u][v]) : xadd(acc[u][v], xmul(w1[u], a1[v]));
                }
            };
            if (lim == kLC) {
#pragma unroll
                for (int ii = 0; ii < kLC; ii += 2) step2(ii);
                continue;
            }
        }
        auto step = [&](int ii) {
            double w[8], a[4];
#pragma unroll
            for (int u = 0; u < 8; ++u) w[u] = sm.W[stg][tk * 8 + u][ii];
#pragma unroll
            for (int v = 0; v < 4; ++v) a[v] = sm.A[stg][ii][ts + 32 * v];
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int v = 0; v < 4; ++v) acc[u][v] = xadd(acc[u][v], xmul(w[u], a[v]));
        };
        if (lim == kLC) {
#pragma unroll
            for (int ii = 0; ii < kLC; ++ii) step(ii);
        } else {
            for (int ii = 0; ii < lim; ++ii) step(ii);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) s = xadd(s, acc[u][v]);
    out[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * kLThreads + t] = s;
}

static bool encode_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
                      uint32_t box_inner, uint32_t box_outer, bool swz = false) {
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
              CU_TENSOR_MAP_INTERLEAVE_NONE, swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- DMMA form (mma.sync m8n8k4 f64): 8 warps = 2 candidate halves x 4 slot
// quarters, 32 x 32 outputs per warp (4 x 4 fragments); W' box 128B-swizzled.
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
constexpr int kAP = kLN;  // (PAD variant: B stage as 8 swizzled 16-slot boxes)
struct SmemD {
    double W[kLS][kLK][kLC];  // [k][i], 128B-swizzled rows
    double A[kLS][kLC][kAP];  // [i][s]
    uint64_t full[kLS];
};
template <bool PAD>
__global__ void __launch_bounds__(kLThreads, 2)
k_price_dmma(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA, int K, int m, double* out) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    SmemD& sm = *reinterpret_cast<SmemD*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const int s0 = blockIdx.x * kLN, k0 = blockIdx.y * kLK;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, g = lane >> 2, tq = lane & 3;
    const int wc = warp & 1, ws = warp >> 1;
    if (t == 0) {
        for (int s = 0; s < kLS; ++s) mbar_init(&sm.full[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    constexpr uint32_t kBytes = (kLK * kLC + kLC * kLN) * 8;
    auto issue = [&](int stage, int i0) {
        mbar_expect_tx(&sm.full[stage], kBytes);
        tma_load_2d(&sm.W[stage][0][0], &tmW, i0, k0, &sm.full[stage]);
        if (PAD)  // 8 boxes of 16 slots x 16 rows, 128B-swizzled, 2 KB each
            for (int b = 0; b < kLN / 16; ++b) tma_load_2d(&sm.A[stage][0][0] + b * 256, &tmA, s0 + 16 * b, i0, &sm.full[stage]);
        else
            tma_load_2d(&sm.A[stage][0][0], &tmA, s0, i0, &sm.full[stage]);
    };
    const int nch = (m + kLC - 1) / kLC;
    if (t == 0)
        for (int st = 0; st < kLS - 1 && st < nch; ++st) issue(st, st * kLC);
    for (int ch = 0; ch < nch; ++ch) {
        __syncthreads();
        if (t == 0 && ch + kLS - 1 < nch) issue((ch + kLS - 1) % kLS, (ch + kLS - 1) * kLC);
        const int stg = ch % kLS;
        mbar_wait(&sm.full[stg], (ch / kLS) & 1);
        const double* Ws = &sm.W[stg][0][0];
#pragma unroll
        for (int kk = 0; kk < kLC / 4; ++kk) {
            const int e = kk * 4 + tq;
            double af[4], bf[4];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {
                const int r = wc * 32 + cb * 8 + g;
                af[cb] = Ws[r * kLC + ((((e >> 1) ^ (r & 7)) << 1) | (e & 1))];
            }
#pragma unroll
            const double* As = &sm.A[stg][0][0];
            for (int sb = 0; sb < 4; ++sb) {
                if (PAD) {
                    const int c = (sb & 1) * 8 + g;
                    bf[sb] = As[(ws * 2 + (sb >> 1)) * 256 + e * 16 + ((((c >> 1) ^ (e & 7)) << 1) | (c & 1))];
                } else {
                    bf[sb] = As[e * kLN + ws * 32 + sb * 8 + g];
                }
            }
#pragma unroll
            for (int cb = 0; cb < 4; ++cb)
#pragma unroll
                for (int sb = 0; sb < 4; ++sb) dmma(acc[cb][sb], af[cb], bf[sb]);
        }
    }
    double sum = 0.0;
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) sum += acc[a][b][0] + acc[a][b][1];
    out[((size_t)blockIdx.y * gridDim.x + blockIdx.x) * kLThreads + t] = sum;
}

static bool encode_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
                      uint32_t box_inner, uint32_t box_outer, bool swz);
int main() {
    const int m = 4000, K = 1000;
    const int nmax = 8064;
    const long long ldx = m + 8, ld_nb = nmax;
    double *Wp, *A, *out;
    cudaMalloc(&Wp, sizeof(double) * ldx * K);
    cudaMalloc(&A, sizeof(double) * ld_nb * m);
    cudaMalloc(&out, sizeof(double) * 2048 * 16 * kLThreads);
    cudaMemset(Wp, 0, sizeof(double) * ldx * K);
    cudaMemset(A, 0, sizeof(double) * ld_nb * m);
    cudaFuncSetAttribute(k_price<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaFuncSetAttribute(k_price<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaFuncSetAttribute(k_price<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaFuncSetAttribute(k_price<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaFuncSetAttribute(k_price<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(Smem));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    struct Case { const char* name; int n_scan; int kgrid; };
    // 1008 tiles = C4 (3.41 waves at 296 slots); 888 = exactly 3 waves; 148 = 1 CTA per SM; 296 = one full wave
    const Case cases[] = {{"C4 shape 63x16 (1008 tiles)", 8000, 16},
                          {"3 waves 74x12 (888 tiles)", 74 * 128, 12},
                          {"1 wave 37x8 (296 tiles)", 37 * 128, 8},
                          {"1 CTA/SM 37x4 (148 tiles)", 37 * 128, 4}};
    const char* modes[] = {"as kernel", "no loads", "W 16B copies", "A only", "W only"};
    for (int mode = 0; mode < 5; ++mode)
    for (const Case& c : cases) {
        if (mode && c.kgrid != 12) continue;
        dim3 grid((c.n_scan + kLN - 1) / kLN, c.kgrid);
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            auto f = mode == 0 ? k_price<0> : mode == 1 ? k_price<1> : mode == 2 ? k_price<2> : mode == 3 ? k_price<3> : k_price<4>;
            f<<<grid, kLThreads, sizeof(Smem)>>>(Wp, ldx, K, A, ld_nb, m, c.n_scan, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double inst = 2.0 * m * (double)grid.x * kLN * grid.y * kLK;
        printf("%-13s %-30s %.3f ms  %.2f T fp64 instr/s = %.3f of 18.5  (per tile-wave %.3f ms)\n", modes[mode], c.name, best,
               inst / (best * 1e-3) / 1e12, inst / (best * 1e-3) / 18.5e12,
               best / ((grid.x * grid.y + 295) / 296));
    }
    CUtensorMap tmW, tmA;
    if (!encode_2d(&tmW, Wp, m, K, ldx * 8, kLC, kLK) || !encode_2d(&tmA, A, ld_nb, m, ld_nb * 8, kLN, kLC)) {
        printf("encode failed\n");
        return 1;
    }
    cudaFuncSetAttribute(k_price_tma<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemT));
    cudaFuncSetAttribute(k_price_tma<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemT));
    cudaFuncSetAttribute(k_price_tma<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemT));
    cudaFuncSetAttribute(k_price_tma<1, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemT));
    for (int pair = 0; pair < 4; ++pair)
    for (const Case& c : cases) {
        dim3 grid((c.n_scan + kLN - 1) / kLN, c.kgrid);
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (pair == 3) k_price_tma<1, true, true><<<grid, kLThreads, sizeof(SmemT)>>>(tmW, tmA, K, m, out);
            else if (pair == 2) k_price_tma<1, true><<<grid, kLThreads, sizeof(SmemT)>>>(tmW, tmA, K, m, out);
            else if (pair) k_price_tma<1><<<grid, kLThreads, sizeof(SmemT)>>>(tmW, tmA, K, m, out);
            else k_price_tma<0><<<grid, kLThreads, sizeof(SmemT)>>>(tmW, tmA, K, m, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double inst = 2.0 * m * (double)grid.x * kLN * grid.y * kLK;
        const double in2 = pair >= 2 ? inst / 2 : inst;  // DFMA: one instruction per multiply-add
        printf("%-13s %-30s %.3f ms  %.2f T fp64 instr/s = %.3f of 18.5\n",
               pair == 3 ? "TMA DFMA v-out" : pair == 2 ? "TMA DFMA" : pair ? "TMA pairs" : "TMA", c.name, best,
               in2 / (best * 1e-3) / 1e12, in2 / (best * 1e-3) / 18.5e12);
    }
    CUtensorMap tmWs, tmA1;
    if (!encode_2d(&tmWs, Wp, m, K, ldx * 8, kLC, kLK, true)) { printf("encode swz failed\n"); return 1; }
    if (!encode_2d(&tmA1, A, ld_nb, m, ld_nb * 8, 16, kLC, true)) { printf("encode swzB failed\n"); return 1; }
    cudaFuncSetAttribute(k_price_dmma<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemD) + 1024);
    cudaFuncSetAttribute(k_price_dmma<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SmemD) + 1024);
    for (int pad = 0; pad < 2; ++pad)
    for (const Case& c : cases) {
        dim3 grid((c.n_scan + kLN - 1) / kLN, c.kgrid);
        float best = 1e30f;
        for (int rep = 0; rep < 5; ++rep) {
            cudaEventRecord(e0);
            if (pad) k_price_dmma<true><<<grid, kLThreads, sizeof(SmemD) + 1024>>>(tmWs, tmA1, K, m, out);
            else k_price_dmma<false><<<grid, kLThreads, sizeof(SmemD) + 1024>>>(tmWs, tmA, K, m, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
        }
        const double fl = 2.0 * m * (double)grid.x * kLN * grid.y * kLK;
        printf("%-13s %-30s %.3f ms  %.2f TFLOP/s = %.3f of 37.1 (DMMA)\n", pad ? "DMMA swzB" : "DMMA", c.name, best,
               fl / (best * 1e-3) / 1e12, fl / (best * 1e-3) / 37.1e12);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
