// kernels.cu — sm_100a kernels of the lpsg dense revised simplex.
//
// Arithmetic contract: every reduction is one
// sequential fp64 chain per output in the reference's order, built from
// explicitly rounded __dmul_rn / __dadd_rn (no FMA contraction: the library is
// also compiled with --fmad=false), IEEE division, and the reference's update
// formula including its `temp != 0` store skip. Parallelism comes only from
// independent outputs (columns for pricing, rows for FTRAN / update) and from
// order-independent exact reductions (max/min with index tie-breaks).
#include <cuda_runtime.h>

#include <algorithm>
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>

#include <type_traits>
#include <vector>

#include "device.cuh"

namespace lpsg {
namespace {

constexpr double kInf = __builtin_huge_val();

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

// Pricing order (solver.cpp:88-91): strict '>' while scanning ascending j is
// the lexicographic (max z, min j) for finite z.
__device__ __forceinline__ bool better(double z1, int j1, double z2, int j2) {
    return z1 > z2 || (z1 == z2 && j1 < j2);
}

__device__ __forceinline__ const double* phase_cost(const Dev& d, int phase) {
    return phase == 1 ? d.cost_p1 : d.cost_true;
}

// Block-wide (max z, min j) reduction; result valid in thread 0.
__device__ void block_argmax(double& z, int& j) {
    __shared__ double sz[32];
    __shared__ int sj[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        const double oz = __shfl_down_sync(0xffffffffu, z, o);
        const int oj = __shfl_down_sync(0xffffffffu, j, o);
        if (better(oz, oj, z, j)) { z = oz; j = oj; }
    }
    __syncthreads();
    if (lane == 0) { sz[wid] = z; sj[wid] = j; }
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        z = lane < nw ? sz[lane] : -kInf;
        j = lane < nw ? sj[lane] : INT_MAX;
        for (int o = 16; o > 0; o >>= 1) {
            const double oz = __shfl_down_sync(0xffffffffu, z, o);
            const int oj = __shfl_down_sync(0xffffffffu, j, o);
            if (better(oz, oj, z, j)) { z = oz; j = oj; }
        }
    }
}

__device__ __forceinline__ void warp_argmax(double& z, int& j) {
    for (int o = 16; o > 0; o >>= 1) {
        const double oz = __shfl_down_sync(0xffffffffu, z, o);
        const int oj = __shfl_down_sync(0xffffffffu, j, o);
        if (better(oz, oj, z, j)) { z = oz; j = oj; }
    }
}

// price's outcome (solver.cpp:124-127) and the loop-top budget check (281).
__device__ __forceinline__ void price_decide(const Dev& d, Ctl* c, bool budget_hit, double z, int j) {
    if (budget_hit) {
        c->status = ST_ITER_LIMIT;
    } else {
        c->q = j == INT_MAX ? -1 : j;
        c->d = j == INT_MAX ? 0.0 : z;
        if (j == INT_MAX || (z <= d.opt_tol && !LPSG_XP(d, 15))) c->status = ST_OPTIMAL;
    }
}

// std::min(theta, r) semantics: r replaces theta only when r < theta (NaN never does).
__device__ __forceinline__ double min_keep(double theta, double r) { return (r < theta) ? r : theta; }

__device__ double block_min(double v) {
    __shared__ double s[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) v = min_keep(v, __shfl_down_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) s[wid] = v;
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        v = lane < nw ? s[lane] : kInf;
        for (int o = 16; o > 0; o >>= 1) v = min_keep(v, __shfl_down_sync(0xffffffffu, v, o));
    }
    return v;
}

// Programmatic dependent launch (PDL): the pivot-chain kernels are launched
// with programmatic stream serialization, so kernel t+1's CTAs are dispatched
// while kernel t drains; griddepcontrol.wait then blocks until kernel t has
// completed and its writes are visible. Both are no-ops without PDL.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Returns true in exactly one thread of the last CTA to arrive (threadfence
// reduction pattern); all CTAs must call it.
__device__ bool last_block(unsigned int* ticket) {
    __shared__ bool is_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned int t = atomicAdd(ticket, 1u);
        is_last = (t == gridDim.x * gridDim.y - 1);
    }
    __syncthreads();
    return is_last;
}

// ---------------------------------------------------------------- init ---
// Shard rows li < mloc hold global rows i = row0 + li: B^-1 = I, b_bar = b.
__global__ void k_init_tableau(Dev d, const double* __restrict__ b) {
    const int li = blockIdx.x * blockDim.x + threadIdx.x;
    if (li < d.mloc) {
        const int i = d.row0 + li;
        d.T[(size_t)i * d.ldT + li] = 1.0;
        d.T[(size_t)d.m * d.ldT + li] = b[i];
    }
}

// A_cm[j*ld + i] = A_rm[i*n + j]  (tiled transpose through shared memory)
// Also flags a non-finite coefficient (*nonfinite = 1): the pricing argmax
// equals the reference's first-scanned-column rule only for finite reduced
// costs, so such inputs are rejected.
__global__ void k_transpose(const double* __restrict__ A_rm, double* __restrict__ A_cm, int m,
                            int n, long long ld, int* nonfinite) {
    __shared__ double tile[32][33];
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    bool bad = false;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = i0 + k, j = j0 + threadIdx.x;
        if (i < m && j < n) {
            const double v = A_rm[(size_t)i * n + j];
            bad |= !isfinite(v);
            tile[k][threadIdx.x] = v;
        }
    }
    if (bad) atomicOr(nonfinite, 1);
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = j0 + k, i = i0 + threadIdx.x;
        if (i < m && j < n) A_cm[(size_t)j * ld + i] = tile[threadIdx.x][k];
    }
}

// A_nb[i*ld_nb + s] = A_cm[slot2col[s]*ld_cm + i]: a gathered transpose through
// 32 x 32 shared tiles, coalesced along i on the read and along s on the write.
__global__ void k_build_nb_cm(Dev d, int n_scan) {
    __shared__ double tile[32][33];
    __shared__ int col[32];
    const int s0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    if (threadIdx.y == 0) col[threadIdx.x] = s0 + (int)threadIdx.x < n_scan ? d.slot2col[s0 + threadIdx.x] : -1;
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = i0 + threadIdx.x, j = col[k];
        tile[k][threadIdx.x] = (j >= 0 && i < d.m) ? d.A_cm[(size_t)j * d.ld_cm + i] : 0.0;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = i0 + k, s = s0 + threadIdx.x;
        if (i < d.m && s < n_scan) d.A_nb[(size_t)i * d.ld_nb + s] = tile[threadIdx.x][k];
    }
}

// ------------------------------------------------------ rebuild_top_row ---
// solver.cpp:318-329: W_j = sum_i c_B[i] * B^-1[i][j] (ascending i); obj likewise
// over b_bar (column m). One output per lane of warp 0; 32x32 tiles of T are
// staged through shared memory so the column walk stays coalesced. A shard
// sums its own rows, continuing the chain from the previous shard's partials
// (`init`), so the sharded result is the same sequential sum.
__global__ void k_rebuild_top(Dev d, const double* __restrict__ init, double* __restrict__ out) {
    __shared__ double tile[32][33];
    __shared__ double cb[32];
    const int j0 = blockIdx.x * 32;
    const int ncols = d.m + 1;
    const int mloc = d.mloc;
    const double* cost = phase_cost(d, d.ctl->phase);
    double acc = 0.0;
    if (init && threadIdx.y == 0 && j0 + (int)threadIdx.x < ncols) acc = init[j0 + threadIdx.x];
    for (int i0 = 0; i0 < mloc; i0 += 32) {
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            const int j = j0 + k, i = i0 + threadIdx.x;
            tile[k][threadIdx.x] = (j < ncols && i < mloc) ? d.T[(size_t)j * d.ldT + i] : 0.0;
        }
        if (threadIdx.y == 0) {
            const int i = i0 + threadIdx.x;
            cb[threadIdx.x] = i < mloc ? cost[d.basic[d.row0 + i]] : 0.0;
        }
        __syncthreads();
        if (threadIdx.y == 0) {
            const int lim = min(32, mloc - i0);
            for (int k = 0; k < lim; ++k) acc = dadd(acc, dmul(cb[k], tile[threadIdx.x][k]));
        }
    }
    if (threadIdx.y == 0) {
        const int j = j0 + threadIdx.x;
        if (j < ncols) out[j] = acc;
        if (j == 0 && out == d.top) d.top[d.m + 1] = 0.0;
    }
}

// ------------------------------------------------ async bulk-copy helpers ---
// cp.async.bulk (TMA engine, SASS UBLKCP) moves global -> shared without
// registers; mbarriers (SYNCS.*) carry the byte counts. One producer warp per
// CTA keeps a ring of S stages in flight; consumer warps run the sequential
// fp64 chains out of shared memory.
__device__ __forceinline__ uint32_t su32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(n));
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t ok = 0;
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; "
            "selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(su32(b)), "r"(parity)
            : "memory");
    } while (!ok);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* b) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(dst)),
        "l"(src), "r"(bytes), "r"(su32(b))
        : "memory");
}
__device__ __forceinline__ int even_up(int v) { return (v + 1) & ~1; }

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* b) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
        "{%2, %3}], [%4];" ::"r"(su32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(su32(b))
        : "memory");
}
// L2 prefetch of a tensor box (no shared memory, no completion to wait for)
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* map, int x, int y) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(x), "r"(y)
                 : "memory");
}
// Streaming variants with an L2 eviction-priority hint: A_nb and T are read
// (and T written) once per pivot and exceed L2, so their lines should not
// displace anything worth keeping.
__device__ __forceinline__ uint64_t l2_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y, uint64_t* b,
                                                 uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1, {%2, %3}], [%4], %5;" ::"r"(su32(dst)),
        "l"(map), "r"(x), "r"(y), "r"(su32(b)), "l"(pol)
        : "memory");
}
__device__ __forceinline__ void tma_store_2d_hint(const CUtensorMap* map, int x, int y, const void* src, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group.L2::cache_hint [%0, {%1, %2}], [%3], %4;" ::"l"(map),
        "r"(x), "r"(y), "r"(su32(src)), "l"(pol)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

// TMA tile store (shared -> global) in a bulk async-group.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, int x, int y, const void* src) {
    asm volatile(
        "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(map), "r"(x),
        "r"(y), "r"(su32(src))
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
    asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// 8 rows of a slot pair (col, row pitch in double2) and the matching 8 W values.
__device__ __forceinline__ void lds_group(const double2* col, int pitch, const double* ws, double2 (&a)[8],
                                          double2 (&w)[4]) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a[u].x), "=d"(a[u].y) : "r"(su32(col + u * pitch)));
#pragma unroll
    for (int u = 0; u < 4; ++u)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(w[u].x), "=d"(w[u].y) : "r"(su32(ws + 2 * u)));
}

// Scheduling fence: a volatile no-op that "writes" the accumulators, so the
// chains after it cannot be hoisted above the volatile loads before it.
__device__ __forceinline__ void pin(double& a, double& b) { asm volatile("" : "+d"(a), "+d"(b)); }

// two sequential chains (slot 2t, slot 2t+1) over 8 rows, in row order
__device__ __forceinline__ void chain_group(double& acc0, double& acc1, const double2 (&a)[8],
                                            const double2 (&w)[4]) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        acc0 = dadd(acc0, dmul(w[u].x, a[2 * u].x));
        acc1 = dadd(acc1, dmul(w[u].x, a[2 * u].y));
        acc0 = dadd(acc0, dmul(w[u].y, a[2 * u + 1].x));
        acc1 = dadd(acc1, dmul(w[u].y, a[2 * u + 1].y));
    }
}

// rows per load group of the one-chain pricing path (chain_rate.cu: 32 rows
// 12.6-13.7 cycles/row, 8 rows 13.9-14.7)
constexpr int kNG = 32;
// columns per load group of the FTRAN chain in k_update. A/B: 32 cut the forced
// h = 8 shape 330 -> 307 us and C2's update 32.5 -> 30.6 us but cost C3 (h = 56)
// 2 us; selecting it per h (a runtime branch or a templated kernel) lost the
// gain on both sides, so the headline's 8 stays.
constexpr int kFG = 8;

// ---------------------------------------------------------------- price ---
// solver.cpp:79-129 (+ the loop-top budget check, solver.cpp:281).
// One CTA per SM; CTA b owns the contiguous slot range [b*w, b*w + w) of the
// row-major nonbasic matrix A_nb (w = ceil(n_scan/G) rounded up to 8, split
// into nb TMA boxes of wbx <= 256 slots). A producer warp streams R-row tiles
// through an S-stage ring with 2D TMA (one cp.async.bulk.tensor per box) plus a
// 1D bulk copy of the matching W segment; a consumer lane accumulates
// z_s = sum_i W_i * a_i,s strictly in ascending i for one slot (ranges up to
// 352 slots, spread over >= min(4, w/8) warps) or for a slot pair (wider
// ranges). The grid-wide (max z, min j) reduction is finished by the last CTA.
__global__ void __launch_bounds__(384) k_price(Dev d) {
    extern __shared__ __align__(1024) unsigned char smem[];
    // Under PDL this CTA is resident while k_pivot still runs (~10 us in which
    // HBM idles): warm L2 with the first stages of its A_nb strip. A prefetch
    // is only a hint and L2 is coherent with k_pivot's slot rewrite, so the
    // (possibly not yet final) n_scan read here can at worst waste bandwidth.
    if (threadIdx.x == 0 && d.price_pf > 0) {
        const int ns0 = *reinterpret_cast<volatile const int*>(&d.ctl->n_scan);
        const PriceGeom g0 = price_geom(ns0, gridDim.x, blockIdx.x);
        if (g0.own > 0 && g0.s0 < ns0) {
            const CUtensorMap* map = d.tm_nb + (g0.wbx / 8 - 1);
            const int nst = min(d.price_pf, (d.m + g0.R - 1) / g0.R);
            for (int k = 0; k < nst; ++k)
                for (int q = 0; q < g0.nb; ++q) tma_prefetch_2d(map, g0.s0 + q * g0.wbx, k * g0.R);
        }
    }
    pdl_wait();
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING) return;
    const bool budget_hit = c->total_iter >= c->budget;
    const int n_scan = c->n_scan;
    const double* cost = phase_cost(d, c->phase);
    const int m = d.m;
    const int G = gridDim.x;
    const PriceGeom g = price_geom(n_scan, G, blockIdx.x);
    const int s0 = g.s0;
    const int ns = max(0, min(g.own, n_scan - s0));
    const int nwc = d.price_nwc;
    const int S = d.price_S;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double bz = -kInf;
    int bj = INT_MAX;
    if (!budget_hit && ns > 0) {
        const int R = g.R, w = g.w;
        const size_t stage_el = (size_t)R * w + R;  // tile + W segment (doubles)
        const size_t stage_stride = (stage_el * 8 + 1023) / 1024 * 1024;
        uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * d.price_stage_bytes);
        uint64_t* empty = full + S;
        if (threadIdx.x == 0) {
            for (int k = 0; k < S; ++k) {
                mbar_init(&full[k], 1);
                mbar_init(&empty[k], nwc);
            }
            mbar_fence_init();
        }
        __syncthreads();
        const int nst = (m + R - 1) / R;
        const CUtensorMap* map = d.tm_nb + (g.wbx / 8 - 1);
        if (warp == nwc) {
            if (lane == 0) {
                const uint64_t pol = l2_evict_first();
                int st = 0;
                uint32_t ph = 0;
                for (int k = 0; k < nst; ++k) {
                    if (k >= S) mbar_wait(&empty[st], ph ^ 1);
                    const int i0 = k * R;
                    unsigned char* sb = smem + (size_t)st * stage_stride;
                    double* ws = reinterpret_cast<double*>(sb) + (size_t)R * w;
                    if (LPSG_XP(d, 2)) {  // experiment: no loads (compute-only rate)
                        mbar_arrive(&full[st]);
                    } else {
                        mbar_expect_tx(&full[st], (uint32_t)(R * w * 8 + R * 8));
                        for (int q = 0; q < g.nb; ++q)
                            if (d.l2_hint)
                                tma_load_2d_hint(sb + (size_t)q * g.wbx * R * 8, map, s0 + q * g.wbx, i0, &full[st], pol);
                            else
                                tma_load_2d(sb + (size_t)q * g.wbx * R * 8, map, s0 + q * g.wbx, i0, &full[st]);
                        bulk_g2s(ws, d.top + i0, (uint32_t)R * 8u, &full[st]);
                    }
                    if (++st == S) { st = 0; ph ^= 1; }
                }
            }
        } else if (warp < nwc && d.price_spt == 1) {
            // one slot per consumer lane, the CTA's slots split evenly over the
            // nwc consumer warps: a warp then issues 2 fp64 instructions per row
            // instead of 4 (one warp issues an fp64 instruction per ~3 cycles:
            // one chain per lane runs at 8-11 cycles a row, two at 16-19). That
            // matters where the chains, not the stream, bound the kernel: few
            // slots per CTA (sharded pricing, small n).
            const int spw = (ns + nwc - 1) / nwc;
            const int s = warp * spw + lane;
            const bool act = lane < spw && s < ns;
            const int wbx = g.wbx;
            const int q = s / wbx, tq = s - q * wbx;
            double acc = 0.0;
            int st = 0;
            uint32_t ph = 0;
            for (int k = 0; k < nst; ++k) {
                mbar_wait(&full[st], ph);
                const int nr = min(R, m - k * R);
                const double* sb = reinterpret_cast<const double*>(smem + (size_t)st * stage_stride);
                const double* ws = sb + (size_t)R * w;
                if (act && !LPSG_XP(d, 1)) {
                    // plain loads, scheduled by the compiler: 14-15 cycles a row,
                    // against 17-20 for volatile software-pipelined loads
                    // (tools/microbench/chain_rate.cu)
                    const double* col = sb + q * wbx * R + tq;
                    int rr = 0;
                    for (; rr + kNG <= nr; rr += kNG) {
                        double v[kNG], wv[kNG];
#pragma unroll
                        for (int u = 0; u < kNG; ++u) {
                            v[u] = col[(rr + u) * wbx];
                            wv[u] = ws[rr + u];
                        }
#pragma unroll
                        for (int u = 0; u < kNG; ++u) acc = dadd(acc, dmul(wv[u], v[u]));
                    }
                    for (; rr < nr; ++rr) acc = dadd(acc, dmul(ws[rr], col[rr * wbx]));
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == S) { st = 0; ph ^= 1; }
            }
            if (act) {
                const int j = d.slot2col[s0 + s];
                bz = dsub(acc, cost[j]);
                bj = j;
            }
        } else if (warp < nwc) {
            // consumer thread t owns the adjacent slot pair (2t, 2t+1): one
            // LDS.128 per row feeds two independent sequential chains
            const int t = threadIdx.x;
            const int s2 = 2 * t;
            // box q holds slots [q*wbx, (q+1)*wbx) as R rows of wbx doubles (wbx % 8 == 0,
            // so a pair never straddles two boxes)
            const int q = s2 / g.wbx, tq = s2 - q * g.wbx;
            const int wbx = g.wbx;
            double acc0 = 0.0, acc1 = 0.0;
            int st = 0;
            uint32_t ph = 0;
            for (int k = 0; k < nst; ++k) {
                mbar_wait(&full[st], ph);
                const int nr = min(R, m - k * R);
                const double* sb = reinterpret_cast<const double*>(smem + (size_t)st * stage_stride);
                const double* ws = sb + (size_t)R * w;
                if (s2 < ns && !LPSG_XP(d, 1)) {  // experiment bit 0: no math (memory-only rate)
                    const double2* col = reinterpret_cast<const double2*>(sb + q * wbx * R + tq);
                    const int pitch = wbx / 2;  // row pitch in double2
                    const int ng = nr >> 3;
                    // software pipeline: group g+1's shared loads are issued
                    // (volatile, in order) before group g's two chains run
                    double2 a0[8], w0[4], a1[8], w1[4];
                    if (ng > 0) lds_group(col, pitch, ws, a0, w0);
                    int gi = 0;
                    for (; gi + 2 <= ng; gi += 2) {
                        lds_group(col + (gi + 1) * 8 * pitch, pitch, ws + (gi + 1) * 8, a1, w1);
                        pin(acc0, acc1);  // keeps group g's chain behind group g+1's loads
                        chain_group(acc0, acc1, a0, w0);
                        if (gi + 2 < ng) lds_group(col + (gi + 2) * 8 * pitch, pitch, ws + (gi + 2) * 8, a0, w0);
                        pin(acc0, acc1);
                        chain_group(acc0, acc1, a1, w1);
                    }
                    if (gi < ng) chain_group(acc0, acc1, a0, w0);
                    for (int rr = ng * 8; rr < nr; ++rr) {
                        const double2 a2 = col[rr * pitch];
                        acc0 = dadd(acc0, dmul(ws[rr], a2.x));
                        acc1 = dadd(acc1, dmul(ws[rr], a2.y));
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[st]);
                if (++st == S) { st = 0; ph ^= 1; }
            }
            if (s2 < ns) {
                const int j0 = d.slot2col[s0 + s2];
                bz = dsub(acc0, cost[j0]);
                bj = j0;
                if (s2 + 1 < ns) {
                    const int j1 = d.slot2col[s0 + s2 + 1];
                    const double z1 = dsub(acc1, cost[j1]);
                    if (better(z1, j1, bz, bj)) { bz = z1; bj = j1; }
                }
            }
        }
    }
    // the next kernel's CTAs may launch now, during this kernel's tail only: early
    // resident-but-waiting CTAs would crowd this kernel's latency-bound warps
    pdl_trigger();
    block_argmax(bz, bj);
    if (threadIdx.x == 0) { d.pz[blockIdx.x] = bz; d.pj[blockIdx.x] = bj; }
    if (!last_block(&c->ticket_price)) return;
    if (threadIdx.x < 32) {
        double z = -kInf;
        int j = INT_MAX;
        for (int b = threadIdx.x; b < gridDim.x; b += 32) {
            const double oz = ((volatile double*)d.pz)[b];
            const int oj = ((volatile int*)d.pj)[b];
            if (better(oz, oj, z, j)) { z = oz; j = oj; }
        }
        warp_argmax(z, j);
        if (threadIdx.x == 0) {
            c->ticket_price = 0;
            if (!budget_hit) c->work[0] += 1;  // a real pricing pass (profile byte accounting)
            if (d.sharded) {
                d.pmsg[0] = PriceMsg{z, j, 0};  // merged across shards by k_price_final
                if (d.fused) {
                    // P2P: straight into every peer's mailbox slot [rank], then the flags
                    const PeerArgs& a = d.px_price;
                    for (int g = 0; g < a.size; ++g)
                        *reinterpret_cast<PriceMsg*>(a.peers[g] + a.mbox + (size_t)a.rank * sizeof(PriceMsg)) =
                            PriceMsg{z, j, 0};
                    __threadfence_system();
                    for (int g = 0; g < a.size; ++g)
                        st_flag(reinterpret_cast<unsigned long long*>(a.peers[g]) + a.rank, a.seq);
                }
            } else {
                price_decide(d, c, budget_hit, z, j);
            }
        }
    }
}

// world > 1: (max z, min j) over the gathered shard results, then the same
// decision as the single-GPU epilogue. Exact, so independent of shard order.
__global__ void k_price_final(Dev d) {
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING) return;
    if (d.fused) peer_wait(d.px_price);
    double z = -kInf;
    int j = INT_MAX;
    for (int g = threadIdx.x; g < d.world; g += 32) {
        PriceMsg mm;
        if (d.fused) {
            const PeerArgs& a = d.px_price;
            const double2 v = __ldcg(reinterpret_cast<const double2*>(a.peers[a.rank] + a.mbox + (size_t)g * sizeof(PriceMsg)));
            mm.z = v.x;
            mm.j = (int)__double_as_longlong(v.y);
        } else {
            mm = d.pmsg[1 + g];
        }
        if (better(mm.z, mm.j, z, j)) { z = mm.z; j = mm.j; }
    }
    warp_argmax(z, j);
    if (threadIdx.x == 0) price_decide(d, c, c->total_iter >= c->budget, z, j);
}

// Update warps of k_update: warp-per-column, lane-per-row-pair (double2), rows
// 2*lane + 64*u for u < NIT. Row r was already replaced by x in place
// (k_pivot), so its multiplier is 0 and the skip leaves it untouched, exactly
// like the zeroed multiplier of tiled_engine.cpp:241.
template <int NIT>
__device__ __forceinline__ void update_role(const Dev& d, unsigned char* smem, uint64_t* full,
                                            uint64_t* upd, size_t stage_stride, size_t tile_el,
                                            int nst, int S, int C, int h, int i0, int r, int U,
                                            bool up, int warp, int lane) {
    const int m = d.m, mloc = d.mloc;
    const bool naive = d.naive != 0;
    const double nz_r = naive ? -0.0 : 0.0;  // row r's multiplier: -(zeroed y_r) (tiled_engine.cpp:241)
    double ny0[NIT], ny1[NIT];
    bool ok[NIT];
#pragma unroll
    for (int u = 0; u < NIT; ++u) {
        const int t = 2 * lane + 64 * u;
        const int i = i0 + t;  // local row
        ok[u] = t < h;
        ny0[u] = (ok[u] && i < mloc && i != r) ? -d.Y[i] : (i == r ? nz_r : 0.0);
        ny1[u] = (ok[u] && i + 1 < mloc && i + 1 != r) ? -d.Y[i + 1] : (i + 1 == r ? nz_r : 0.0);
    }
    const size_t ldT = (size_t)d.ldT;
    const bool nomath = LPSG_XP(d, 4);  // experiment: stores without the update math
    const bool tstore = d.upd_tma_store != 0;  // the tile goes back by TMA store (producer warp)
    double2* const gbase = reinterpret_cast<double2*>(d.T + i0) + lane;  // + col * ldT/2
    const int ncols = m + 1;
    int st = 0;
    uint32_t ph = 0;
    for (int k = 0; k < nst; ++k) {
        mbar_wait(&full[st], ph);
        if (up) {
            const int j0 = k * C, nc = min(C, ncols - j0);
            double* tile = reinterpret_cast<double*>(smem + (size_t)st * stage_stride);
            const double* xs = tile + tile_el;
            double2* tcol = reinterpret_cast<double2*>(tile + warp * h) + lane;
            double2* gcol = gbase + (size_t)(j0 + warp) * (ldT / 2);
            const size_t gstep = (size_t)U * (ldT / 2);
            const int tstep = U * h / 2;
            for (int jj = warp; jj < nc; jj += U, tcol += tstep, gcol += gstep) {
                const double xj = xs[jj];
#pragma unroll
                for (int u = 0; u < NIT; ++u) {
                    if (ok[u]) {
                        double2 tv = tcol[32 * u];
                        if (nomath) {
                            if (!tstore) gcol[32 * u] = tv;
                            continue;
                        }
                        const double p0 = dmul(ny0[u], xj);
                        const double p1 = dmul(ny1[u], xj);
                        const double s0v = dadd(tv.x, p0);
                        const double s1v = dadd(tv.y, p1);
                        tv.x = (naive || p0 != 0.0) ? s0v : tv.x;
                        tv.y = (naive || p1 != 0.0) ? s1v : tv.y;
                        tcol[32 * u] = tv;
                        if (!tstore) gcol[32 * u] = tv;
                    }
                }
            }
            fence_proxy_async_smem();
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&upd[st]);
        if (++st == S) { st = 0; ph ^= 1; }
    }
}

// Short row blocks (h <= 32): a column has only h/2 row pairs, so one warp
// covers 32 / (h/2) columns per iteration (lane = column offset x row pair)
// instead of leaving most lanes idle on one column. Same per-element
// arithmetic as update_role.
__device__ __forceinline__ void update_role_small(const Dev& d, unsigned char* smem, uint64_t* full,
                                                  uint64_t* upd, size_t stage_stride, size_t tile_el,
                                                  int nst, int S, int C, int h, int i0, int r, int U,
                                                  bool up, int warp, int lane) {
    const int m = d.m, mloc = d.mloc;
    const int hp = h >> 1;                 // row pairs per column (h is even)
    const int cpw = 32 / hp;               // columns per warp iteration
    const int lc = lane / hp, lr = lane - lc * hp;
    const bool act = lc < cpw;
    const int i = i0 + 2 * lr;             // local row of this lane's pair
    const bool naive = d.naive != 0;
    const double nz_r = naive ? -0.0 : 0.0;
    const double ny0 = (act && i < mloc && i != r) ? -d.Y[i] : (i == r ? nz_r : 0.0);
    const double ny1 = (act && i + 1 < mloc && i + 1 != r) ? -d.Y[i + 1] : (i + 1 == r ? nz_r : 0.0);
    const size_t ldT = (size_t)d.ldT;
    const bool nomath = LPSG_XP(d, 4);
    const bool tstore = d.upd_tma_store != 0;
    double2* const gbase = reinterpret_cast<double2*>(d.T + i0) + lr;
    const int ncols = m + 1;
    const int step = U * cpw;
    int st = 0;
    uint32_t ph = 0;
    for (int k = 0; k < nst; ++k) {
        mbar_wait(&full[st], ph);
        if (up && act) {
            const int j0 = k * C, nc = min(C, ncols - j0);
            double* tile = reinterpret_cast<double*>(smem + (size_t)st * stage_stride);
            const double* xs = tile + tile_el;
            for (int jj = warp * cpw + lc; jj < nc; jj += step) {
                double2* tp = reinterpret_cast<double2*>(tile + (size_t)jj * h) + lr;
                double2 tv = *tp;
                if (!nomath) {
                    const double xj = xs[jj];
                    const double p0 = dmul(ny0, xj);
                    const double p1 = dmul(ny1, xj);
                    const double s0v = dadd(tv.x, p0);
                    const double s1v = dadd(tv.y, p1);
                    tv.x = (naive || p0 != 0.0) ? s0v : tv.x;
                    tv.y = (naive || p1 != 0.0) ? s1v : tv.y;
                    *tp = tv;
                }
                if (!tstore) gbase[(size_t)(j0 + jj) * (ldT / 2)] = tv;
            }
        }
        if (up) fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&upd[st]);
        if (++st == S) { st = 0; ph ^= 1; }
    }
}

// P2P, fused: the last CTA of k_update copies this shard's RatioMsg (just
// written to d.rmsg by its threads) into every peer's mailbox slot [rank] and
// raises the flags. All threads of the CTA call it.
__device__ __forceinline__ void ratio_put(const Dev& d) {
    __syncthreads();
    const PeerArgs& a = d.px_ratio;
    constexpr int kWords = sizeof(RatioMsg) / 8;
    const unsigned long long* src = reinterpret_cast<const unsigned long long*>(d.rmsg);
    for (int g = 0; g < a.size; ++g) {
        unsigned long long* dst =
            reinterpret_cast<unsigned long long*>(a.peers[g] + a.mbox + (size_t)a.rank * sizeof(RatioMsg));
        for (int w = threadIdx.x; w < kWords; w += blockDim.x) dst[w] = ((volatile const unsigned long long*)src)[w];
    }
    __syncthreads();
    peer_signal(a);
}

// pivot_update (solver.cpp:240-254) of row r = ctl.r, run by ONE CTA: the
// tail of k_update once its last CTA has decided r (single GPU, no tie,
// m + 1 <= kPivotPF * blockDim.x). Same arithmetic and bookkeeping as k_pivot,
// which it replaces on that path: one kernel boundary per pivot less.
constexpr int kPivotPF = 4;
__device__ __forceinline__ void pivot_cta(const Dev& d, Ctl* c) {
    const int m = d.m;
    const int r = ((volatile int*)&c->r)[0], q = c->q, n_scan = c->n_scan;
    const size_t ldT = (size_t)d.ldT;
    const double yr = __ldcg(d.Y + r);
    if (fabs(yr) <= d.pivot_tol) {
        if (threadIdx.x == 0) c->status = ST_PIVOT_ERR;
        return;
    }
    const double dk = ((volatile double*)d.top)[m + 1];
    const double ndk = -dk;
    const int p_leave = d.basic[r];
    const int s_q = q < d.n_total ? d.col2slot[q] : -1;
    const int last_col = n_scan > 0 ? d.slot2col[n_scan - 1] : -1;
    const bool p_local = p_leave < d.n_total && p_leave >= d.col0 && p_leave < d.col1;
    const bool q_local = s_q >= 0;
    int dst = -1, src_col = -1;
    if (p_local) {
        dst = q_local ? s_q : n_scan;
        src_col = p_leave;
    } else if (q_local && s_q != n_scan - 1) {
        dst = s_q;
        src_col = last_col;
    }
    const double xl = ddiv(yr, yr);
    const int li = c->log_len;
    LogEntry* const ent = d.log + li % d.log_cap;
    // every load first (kPivotPF per thread, all in flight together), then the
    // arithmetic and the stores: row r of T is m+1 strided elements, and a
    // load-divide-store loop would serialise one memory round trip per element
    double tv[kPivotPF], wv[kPivotPF], av[kPivotPF];
    const double* __restrict__ src = d.A_cm + (size_t)(dst >= 0 ? src_col : 0) * d.ld_cm;
#pragma unroll
    for (int u = 0; u < kPivotPF; ++u) {
        const int j = threadIdx.x + u * blockDim.x;
        tv[u] = j <= m ? __ldcg(d.T + (size_t)j * ldT + r) : 0.0;
        wv[u] = j <= m ? d.top[j] : 0.0;
        av[u] = (dst >= 0 && j < m) ? src[j] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kPivotPF; ++u) {
        const int j = threadIdx.x + u * blockDim.x;
        if (j <= m) {
            const double x = ddiv(tv[u], yr);
            d.xrow[j] = x;
            d.T[(size_t)j * ldT + r] = x;  // in place, like pr[j] /= y_rk (solver.cpp:246-247)
            const double p = dmul(ndk, x);
            const bool wr = d.naive || p != 0.0;
            const double nt = wr ? dadd(wv[u], p) : wv[u];
            if (wr) d.top[j] = nt;
            if (j == m) ent->objective = nt;
            if (dst >= 0 && j < m) d.A_nb[(size_t)j * d.ld_nb + dst] = av[u];
        }
    }
    __syncthreads();  // every read of the d slot and the slot maps precedes their rewrite
    if (threadIdx.x != 0) return;
    d.xrow[m + 1] = xl;
    c->work[2] += 1;
    {
        const double p = dmul(ndk, xl);
        if (d.naive || p != 0.0) d.top[m + 1] = dadd(dk, p);
    }
    int ns = n_scan;
    if (p_local) {
        if (!q_local) ++ns;
        d.slot2col[dst] = p_leave;
        d.col2slot[p_leave] = dst;
    } else if (q_local) {
        if (dst >= 0) {
            d.slot2col[dst] = src_col;
            d.col2slot[src_col] = dst;
        }
        --ns;
    }
    if (q < d.n_total) d.col2slot[q] = -1;
    c->n_scan = ns;
    d.basic[r] = q;
    c->total_iter += 1;
    ent->iteration = c->total_iter;
    ent->phase = c->phase;
    ent->row = r;
    ent->leaving = p_leave;
    ent->entering = q;
    c->log_len = li + 1;
    c->pending = 1;
    c->upd_r = r;
    c->upd_q = q;
}

// --------------------------------------------------------- update+FTRAN ---
// tiled_engine.cpp:230-266 with tile_kernel's cached mode (79-106) fused with the
// NEXT pivot's compute_direction (solver.cpp:131-136), SURVEY.md Appendix B.
// CTA b owns rows [b*h, b*h + h) of the column-major [B^-1 | b_bar]; a producer
// lane streams h-row x C-column boxes with 2D TMA (+ the x and a_q segments).
// Warp roles per stage:
//   U update warps (warp-per-column, lane-per-row): T_ij += (-y_i) * x_j unless
//     that product is 0, row r takes x_j; written back in place in shared
//     memory and to HBM with coalesced stores;
//   F FTRAN warps (thread-per-row): Y_i = sum_j T_new[i][j] * a_q[j] as one
//     sequential chain in ascending j, reading the updated tile.
__global__ void __launch_bounds__(512) k_update(Dev d) {
    extern __shared__ __align__(1024) unsigned char smem[];
    pdl_wait();
    Ctl* c = d.ctl;
    const int status = c->status;
    const bool up = c->pending != 0;
    const bool ft = status == ST_RUNNING && !c->no_ftran && c->q >= 0;
    if (!up && !ft) return;
    const int m = d.m, mloc = d.mloc, h = d.upd_h, C = d.upd_C, S = d.upd_S, U = d.upd_U;
    const int F = (h + 31) >> 5;
    // pivot row in shard-local numbering (-1: another shard owns it)
    const int r = (c->upd_r >= d.row0 && c->upd_r < d.row0 + mloc) ? c->upd_r - d.row0 : -1;
    const int i0 = blockIdx.x * h;
    const int ncols = m + 1;
    const int nst = (ncols + C - 1) / C;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const size_t tile_el = (size_t)C * h;
    const size_t stage_stride = ((tile_el + 2 * (size_t)C) * 8 + 1023) / 1024 * 1024;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)S * stage_stride);
    uint64_t* upd = full + S;
    uint64_t* empty = upd + S;
    if (threadIdx.x == 0) {
        for (int k = 0; k < S; ++k) {
            mbar_init(&full[k], 1);
            mbar_init(&upd[k], U);
            mbar_init(&empty[k], F + (up && d.upd_tma_store ? 1 : 0));
        }
        mbar_fence_init();
    }
    __syncthreads();
    const double* __restrict__ a = ft ? d.A_cm + (size_t)c->q * d.ld_cm : nullptr;
    double f_y = 0.0, f_bbar = 0.0;  // this thread's y_i, b_bar_i (FTRAN warps)
    bool f_ok = false;
    if (warp == U + F) {
        // ---- producer
        if (lane == 0) {
            const uint64_t pol = l2_evict_first();
            int st = 0;
            uint32_t ph = 0;
            for (int k = 0; k < nst; ++k) {
                if (k >= S) mbar_wait(&empty[st], ph ^ 1);
                const int j0 = k * C, nc = min(C, ncols - j0);
                const uint32_t seg = (uint32_t)even_up(nc) * 8u;
                unsigned char* sb = smem + (size_t)st * stage_stride;
                double* xs = reinterpret_cast<double*>(sb) + tile_el;
                double* as = xs + C;
                if (LPSG_XP(d, 8)) {  // experiment: no loads (compute-only rate)
                    mbar_arrive(&full[st]);
                } else {
                    mbar_expect_tx(&full[st], (uint32_t)(tile_el * 8) + (up ? seg : 0u) + (ft ? seg : 0u));
                    if (d.l2_hint) tma_load_2d_hint(sb, d.tm_T, i0, j0, &full[st], pol);
                    else tma_load_2d(sb, d.tm_T, i0, j0, &full[st]);
                    if (up) bulk_g2s(xs, d.xrow + j0, seg, &full[st]);
                    if (ft) bulk_g2s(as, a + j0, seg, &full[st]);
                }
                if (++st == S) { st = 0; ph ^= 1; }
            }
        } else if (lane == 1 && up && d.upd_tma_store) {
            // ---- storer: each updated tile goes back to HBM with one TMA store;
            // the stage is released once the store has read shared memory
            int st = 0;
            uint32_t ph = 0;
            // up to kStoreLag stores stay in flight; a stage is released once its
            // store has read shared memory (wait_group.read), kStoreLag behind
            constexpr int kStoreLag = 2;
            const uint64_t spol = l2_evict_first();
            int rel = 0;  // next stage index to release
            for (int k = 0; k < nst; ++k) {
                mbar_wait(&upd[st], ph);
                if (d.l2_hint) tma_store_2d_hint(d.tm_T, i0, k * C, smem + (size_t)st * stage_stride, spol);
                else tma_store_2d(d.tm_T, i0, k * C, smem + (size_t)st * stage_stride);
                if (++st == S) { st = 0; ph ^= 1; }
                if (k >= kStoreLag) {
                    bulk_wait_read<kStoreLag>();
                    mbar_arrive(&empty[rel]);
                    if (++rel == S) rel = 0;
                }
            }
            bulk_wait_read<0>();
            for (int k = nst > kStoreLag ? nst - kStoreLag : 0; k < nst; ++k) {
                mbar_arrive(&empty[rel]);
                if (++rel == S) rel = 0;
            }
            bulk_wait_all();
            // the fused pivot in the last CTA reads row r of T with generic
            // loads: order these async-proxy writes before them
            asm volatile("fence.proxy.async.global;" ::: "memory");
        }
    } else if (warp < U) {
        // ---- update warps: warp-per-column, lane-per-row-pair (double2), rows
        // 2*lane + 64*u. Row r was already replaced by x in place (k_pivot), so
        // its multiplier is 0 and the skip leaves it untouched, exactly like the
        // zeroed multiplier of tiled_engine.cpp:241.
        const int nit = (h + 63) >> 6;
        if (h <= 32 && !LPSG_XP(d, 32)) {  // experiment bit 5: the one-column-per-warp path (A/B)
            update_role_small(d, smem, full, upd, stage_stride, tile_el, nst, S, C, h, i0, r, U, up, warp, lane);
        } else switch (nit) {
            case 1: update_role<1>(d, smem, full, upd, stage_stride, tile_el, nst, S, C, h, i0, r, U, up, warp, lane); break;
            case 2: update_role<2>(d, smem, full, upd, stage_stride, tile_el, nst, S, C, h, i0, r, U, up, warp, lane); break;
            case 3: update_role<3>(d, smem, full, upd, stage_stride, tile_el, nst, S, C, h, i0, r, U, up, warp, lane); break;
            default: update_role<4>(d, smem, full, upd, stage_stride, tile_el, nst, S, C, h, i0, r, U, up, warp, lane); break;
        }
    } else if (warp < U + F) {
        // ---- FTRAN warps: thread-per-row sequential chains over the updated tile
        const int t = threadIdx.x - U * 32;
        const int i = i0 + t;  // local row
        const bool valid = t < h && i < mloc;
        double acc = 0.0;
        int st = 0;
        uint32_t ph = 0;
        for (int k = 0; k < nst; ++k) {
            mbar_wait(&upd[st], ph);
            if (ft && valid && !LPSG_XP(d, 4)) {  // experiment bit 2: no FTRAN math
                const int j0 = k * C, nf = min(C, m - j0);
                const double* tile = reinterpret_cast<const double*>(smem + (size_t)st * stage_stride);
                if (m - j0 < C) f_bbar = tile[(m - j0) * h + t];  // updated b_bar_i (column m)
                const double* as = tile + tile_el + C;
                const double* col = tile + t;
                // plain loads, scheduled by the compiler (volatile software
                // pipelining is slower for a single chain: chain_rate.cu)
                int jj = 0;
                for (; jj + kFG <= nf; jj += kFG) {
                    double tv[kFG], av[kFG];
#pragma unroll
                    for (int u = 0; u < kFG; ++u) tv[u] = col[(jj + u) * h];
#pragma unroll
                    for (int u = 0; u < kFG; u += 2) {
                        const double2 a2 = *reinterpret_cast<const double2*>(as + jj + u);
                        av[u] = a2.x;
                        av[u + 1] = a2.y;
                    }
#pragma unroll
                    for (int u = 0; u < kFG; ++u) acc = dadd(acc, dmul(tv[u], av[u]));
                }
                for (; jj < nf; ++jj) acc = dadd(acc, dmul(col[jj * h], as[jj]));
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == S) { st = 0; ph ^= 1; }
        }
        if (LPSG_XP(d, 12) && ft) acc = 1.0 + 1e-6 * i;  // experiments: keep pivoting on a valid column
        if (valid) {
            if (ft) {
                d.Y[i] = acc;
                f_y = acc;
                f_ok = true;
            } else {
                // Reference post-pivot column m+1: row r = 1, others y + (-y)*1 (skip 0).
                const double yi = d.Y[i];
                if (i == r) d.Y[i] = 1.0;
                else {
                    const double p = dmul(-yi, d.xrow[m + 1]);
                    if (d.naive || p != 0.0) d.Y[i] = dadd(yi, p);
                }
            }
        }
    }
    pdl_trigger();  // tail only (see k_price)
    // ---- fused ratio test, CTA-local part (solver.cpp:138-162): theta_b over this
    // CTA's eligible rows and the rows within window(theta_b), in row order.
    // The global theta <= theta_b and window() is monotone, so the union of the
    // local lists is a superset of the global candidates; the last CTA filters it.
    const bool do_ratio = ft && !c->no_ratio;
    if (do_ratio) {
        __shared__ int s_cnt[32];
        __shared__ double s_theta;
        __shared__ int s_any;
        const int i = d.row0 + i0 + (threadIdx.x - U * 32);  // global row
        bool elig = f_ok && !d.frozen[i] && !(f_y <= d.pivot_tol);
        const double ratio = elig ? ddiv(f_bbar, f_y) : kInf;
        // std::min(theta, NaN) keeps theta (solver.cpp:147): a NaN ratio must not
        // reach block_min, whose shuffle steps keep a NaN left operand
        const double th = block_min((elig && !isnan(ratio)) ? ratio : kInf);
        const int any = __syncthreads_or(elig);
        if (threadIdx.x == 0) { s_theta = th; s_any = any; }
        __syncthreads();
        const double wloc = dadd(s_theta, dmul(d.ratio_tie_tol, fmax(1.0, fabs(s_theta))));
        const bool cand = elig && ratio <= wloc;
        const unsigned bal = __ballot_sync(0xffffffffu, cand);
        if (lane == 0) s_cnt[warp] = __popc(bal);
        __syncthreads();
        if (cand) {
            int off = __popc(bal & ((1u << lane) - 1u));
            for (int w2 = U; w2 < warp; ++w2) off += s_cnt[w2];
            const size_t slot = (size_t)blockIdx.x * h + off;
            d.rc_row[slot] = i;
            d.rc_ratio[slot] = ratio;
        }
        if (threadIdx.x == 0) {
            int tot = 0;
            for (int w2 = U; w2 < U + F; ++w2) tot += s_cnt[w2];
            d.rc_cnt[blockIdx.x] = s_any ? tot : -1;
            d.rc_theta[blockIdx.x] = s_theta;
        }
    }
    if (!last_block(&c->ticket_update)) return;
    if (threadIdx.x == 0) {
        c->ticket_update = 0;
        if (up && !d.keep_pending) c->pending = 0;
        if (ft) d.top[m + 1] = c->d;
        if (up) c->work[1] += 1;  // credited as an update pass (an FTRAN-only pass is not)
    }
    if (!do_ratio) return;
    // ---- fused ratio test, global part: the last CTA, one thread per producing
    // CTA b (gridDim.x <= blockDim.x), then an ordered block scan.
    __shared__ int s_pre[32];
    __shared__ double s_th2;
    __shared__ int s_first;
    const int G = gridDim.x;
    const int b = threadIdx.x;
    const int cnt = b < G ? __ldcg(d.rc_cnt + b) : -1;
    const double thb = cnt >= 0 ? __ldcg(d.rc_theta + b) : kInf;
    const double th = block_min(thb);
    const int any = __syncthreads_or(cnt >= 0);
    if (threadIdx.x == 0) { s_th2 = th; s_first = -1; }
    __syncthreads();
    if (!any) {
        if (threadIdx.x == 0) {
            if (d.sharded) {
                d.rmsg->any = 0;
                d.rmsg->n = 0;
                d.rmsg->theta = kInf;
            } else {
                c->status = ST_UNBOUNDED;
            }
        }
        if (d.sharded && d.fused) ratio_put(d);
        return;
    }
    const double gth = s_th2;
    const double window = dadd(gth, dmul(d.ratio_tie_tol, fmax(1.0, fabs(gth))));
    // (no per-thread candidate arrays: dynamically indexed, they would live in
    // local memory; the few in-window entries are re-read from L2 below)
    int n = 0, first_row = -1;
    for (int e = 0; e < cnt; ++e) {
        const double ra = __ldcg(d.rc_ratio + (size_t)b * h + e);
        if (ra <= window) {
            if (n == 0) first_row = __ldcg(d.rc_row + (size_t)b * h + e);
            ++n;
        }
    }
    // exclusive scan of n over the block, in thread (= CTA = row) order
    int incl = n;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) s_pre[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        const int nw = (blockDim.x + 31) >> 5;
        int v = lane < nw ? s_pre[lane] : 0;
        int inc2 = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int u = __shfl_up_sync(0xffffffffu, inc2, o);
            if (lane >= o) inc2 += u;
        }
        if (lane < nw) s_pre[lane] = inc2 - v;  // exclusive warp offsets
        if (lane == 31) s_pre[31] = inc2;       // total (nw <= 16 < 31)
    }
    __syncthreads();
    int pos = s_pre[warp] + incl - n;
    if (n > 0) {
        if (pos == 0) s_first = first_row;
        for (int e = 0; e < cnt; ++e) {
            const double ra = __ldcg(d.rc_ratio + (size_t)b * h + e);
            if (ra <= window) {
                d.cand_ratio[pos] = ra;
                d.cand[pos++] = __ldcg(d.rc_row + (size_t)b * h + e);
            }
        }
    }
    __syncthreads();
    if (d.sharded) {
        // this shard's theta and its candidates within the shard-local window
        // (a superset of its rows inside the global window): k_ratio_final merges
        if (threadIdx.x < kRatioMsgCap) {
            const int e = threadIdx.x;
            const int total = s_pre[31];
            RatioMsg* mm = d.rmsg;
            mm->rows[e] = e < total ? ((volatile int*)d.cand)[e] : -1;
            const double rv = e < total ? (double)((volatile double*)d.cand_ratio)[e] : (double)kInf;
            mm->ratios[e] = rv;
            if (e == 0) {
                mm->theta = gth;
                mm->any = 1;
                mm->n = total;
            }
        }
        if (d.fused) ratio_put(d);
        return;
    }
    if (threadIdx.x == 0) {
        const int total = s_pre[31];
        c->ncand = total;
        c->theta = gth;
        if (total == 1 || d.anticycle == 1)
            c->r = s_first >= 0 ? s_first : ((volatile int*)d.cand)[0];
        else
            c->status = ST_TIE;
    }
    if (!d.fuse_pivot) return;
    __syncthreads();
    if (((volatile int*)&c->status)[0] == ST_RUNNING) pivot_cta(d, c);
}

// world > 1: global ratio test over the gathered shard messages
// (solver.cpp:138-162). theta = min over shards (exact); shards are contiguous
// row blocks in rank order, so concatenating their in-window candidates in rank
// order is the ascending candidate list. A shard with more local candidates
// than a message holds sends the host the full lists (ST_OVERFLOW).
__global__ void k_ratio_final(Dev d) {
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING || c->no_ratio || c->no_ftran || c->q < 0) return;
    if (d.fused) peer_wait(d.px_ratio);
    const int g = threadIdx.x;  // one lane per shard (world <= 32)
    const bool have = g < d.world;
    RatioMsg mm;
    if (have) {
        if (d.fused) {
            const PeerArgs& a = d.px_ratio;
            const unsigned long long* src =
                reinterpret_cast<const unsigned long long*>(a.peers[a.rank] + a.mbox + (size_t)g * sizeof(RatioMsg));
            unsigned long long* dst = reinterpret_cast<unsigned long long*>(&mm);
            for (int w = 0; w < (int)(sizeof(RatioMsg) / 8); ++w) dst[w] = __ldcg(src + w);
            d.rmsg[1 + g] = mm;  // the host's overflow path reads the gathered messages here
        } else {
            mm = d.rmsg[1 + g];
        }
    }
    const bool any_g = have && mm.any;
    double th = any_g ? mm.theta : kInf;
    for (int o = 16; o > 0; o >>= 1) th = min_keep(th, __shfl_xor_sync(0xffffffffu, th, o));
    const unsigned anyb = __ballot_sync(0xffffffffu, any_g);
    if (!anyb) {
        if (g == 0) c->status = ST_UNBOUNDED;
        return;
    }
    const double window = dadd(th, dmul(d.ratio_tie_tol, fmax(1.0, fabs(th))));
    const bool over = any_g && mm.n > kRatioMsgCap;
    int n = 0;
    if (any_g && !over)
        for (int e = 0; e < mm.n; ++e) n += mm.ratios[e] <= window;
    const unsigned overb = __ballot_sync(0xffffffffu, over);
    int incl = n;
    for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (g >= o) incl += v;
    }
    const int total = __shfl_sync(0xffffffffu, incl, 31);
    if (!overb && n > 0) {
        int pos = incl - n;
        for (int e = 0; e < mm.n; ++e)
            if (mm.ratios[e] <= window) d.cand[pos++] = mm.rows[e];
    }
    __syncwarp();
    if (g == 0) {
        c->theta = th;
        if (overb) {
            c->status = ST_OVERFLOW;
            return;
        }
        c->ncand = total;
        if (total == 1 || d.anticycle == 1)
            c->r = ((volatile int*)d.cand)[0];
        else
            c->status = ST_TIE;
    }
}

// Case 2 (out-of-core, tiled): the partitions of T were updated one after the
// other on one device, each leaving a RatioMsg (its theta, whether any row was
// eligible, and the count of its rows inside its own window) and its full
// in-window list at d.cand + row0[p]. Same merge as k_ratio_final (global theta
// = min, window, concatenation in partition = row order), but over any number
// of partitions and without the 30-entry message cap. One thread: the lists
// are read ascending and the merged list is written into d.cand from the
// front, never past an entry still to be read.
__global__ void k_ratio_merge_parts(Dev d, const RatioMsg* __restrict__ msgs, const int* __restrict__ row0, int P) {
    Ctl* c = d.ctl;
    if (threadIdx.x != 0 || c->status != ST_RUNNING || c->no_ratio || c->no_ftran || c->q < 0) return;
    double th = kInf;
    bool any = false;
    for (int p = 0; p < P; ++p)
        if (msgs[p].any) {
            any = true;
            th = min_keep(th, msgs[p].theta);
        }
    if (!any) {
        c->status = ST_UNBOUNDED;
        return;
    }
    const double window = dadd(th, dmul(d.ratio_tie_tol, fmax(1.0, fabs(th))));
    int total = 0;
    for (int p = 0; p < P; ++p) {
        if (!msgs[p].any) continue;
        for (int e = 0; e < msgs[p].n; ++e) {
            const int src = row0[p] + e;
            const double ra = d.cand_ratio[src];
            if (ra <= window) {
                const int row = d.cand[src];
                d.cand_ratio[total] = ra;
                d.cand[total++] = row;
            }
        }
    }
    c->theta = th;
    c->ncand = total;
    if (total == 1 || d.anticycle == 1) c->r = d.cand[0];
    else c->status = ST_TIE;
}

// ---------------------------------------------------------------- ratio ---
// solver.cpp:138-162. One CTA: theta = min over eligible rows of b_bar_i / y_i,
// window = theta + tol * max(1, |theta|), candidates ascending via an ordered
// block compaction. One candidate (or anticycle = none) resolves on device;
// two or more under tabu hand over to the host (ST_TIE).
__global__ void __launch_bounds__(1024) k_ratio(Dev d) {
    pdl_wait();
    pdl_trigger();
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING || c->pending) return;
    const int m = d.m;
    const double* __restrict__ bbar = d.T + (size_t)m * d.ldT;
    const double ptol = d.pivot_tol;
    double theta = kInf;
    int any = 0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        if (d.frozen[i]) continue;
        const double y = d.Y[i];
        if (y <= ptol) continue;
        any = 1;
        theta = min_keep(theta, ddiv(bbar[i], y));
    }
    any = __syncthreads_or(any);
    theta = block_min(theta);
    __shared__ double s_theta;
    __shared__ int s_warp[32];
    __shared__ int s_base;
    if (threadIdx.x == 0) { s_theta = theta; s_base = 0; }
    __syncthreads();
    if (!any) {
        if (threadIdx.x == 0) c->status = ST_UNBOUNDED;
        return;
    }
    theta = s_theta;
    const double window = dadd(theta, dmul(d.ratio_tie_tol, fmax(1.0, fabs(theta))));
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    for (int base = 0; base < m; base += blockDim.x) {
        const int i = base + threadIdx.x;
        bool f = false;
        if (i < m && !d.frozen[i]) {
            const double y = d.Y[i];
            if (!(y <= ptol)) f = ddiv(bbar[i], y) <= window;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, f);
        if (lane == 0) s_warp[wid] = __popc(bal);
        __syncthreads();
        if (threadIdx.x == 0) {
            int acc = 0;
            for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
                const int t = s_warp[w];
                s_warp[w] = acc;
                acc += t;
            }
        }
        __syncthreads();
        if (f) d.cand[s_base + s_warp[wid] + __popc(bal & ((1u << lane) - 1u))] = i;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) s_base += s_warp[wid] + __popc(bal);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int n = s_base;
        c->ncand = n;
        c->theta = theta;
        if (n == 1 || d.anticycle == 1) c->r = d.cand[0];
        else c->status = ST_TIE;
    }
}

// ---------------------------------------------------------------- pivot ---
// solver.cpp:240-254 minus the elimination (k_update): divide row r by y_rk
// (IEEE '/'), apply the row-0 part of the update (W, obj and the d slot; the
// multiplier is T[0][m+1], tiled_engine.cpp:240), swap the basis, maintain the
// nonbasic pricing slots, and log the pivot (note_iteration's observer data).
//
// world > 1: the owner of row r divides it in k_pivot_row and the shards sum
// their xbuf as int64 bit patterns (the others contribute 0), which delivers
// the owner's doubles bit for bit; k_pivot then runs on every shard from xbuf.
// P2P, fused (d.fused_x): the owner's threads also store their x_j straight
// into every peer's xbuf (same symmetric offset) and every shard's last CTA
// raises its flag for px_x (always, even when the device has stopped, so the
// wait that follows can never hang); k_peer_wait then completes the exchange.
__device__ __forceinline__ void pivot_row_signal(const Dev& d) {
    if (!d.fused_x) return;
    __threadfence_system();
    if (!last_block(&d.ctl->ticket_x)) return;
    if (threadIdx.x == 0) d.ctl->ticket_x = 0;
    peer_signal(d.px_x);
}

__device__ __forceinline__ void put_x(const Dev& d, int j, double v) {
    const PeerArgs& a = d.px_x;
    for (int g = 0; g < a.size; ++g)
        if (g != a.rank) reinterpret_cast<double*>(a.peers[g] + d.xbuf_off)[j] = v;
}

__global__ void __launch_bounds__(256) k_pivot_row(Dev d) {
    Ctl* c = d.ctl;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    if (c->status != ST_RUNNING) {
        if (gtid == 0) c->x_owner = 0;
        pivot_row_signal(d);
        return;
    }
    const int m = d.m;
    const int li = c->r - d.row0;
    const int gstride = gridDim.x * blockDim.x;
    long long* xb = reinterpret_cast<long long*>(d.xbuf);
    const bool own = li >= 0 && li < d.mloc;
    if (gtid == 0) c->x_owner = own ? 1 : 0;
    if (!own) {
        // summing transports need zeros from non-owners; a P2P owner writes our
        // xbuf remotely, so we must not touch it
        if (d.xbuf_zero)
            for (int j = gtid; j <= m + 2; j += gstride) xb[j] = 0;
        pivot_row_signal(d);
        return;
    }
    const double yr = d.Y[li];
    const bool ok = fabs(yr) > d.pivot_tol;
    for (int j = gtid; j <= m; j += gstride) {
        const double xj = ddiv(d.T[(size_t)j * d.ldT + li], yr);
        d.xbuf[j] = xj;
        if (d.fused_x) put_x(d, j, xj);
        if (ok) d.T[(size_t)j * d.ldT + li] = xj;  // in place (solver.cpp:246-247)
    }
    if (gtid == 0) {
        d.xbuf[m + 1] = ddiv(yr, yr);
        d.xbuf[m + 2] = yr;
        if (d.fused_x) {
            put_x(d, m + 1, d.xbuf[m + 1]);
            put_x(d, m + 2, yr);
        }
    }
    pivot_row_signal(d);
}

// Latency-bound (one element per thread): every load the kernel needs is issued
// up front in parallel, the CTA ticket is taken as soon as the loaded values are
// in registers (so the last CTA may overwrite the d slot and the slot maps that
// every CTA read), and the pivot-row / top-row / A_nb stores drain after it. The
// logged objective is recomputed from T[m][r] by the bookkeeping thread with the
// (the new T[0][m]) is written into the log entry by the thread that owns j = m,
// so no CTA ever reads another CTA's store.
__global__ void __launch_bounds__(256) k_pivot(Dev d) {
    pdl_wait();
    pdl_trigger();
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING) return;
    const int m = d.m;
    const int r = c->r, q = c->q, n_scan = c->n_scan;
    const bool sharded = d.sharded != 0;
    const int gtid = blockIdx.x * blockDim.x + threadIdx.x;
    const int gstride = gridDim.x * blockDim.x;
    const size_t ldT = (size_t)d.ldT;
    // independent loads, all in flight together
    const double yr = sharded ? d.xbuf[m + 2] : d.Y[r];
    const double dk = d.top[m + 1];
    const int p_leave = d.basic[r];
    const int s_q = q < d.n_total ? d.col2slot[q] : -1;  // artificials have no slot
    const int last_col = n_scan > 0 ? d.slot2col[n_scan - 1] : -1;
    const bool one = gtid <= m && gtid + gstride > m;  // this thread owns at most one j
    double tj = 0.0, topj = 0.0;
    if (one) {
        tj = sharded ? d.xbuf[gtid] : d.T[(size_t)gtid * ldT + r];
        topj = d.top[gtid];
    }
    if (fabs(yr) <= d.pivot_tol) {
        if (blockIdx.x == 0 && threadIdx.x == 0) c->status = ST_PIVOT_ERR;
        return;
    }
    const double ndk = -dk;
    // nonbasic slot maintenance for this shard's columns [col0, col1): the
    // leaving column takes the entering column's slot, or is appended when the
    // entering column lives on another shard; an entering column whose leaver
    // is not ours (artificial or another shard's) is removed by moving the
    // last slot into its place.
    const bool p_local = p_leave < d.n_total && p_leave >= d.col0 && p_leave < d.col1;
    const bool q_local = s_q >= 0;
    int dst = -1, src_col = -1;
    if (p_local) {
        dst = q_local ? s_q : n_scan;
        src_col = p_leave;
    } else if (q_local && s_q != n_scan - 1) {
        dst = s_q;
        src_col = last_col;
    }
    const double* __restrict__ src = d.A_cm + (size_t)(dst >= 0 ? src_col : 0) * d.ld_cm;
    const bool one_i = dst >= 0 && gtid < m && gtid + gstride >= m;
    const double ai = one_i ? src[gtid] : 0.0;
    // every value read above is in registers once it has been used: take the
    // ticket now; the stores below never feed another CTA's loads
    const double xl = ddiv(yr, yr);
    double xj = 0.0;
    if (one) xj = sharded ? tj : ddiv(tj, yr);
    const int li = c->log_len;  // monotonic; the log is a ring the host drains
    LogEntry* const ent = d.log + li % d.log_cap;
    const bool last = last_block(&c->ticket_misc);
    if (one) {
        if (!sharded) {
            d.xrow[gtid] = xj;
            d.T[(size_t)gtid * ldT + r] = xj;  // in place, like pr[j] /= y_rk (solver.cpp:246-247)
        }
        const double p = dmul(ndk, xj);
        const bool wr = d.naive || p != 0.0;
        const double nt = wr ? dadd(topj, p) : topj;
        if (wr) d.top[gtid] = nt;
        if (gtid == m) ent->objective = nt;
    } else {
        for (int j = gtid; j <= m; j += gstride) {
            const double x = sharded ? d.xbuf[j] : ddiv(d.T[(size_t)j * ldT + r], yr);
            if (!sharded) {
                d.xrow[j] = x;
                d.T[(size_t)j * ldT + r] = x;
            }
            const double p = dmul(ndk, x);
            const double t0 = d.top[j];
            const bool wr = d.naive || p != 0.0;
            const double nt = wr ? dadd(t0, p) : t0;
            if (wr) d.top[j] = nt;
            if (j == m) ent->objective = nt;
        }
    }
    if (dst >= 0) {
        if (one_i) d.A_nb[(size_t)gtid * d.ld_nb + dst] = ai;
        else
            for (int i = gtid; i < m; i += gstride) d.A_nb[(size_t)i * d.ld_nb + dst] = src[i];
    }
    if (gtid == 0 && !sharded) d.xrow[m + 1] = xl;
    if (!last || threadIdx.x != 0) return;
    c->ticket_misc = 0;
    c->work[2] += 1;
    {
        // the d slot (T[0][m+1]) is every CTA's multiplier source
        const double p = dmul(ndk, xl);
        if (d.naive || p != 0.0) d.top[m + 1] = dadd(dk, p);
    }
    int ns = n_scan;
    if (p_local) {
        if (!q_local) ++ns;
        d.slot2col[dst] = p_leave;
        d.col2slot[p_leave] = dst;
    } else if (q_local) {
        if (dst >= 0) {
            d.slot2col[dst] = src_col;
            d.col2slot[src_col] = dst;
        }
        --ns;
    }
    if (q < d.n_total) d.col2slot[q] = -1;
    c->n_scan = ns;
    d.basic[r] = q;
    c->total_iter += 1;
    ent->iteration = c->total_iter;
    ent->phase = c->phase;
    ent->row = r;
    ent->leaving = p_leave;
    ent->entering = q;
    c->log_len = li + 1;
    c->pending = 1;
    c->upd_r = r;
    c->upd_q = q;
}

// --------------------------------------------------------- drive-out scan ---
// solver.cpp:295-316: first j < n_total, nonbasic, with |dot(B^-1 row i, a_j)| >
// pivot_tol (ascending i in the dot), as a min-j reduction over this shard's
// slots into ctl.found (the host pre-sets INT_MAX; shards then take the min);
// k_drive_red computes the entering reduced cost dot(W, a_j) - c_j.
__global__ void k_gather_row(Dev d, int li, double* out) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= d.m; k += gridDim.x * blockDim.x)
        out[k] = d.T[(size_t)k * d.ldT + li];
}

__global__ void __launch_bounds__(256) k_drive_scan(Dev d, const double* __restrict__ g) {
    Ctl* c = d.ctl;
    const int n_scan = c->n_scan;
    const int m = d.m;
    int best = INT_MAX;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_scan; s += gridDim.x * blockDim.x) {
        const double* __restrict__ a = d.A_nb + s;
        double acc = 0.0;
        for (int i = 0; i < m; ++i) acc = dadd(acc, dmul(g[i], a[(size_t)i * d.ld_nb]));
        if (fabs(acc) > d.pivot_tol) best = min(best, d.slot2col[s]);
    }
    for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_down_sync(0xffffffffu, best, o));
    __shared__ int sb[32];
    if ((threadIdx.x & 31) == 0) sb[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = min(best, sb[w]);
        atomicMin(&c->found, best);
    }
}

__global__ void k_drive_red(Dev d) {
    Ctl* c = d.ctl;
    const int j = c->found;
    if (j == INT_MAX) {
        if (threadIdx.x == 0) c->found = -1;
        return;
    }
    if (threadIdx.x != 0) return;
    const double* cost = phase_cost(d, c->phase);
    const double* __restrict__ a = d.A_cm + (size_t)j * d.ld_cm;
    double acc = 0.0;
    for (int i = 0; i < d.m; ++i) acc = dadd(acc, dmul(d.top[i], a[i]));
    c->found_red = dsub(acc, cost[j]);
}

// ------------------------------------------------------------ lookahead ---
// solver.cpp:164-213, batched over K candidate rows without materialising the
// K pivoted tableaus: (1) X_k = T_r / piv, W'_k = W - d*X_k; (2) pricing of
// W'_k over the nonbasic set with q removed and basic[r_k] added; (3) y'_ik =
// sum_j (T_ij - y_i X_kj) a_best[j] (ascending j) and theta'_k; (4) score.
// Sharded: X_k comes from the owner of row r_k (int64 bit-pattern sum, like
// k_pivot_row); pricing and theta' run over the shard's columns / rows and are
// merged exactly (max/min) across shards.
__global__ void k_la_x(Dev d, LookaheadDev la) {
    const int k = blockIdx.y;
    const int li = la.rows[k] - d.row0;
    const bool own = li >= 0 && li < d.mloc;
    double* X = la.X + (size_t)k * la.ldx;
    const double piv = own ? d.Y[li] : 0.0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= d.m; j += gridDim.x * blockDim.x) {
        if (own) X[j] = ddiv(d.T[(size_t)j * d.ldT + li], piv);
        else if (!la.x_owned_only) reinterpret_cast<long long*>(X)[j] = 0;
    }
}

__global__ void k_la_wp(Dev d, LookaheadDev la) {
    const int k = blockIdx.y;
    const double dk = d.top[d.m + 1];
    const double* X = la.X + (size_t)k * la.ldx;
    bool bad = false;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d.m; j += gridDim.x * blockDim.x) {
        const double w = d.top[j];
        const double x = X[j];
        bad |= !isfinite(x);
        la.Wp[(size_t)k * la.ldx + j] = dk == 0.0 ? w : dsub(w, dmul(dk, x));
    }
    if (bad) atomicOr(la.nonfinite, 1);
}

// ---- register-tiled batched lookahead (a SIMT "GEMM" with sequential sums) --
// The K candidates share every A_nb / T element they read. Pricing
// (k_la_gemm_price): a CTA of 256 threads computes a 64-candidate x 128-slot
// tile of outputs, 8 x 4 per thread (32 independent chains per thread); theta'
// (k_la_gemm_theta): 64 candidates x 64 rows, 4 x 4 per thread. Both stream
// 16-deep chunks of their operands into a 3-stage shared-memory ring with 2D
// TMA tensor copies issued by one thread (a full mbarrier per stage carries
// the bytes; the chunk barrier frees the stage two chunks ahead), so no thread
// spends issue slots on loads: on the C4 shape the per-thread cp.async form of
// the same loop ran at 0.80 of the fp64 peak, the TMA form at 0.92, the loop
// with no loads at all at 0.95 (tools/microbench/la_price_rate.cu). The
// candidate-side operands land as [64 k][16 i] boxes and are read two chunk
// rows at a time (LDS.128 broadcasts). <= 128 registers per thread keep 16
// warps per SM to hide the DMUL -> DADD dependency. Each output is one chain in
// ascending reduction index, bit for bit the reference's dot (solver.cpp:
// 190-200, 203-210): DMUL + DADD, never DFMA.
constexpr int kLK = 64;    // candidates per CTA tile
constexpr int kLN = 128;   // slots per pricing tile
constexpr int kLC = 16;    // reduction chunk
constexpr int kLS = 3;     // ring stages
constexpr int kLThreads = 256;

struct LaPriceSmem {
    double W[kLS][kLK][kLC];   // [k][i]  W'_k, i = chunk row
    double A[kLS][kLC][kLN];   // [i][s]  A_nb slots
    uint64_t full[kLS];
};

// z_k(s) = dot(W'_k, a_s) - c_j over this shard's slots (j = slot2col[s] != q):
// the best (z, j) of the tile's 128 slots per candidate -> part_z/part_j[k][bx].
// tmW: W' as {m, K} with box {16, 64}; tmA: A_nb as {ld_nb, m} with box
// {128, 16} (slots past n_scan hold stale values whose outputs are discarded).
//
// only_if_fail: the fallback of the bounded pricing (exits at once unless
// la.fail was set).
__global__ void __launch_bounds__(kLThreads, 2)
k_la_gemm_price(Dev d, LookaheadDev la, const __grid_constant__ CUtensorMap tmW,
                const __grid_constant__ CUtensorMap tmA, int only_if_fail) {
    if (only_if_fail && !*la.fail) return;
    extern __shared__ __align__(128) unsigned char la_smem[];
    LaPriceSmem& sm = *reinterpret_cast<LaPriceSmem*>(la_smem);
    const int n_scan = d.ctl->n_scan;
    const double* cost = phase_cost(d, d.ctl->phase);
    const int s0 = blockIdx.x * kLN, k0 = blockIdx.y * kLK;
    // warp = one group of 8 candidates tk * 8 + u; lanes = 32 consecutive slots ts + 32 v
    const int t = threadIdx.x, tk = t >> 5, ts = t & 31;
    const int m = d.m;
    if (t == 0) {
        for (int s = 0; s < kLS; ++s) mbar_init(&sm.full[s], 1);
        mbar_fence_init();
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
        __syncthreads();  // every thread is done with chunk ch - 1: its stage takes chunk ch + 2
        if (t == 0 && ch + kLS - 1 < nch) issue((ch + kLS - 1) % kLS, (ch + kLS - 1) * kLC);
        const int stg = ch % kLS;
        mbar_wait(&sm.full[stg], (uint32_t)(ch / kLS) & 1u);
        const int lim = min(kLC, m - ch * kLC);
        if (lim == kLC) {
#pragma unroll
            for (int ii = 0; ii < kLC; ii += 2) {
                double w0[8], w1[8], a0[4], a1[4];
#pragma unroll
                for (int u = 0; u < 8; ++u) {  // broadcast: the warp shares its 8 candidates
                    const double2 v2 = *reinterpret_cast<const double2*>(&sm.W[stg][tk * 8 + u][ii]);
                    w0[u] = v2.x;
                    w1[u] = v2.y;
                }
#pragma unroll
                for (int v = 0; v < 4; ++v) {
                    a0[v] = sm.A[stg][ii][ts + 32 * v];
                    a1[v] = sm.A[stg][ii + 1][ts + 32 * v];
                }
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = dadd(acc[u][v], dmul(w0[u], a0[v]));
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = dadd(acc[u][v], dmul(w1[u], a1[v]));
            }
        } else {
            for (int ii = 0; ii < lim; ++ii) {
                double w[8], a[4];
#pragma unroll
                for (int u = 0; u < 8; ++u) w[u] = sm.W[stg][tk * 8 + u][ii];
#pragma unroll
                for (int v = 0; v < 4; ++v) a[v] = sm.A[stg][ii][ts + 32 * v];
#pragma unroll
                for (int u = 0; u < 8; ++u)
#pragma unroll
                    for (int v = 0; v < 4; ++v) acc[u][v] = dadd(acc[u][v], dmul(w[u], a[v]));
            }
        }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        double bz = -kInf;
        int bj = INT_MAX;
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int sl = s0 + ts + 32 * v;
            if (sl < n_scan) {
                const int j = d.slot2col[sl];
                if (j != la.q) {
                    const double z = dsub(acc[u][v], cost[j]);
                    if (better(z, j, bz, bj)) { bz = z; bj = j; }
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {  // the warp's 32 lanes share candidate tk * 8 + u
            const double oz = __shfl_xor_sync(0xffffffffu, bz, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (better(oz, oj, bz, bj)) { bz = oz; bj = oj; }
        }
        const int k = k0 + tk * 8 + u;
        if (ts == 0 && k < la.K) {
            la.part_z[(size_t)k * la.nblk + blockIdx.x] = bz;
            la.part_j[(size_t)k * la.nblk + blockIdx.x] = bj;
        }
    }
}

// CTA-batched per-candidate sequential dots acc_c = sum_i u_c[i] v_c[i] for
// kDC candidates per CTA (u_c = a row of X or W', v_c = A_cm column vcol_c;
// vcol_c < 0: no dot). All kDT threads stage kDR-row chunks of the 2 x kDC
// vectors in shared memory (each warp load is 32 consecutive rows of one
// vector: 256 contiguous bytes), double-buffered so the next chunk's loads are
// in flight while threads 0..kDC-1 run their chains over the current one in
// ascending i. The chains are latency-bound (8 cycles per DADD), so a CTA per
// 16 candidates spreads them over ~K/16 SMs; the earlier warp-per-32-candidates
// form kept 32 warps busy for 0.4-1.2 ms at K = 1000, m = 4000.
constexpr int kDC = 16;   // candidates per CTA
constexpr int kDR = 64;   // rows per chunk
constexpr int kDT = 128;  // threads per CTA

struct DotSmem {
    double u[2][kDC][kDR + 1];  // +1: chain reads of 16 candidates hit 16 bank pairs
    double v[2][kDC][kDR + 1];
    const double* ub[kDC];
    int vc[kDC];
};

// Returns acc in threads c < kDC (candidate c of the CTA); sm.ub / sm.vc set
// and synchronised by the caller.
__device__ __forceinline__ double cta_batched_dot(DotSmem& sm, const double* __restrict__ A_cm, size_t ld_cm,
                                                  int n) {
    const int t = threadIdx.x;
    const int r = t & (kDR - 1), c0 = t / kDR;  // row in chunk, first candidate
    constexpr int kPer = kDC * kDR / kDT;       // loads per thread per vector
    double ru[kPer], rv[kPer];
    auto fetch = [&](int i0) {
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int c = c0 + q * (kDT / kDR);
            const int i = i0 + r;
            const double* ub = sm.ub[c];
            const int vc = sm.vc[c];
            ru[q] = (ub && i < n) ? __ldg(ub + i) : 0.0;
            rv[q] = (vc >= 0 && i < n) ? __ldg(A_cm + (size_t)vc * ld_cm + i) : 0.0;
        }
    };
    auto stash = [&](int b) {
#pragma unroll
        for (int q = 0; q < kPer; ++q) {
            const int c = c0 + q * (kDT / kDR);
            sm.u[b][c][r] = ru[q];
            sm.v[b][c][r] = rv[q];
        }
    };
    double acc = 0.0;
    const int nch = (n + kDR - 1) / kDR;
    fetch(0);
    stash(0);
    __syncthreads();
    for (int ch = 0; ch < nch; ++ch) {
        const int b = ch & 1;
        if (ch + 1 < nch) fetch((ch + 1) * kDR);
        if (t < kDC && sm.vc[t] >= 0) {
            const int lim = min(kDR, n - ch * kDR);
            const double* __restrict__ uu = sm.u[b][t];
            const double* __restrict__ vv = sm.v[b][t];
            for (int e = 0; e < lim; ++e) acc = dadd(acc, dmul(uu[e], vv[e]));
        }
        if (ch + 1 < nch) stash(b ^ 1);
        __syncthreads();
    }
    return acc;
}

// The leaving variable of candidate k re-enters the nonbasic set
// (solver.cpp:186-188): priced by the shard owning its column, into the last
// partial slot (index nblk - 1).
__global__ void __launch_bounds__(kDT) k_la_leave(Dev d, LookaheadDev la) {
    __shared__ DotSmem sm;
    const int k0 = blockIdx.x * kDC;
    if (threadIdx.x < kDC) {
        const int k = k0 + threadIdx.x;
        int p = -1;
        if (k < la.K) {
            const int pl = d.basic[la.rows[k]];
            if (pl < d.n_total && pl != la.q && pl >= d.col0 && pl < d.col1) p = pl;
        }
        sm.vc[threadIdx.x] = p;
        sm.ub[threadIdx.x] = k < la.K ? la.Wp + (size_t)k * la.ldx : nullptr;
    }
    __syncthreads();
    const double acc = cta_batched_dot(sm, d.A_cm, d.ld_cm, d.m);
    const int k = k0 + threadIdx.x;
    if (threadIdx.x >= kDC || k >= la.K) return;
    const int p = sm.vc[threadIdx.x];
    double bz = -kInf;
    int bj = INT_MAX;
    if (p >= 0) {
        bz = dsub(acc, phase_cost(d, d.ctl->phase)[p]);
        bj = p;
    }
    la.part_z[(size_t)k * la.nblk + la.nblk - 1] = bz;
    la.part_j[(size_t)k * la.nblk + la.nblk - 1] = bj;
}

// The candidate's own pivot row r_k becomes X_k (solver.cpp:176): its y' is
// dot(X_k, a_{b_k}) and its b_bar' is X_k[m]. The tiled kernel skips that row;
// this one computes its ratio into own_t[k].
__global__ void __launch_bounds__(kDT) k_la_own(Dev d, LookaheadDev la) {
    __shared__ DotSmem sm;
    const int k0 = blockIdx.x * kDC;
    if (threadIdx.x < kDC) {
        const int k = k0 + threadIdx.x;
        int col = -1;
        if (k < la.K) {
            const int rk = la.rows[k], bj = la.bj[k];
            if (bj >= 0 && rk >= d.row0 && rk < d.row0 + d.mloc && !d.frozen[rk]) col = bj;
        }
        sm.vc[threadIdx.x] = col;
        sm.ub[threadIdx.x] = k < la.K ? la.X + (size_t)k * la.ldx : nullptr;
    }
    __syncthreads();
    const double acc = cta_batched_dot(sm, d.A_cm, d.ld_cm, d.m);
    const int k = k0 + threadIdx.x;
    if (threadIdx.x >= kDC || k >= la.K) return;
    double th = kInf;
    if (sm.vc[threadIdx.x] >= 0 && !(acc <= d.pivot_tol)) th = ddiv(sm.ub[threadIdx.x][d.m], acc);
    la.own_t[k] = th;
}

constexpr int kLT = 64;  // theta tile edge

struct LaThetaSmem {
    double T[kLS][kLC][kLT];  // [j][i]  T_ij of the tile's 64 rows
    double X[kLS][kLT][kLC];  // [k][j]  X_kj
    double B[kLS][kLT][kLC];  // [k][j]  a_{b_k}[j] (gathered by k_la_gather)
    uint64_t full[kLS];
    int bj[kLT], rk[kLT];
};

// Bg[k][j] = a_{b_k}[j] (j < m), zero rows for candidates without an entering
// column: the theta' GEMM's third operand as one strided matrix that a TMA box
// can stream (it reuses W', which pricing no longer needs).
__global__ void k_la_gather(Dev d, LookaheadDev la) {
    const int k = blockIdx.y;
    const int b = la.bj[k];
    double* out = la.Wp + (size_t)k * la.ldx;
    const double* a = b >= 0 ? d.A_cm + (size_t)b * d.ld_cm : nullptr;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < d.m; j += gridDim.x * blockDim.x)
        out[j] = a ? a[j] : 0.0;
}

// y'_ik = sum_j t_ij(k) a_{b_k}[j] for this shard's rows, t = X_kj on the
// candidate's own row, T_ij where y_i == 0, else T_ij - y_i X_kj (solver.cpp:
// 177-184, 203-210); theta'_k partial (min ratio) per 64-row tile -> part_t[k][bx].
// 64 x 64 tiles, 4 x 4 outputs per thread over 256 threads. tmT: T as
// {mloc, m} with box {64, 16}; tmX / tmB: X and Bg as {m, K} with box {16, 64}.
__global__ void __launch_bounds__(256, 2)
k_la_gemm_theta(Dev d, LookaheadDev la, const __grid_constant__ CUtensorMap tmT,
                const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmB) {
    extern __shared__ __align__(128) unsigned char la_smem[];
    LaThetaSmem& sm = *reinterpret_cast<LaThetaSmem*>(la_smem);
    const int m = d.m;
    const int i0 = blockIdx.x * kLT, k0 = blockIdx.y * kLT;
    const int t = threadIdx.x, ti = t & 15, tk = t >> 4;
    if (t < kLT) {
        const int k = k0 + t;
        sm.bj[t] = k < la.K ? la.bj[k] : -1;
        sm.rk[t] = k < la.K ? la.rows[k] : -1;
    }
    if (t == 0) {
        for (int s = 0; s < kLS; ++s) mbar_init(&sm.full[s], 1);
        mbar_fence_init();
    }
    __syncthreads();
    bool any = false;
    for (int kk = 0; kk < kLT; ++kk) any |= sm.bj[kk] >= 0;
    if (!any) {  // no candidate of this tile has an entering column: score 0
        if (ti == 0)
            for (int v = 0; v < 4; ++v) {
                const int k = k0 + tk + 16 * v;
                if (k < la.K) la.part_t[(size_t)k * la.nblk_t + blockIdx.x] = kInf;
            }
        return;
    }
    double yv[4];
    bool rowok[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int li = i0 + ti + 16 * u;
        rowok[u] = li < d.mloc;
        yv[u] = rowok[u] ? d.Y[li] : 0.0;
    }
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) acc[u][v] = 0.0;
    // Chains use T_ij - y_i X_kj; rows with y_i == 0 keep T_ij exactly as the
    // reference does (solver.cpp:177-184: T - 0*X would flip a -0 entry of a
    // former pivot row). The row kind is fixed per thread row, so it costs one
    // select per element. The candidate's own row (t = X_kj) is skipped here and
    // handled by k_la_own.
    bool zrow[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) zrow[u] = yv[u] == 0.0;
    // some X_kj is inf/NaN: keep the select (la_exact forces it: a parity check
    // of that path, tests/test_gpu_parity.py)
    const bool exact = *la.nonfinite != 0 || d.la_exact != 0;
    constexpr uint32_t kBytes = (kLC * kLT + 2 * kLT * kLC) * 8;
    auto issue = [&](int stage, int j0) {
        mbar_expect_tx(&sm.full[stage], kBytes);
        tma_load_2d(&sm.T[stage][0][0], &tmT, i0, j0, &sm.full[stage]);
        tma_load_2d(&sm.X[stage][0][0], &tmX, j0, k0, &sm.full[stage]);
        tma_load_2d(&sm.B[stage][0][0], &tmB, j0, k0, &sm.full[stage]);
    };
    const int nch = (m + kLC - 1) / kLC;
    if (t == 0)
        for (int st = 0; st < kLS - 1 && st < nch; ++st) issue(st, st * kLC);
    // exact: rows with y_i == 0 take T_ij itself (a select per element).
    // fast: T_ij - y_i X_kj for every row. With y_i = +-0 and X_kj finite
    // that differs from T_ij only in the sign of a zero, and a zero term
    // never changes the chain (acc starts at +0.0 and round-to-nearest
    // never produces -0.0 from it), so the chains are bit-identical.
    auto step = [&](const double (&tv)[4], const double (&xv)[4], const double (&bv)[4], auto sel) {
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                const double sub = dsub(tv[u], dmul(yv[u], xv[v]));
                acc[u][v] = dadd(acc[u][v], dmul(decltype(sel)::value && zrow[u] ? tv[u] : sub, bv[v]));
            }
    };
    auto run = [&](int stg, int lim, auto sel) {
        if (lim == kLC) {
#pragma unroll
            for (int jj = 0; jj < kLC; jj += 2) {
                double t0[4], t1[4], x0[4], x1[4], b0[4], b1[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    t0[u] = sm.T[stg][jj][ti + 16 * u];
                    t1[u] = sm.T[stg][jj + 1][ti + 16 * u];
                    const double2 xx = *reinterpret_cast<const double2*>(&sm.X[stg][tk + 16 * u][jj]);
                    const double2 bb = *reinterpret_cast<const double2*>(&sm.B[stg][tk + 16 * u][jj]);
                    x0[u] = xx.x;
                    x1[u] = xx.y;
                    b0[u] = bb.x;
                    b1[u] = bb.y;
                }
                step(t0, x0, b0, sel);
                step(t1, x1, b1, sel);
            }
        } else {
            for (int jj = 0; jj < lim; ++jj) {
                double tv[4], xv[4], bv[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    tv[u] = sm.T[stg][jj][ti + 16 * u];
                    xv[u] = sm.X[stg][tk + 16 * u][jj];
                    bv[u] = sm.B[stg][tk + 16 * u][jj];
                }
                step(tv, xv, bv, sel);
            }
        }
    };
    for (int ch = 0; ch < nch; ++ch) {
        __syncthreads();  // every thread is done with chunk ch - 1: its stage takes chunk ch + 2
        if (t == 0 && ch + kLS - 1 < nch) issue((ch + kLS - 1) % kLS, (ch + kLS - 1) * kLC);
        const int stg = ch % kLS;
        mbar_wait(&sm.full[stg], (uint32_t)(ch / kLS) & 1u);
        const int lim = min(kLC, m - ch * kLC);
        if (exact) run(stg, lim, std::true_type{});
        else run(stg, lim, std::false_type{});
    }
    const double* bcol = d.T + (size_t)m * d.ldT;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const int kk = tk + 16 * v, k = k0 + kk;
        double th = kInf;
        if (k < la.K && sm.bj[kk] >= 0) {
            const double xm = la.X[(size_t)k * la.ldx + m];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int li = i0 + ti + 16 * u;
                if (!rowok[u] || d.frozen[d.row0 + li] || d.row0 + li == sm.rk[kk]) continue;
                if (acc[u][v] <= d.pivot_tol) continue;
                const double bb = zrow[u] ? bcol[li] : dsub(bcol[li], dmul(yv[u], xm));
                th = min_keep(th, ddiv(bb, acc[u][v]));
            }
        }
        for (int o = 8; o > 0; o >>= 1) th = min_keep(th, __shfl_xor_sync(0xffffffffu, th, o));
        if (ti == 0 && k < la.K) la.part_t[(size_t)k * la.nblk_t + blockIdx.x] = th;
    }
}

// ---- bounded pricing: a DMMA screen, exact chains only where it is unsure --
// z~_k(s) = W'_k . a_s - c_j on the fp64 tensor cores (mma.sync m8n8k4: any
// summation order, so its value differs from the reference's sequential chain
// by at most E = 3 gamma_m ||W'_k|| ||a_j|| + 4 u |z~| + 1e-300: both lie
// within gamma_m sum_i |W'_ki a_ij| (<= the norm product, Cauchy-Schwarz) of
// the exact dot, each subtraction of c_j adds u |z| (Higham, Accuracy and
// Stability of Numerical Algorithms, 3.1), and the absolute term covers
// flushed subnormals). The tile is pricing's 64 candidates x 128 slots; 8
// warps = 2 candidate halves x 4 slot quarters, 32 x 32 outputs per warp as
// 4 x 4 fragments; W' boxes land 128B-swizzled (conflict-free A fragments).
// Per tile and candidate it keeps max(z~ - E) -> part_L, and the few slots
// whose interval reaches that tile bound -> tl_s / tl_z.
// tools/microbench/la_price_rate.cu: 0.83 of the 37 TFLOP/s DMMA peak, against
// 0.69 for the same screen as SIMT DFMA.
__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c[0]), "+d"(c[1])
                 : "d"(a), "d"(b));
}
struct LaScreenSmem {
    double W[kLS][kLK][kLC];  // [k][i], rows 128B-swizzled by TMA
    double A[kLS][kLC][kLN];  // 8 boxes [i][16 s], rows 128B-swizzled (B fragments: 2-way, not 4-way)
    uint64_t full[kLS];
    double lo[kLK][4];        // per candidate x slot quarter
    int cnt[kLK];             // tile list: slots that may reach the candidate's global bound
    int cs[kLK][kLaTile];
    double cz[kLK][kLaTile];
};
//
// PROBE (the bounded selection's screen): the same tiles over a_{b_k} (in W''s
// buffer) x the gathered probe rows Tg (128 of them), split along the
// reduction over gridDim.z segments whose partial dots are atomically added
// into la.yacc (any order is fine for a screen); k_la_probe_cert bounds them.
template <bool PROBE>
__global__ void __launch_bounds__(kLThreads, 2)
k_la_screen(Dev d, LookaheadDev la, const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA) {
    extern __shared__ __align__(1024) unsigned char la_smem[];
    LaScreenSmem& sm =
        *reinterpret_cast<LaScreenSmem*>((reinterpret_cast<uintptr_t>(la_smem) + 1023) & ~uintptr_t(1023));
    const int n_scan = PROBE ? 0 : d.ctl->n_scan;
    const double* cost = PROBE ? nullptr : phase_cost(d, d.ctl->phase);
    const int s0 = blockIdx.x * kLN, k0 = blockIdx.y * kLK;
    const int t = threadIdx.x, warp = t >> 5, lane = t & 31, g = lane >> 2, tq = lane & 3;
    const int wc = warp & 1, ws = warp >> 1;
    const int m = d.m;
    if (t == 0) {
        for (int s = 0; s < kLS; ++s) mbar_init(&sm.full[s], 1);
        mbar_fence_init();
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
        for (int b = 0; b < kLN / 16; ++b)  // 8 boxes of 16 slots x 16 rows, 128B-swizzled, 2 KB each
            tma_load_2d(&sm.A[stage][0][0] + b * 16 * kLC, &tmA, s0 + 16 * b, i0, &sm.full[stage]);
    };
    // chunks [c0, c0 + nch) of the reduction (a partial last chunk is zero-filled by TMA)
    const int nall = (m + kLC - 1) / kLC;
    const int per = (nall + gridDim.z - 1) / gridDim.z;
    const int c0 = blockIdx.z * per;
    const int nch = max(0, min(per, nall - c0));
    if (t == 0)
        for (int st = 0; st < kLS - 1 && st < nch; ++st) issue(st, (c0 + st) * kLC);
    for (int ch = 0; ch < nch; ++ch) {
        __syncthreads();  // every thread is done with chunk ch - 1: its stage takes chunk ch + 2
        if (t == 0 && ch + kLS - 1 < nch) issue((ch + kLS - 1) % kLS, (c0 + ch + kLS - 1) * kLC);
        const int stg = ch % kLS;
        mbar_wait(&sm.full[stg], (uint32_t)(ch / kLS) & 1u);
        const double* Ws = &sm.W[stg][0][0];
#pragma unroll
        for (int kk = 0; kk < kLC / 4; ++kk) {
            const int e = kk * 4 + tq;
            double af[4], bf[4];
#pragma unroll
            for (int cb = 0; cb < 4; ++cb) {  // A fragment: row g, column tq (128B swizzle: 16-byte chunk ^ row % 8)
                const int r = wc * 32 + cb * 8 + g;
                af[cb] = Ws[r * kLC + ((((e >> 1) ^ (r & 7)) << 1) | (e & 1))];
            }
            const double* As = &sm.A[stg][0][0];
#pragma unroll
            for (int sb = 0; sb < 4; ++sb) {  // B: row tq, column g, in box ws * 2 + sb / 2 (swizzled like W')
                const int c = (sb & 1) * 8 + g;
                bf[sb] = As[(ws * 2 + (sb >> 1)) * 16 * kLC + e * 16 + ((((c >> 1) ^ (e & 7)) << 1) | (c & 1))];
            }
#pragma unroll
            for (int cb = 0; cb < 4; ++cb)
#pragma unroll
                for (int sb = 0; sb < 4; ++sb) dmma_8x8x4(acc[cb][sb], af[cb], bf[sb]);
        }
    }
    if (PROBE) {
        if (nch == 0) return;
#pragma unroll
        for (int cb = 0; cb < 4; ++cb) {
            const int k = k0 + wc * 32 + cb * 8 + g;
            if (k >= la.K) continue;
#pragma unroll
            for (int sb = 0; sb < 4; ++sb)
#pragma unroll
                for (int h = 0; h < 2; ++h) atomicAdd(la.yacc + (size_t)k * kLN + ws * 32 + sb * 8 + 2 * tq + h,
                                                      acc[cb][sb][h]);
        }
        return;
    }
    const double uu = 1.1102230246251565e-16;
    const double cE = 3.0 * (m * uu / (1.0 - m * uu)) * (1.0 + 1e-6);
    bool bad = false;
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
        const int kl = wc * 32 + cb * 8 + g, k = k0 + kl;
        const double wn = k < la.K ? la.wnorm[k] : 0.0;
        double lo = -kInf;
#pragma unroll
        for (int sb = 0; sb < 4; ++sb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {  // C fragment: row g, columns 2 tq + h
                const int sl = s0 + ws * 32 + sb * 8 + 2 * tq + h;
                if (sl < n_scan && k < la.K) {
                    const int j = d.slot2col[sl];
                    const double z = acc[cb][sb][h] - cost[j];
                    const double e = cE * wn * la.anorm[j] + 4.0 * uu * fabs(z) + 1e-300;
                    bad |= !isfinite(z) || !isfinite(e);
                    acc[cb][sb][h] = j != la.q ? z : -kInf;  // keep z~ (and e below) for the tile list
                    if (j != la.q) lo = fmax(lo, z - e);
                } else {
                    acc[cb][sb][h] = -kInf;
                }
            }
        lo = fmax(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
        lo = fmax(lo, __shfl_xor_sync(0xffffffffu, lo, 2));
        if (tq == 0) sm.lo[kl][ws] = lo;
        if (t < kLK) sm.cnt[t] = 0;
    }
    if (bad) *la.fail = 1;
    __syncthreads();
    // The tile's own best lower bound L_t <= the global L_k, so a slot with
    // z~ + E < L_t can never enter k_la_cands' list: only the few others are
    // kept (slot, z~), kLaTile per (candidate, tile); more sets la.fail.
#pragma unroll
    for (int cb = 0; cb < 4; ++cb) {
        const int kl = wc * 32 + cb * 8 + g, k = k0 + kl;
        if (k >= la.K) continue;
        const double Lt = fmax(fmax(sm.lo[kl][0], sm.lo[kl][1]), fmax(sm.lo[kl][2], sm.lo[kl][3]));
        const double wn = la.wnorm[k];
#pragma unroll
        for (int sb = 0; sb < 4; ++sb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const double z = acc[cb][sb][h];
                if (z == -kInf) continue;
                const int sl = s0 + ws * 32 + sb * 8 + 2 * tq + h;
                const double e = cE * wn * la.anorm[d.slot2col[sl]] + 4.0 * uu * fabs(z) + 1e-300;
                if (z + e >= Lt) {
                    const int c = atomicAdd(&sm.cnt[kl], 1);
                    if (c < kLaTile) {
                        sm.cs[kl][c] = sl;
                        sm.cz[kl][c] = z;
                    }
                }
            }
    }
    __syncthreads();
    if (t < kLK && k0 + t < la.K) {
        const int k = k0 + t;
        la.part_L[(size_t)k * la.nblk + blockIdx.x] =
            fmax(fmax(sm.lo[t][0], sm.lo[t][1]), fmax(sm.lo[t][2], sm.lo[t][3]));
        const int n = sm.cnt[t];
        if (n > kLaTile) *la.fail = 1;
        const size_t base = ((size_t)k * (la.nblk - 1) + blockIdx.x) * kLaTile;
        la.tl_n[(size_t)k * (la.nblk - 1) + blockIdx.x] = min(n, kLaTile);
        for (int c = 0; c < min(n, kLaTile); ++c) {
            la.tl_s[base + c] = sm.cs[t][c];
            la.tl_z[base + c] = sm.cz[t][c];
        }
    }
}

// exact chains only where the screen is unsure:

__global__ void k_colnorm(Dev d, double* out) {  // one warp per column
    const int j = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x & 31;
    if (j >= d.n_total) return;
    const double* a = d.A_cm + (size_t)j * d.ld_cm;
    double s = 0.0;
    for (int i = lane; i < d.m; i += 32) s = fma(a[i], a[i], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[j] = sqrt(s);
}

__global__ void k_la_wnorm(Dev d, LookaheadDev la) {  // one CTA per candidate
    __shared__ double red[32];
    const int k = blockIdx.x;
    const double* w = la.Wp + (size_t)k * la.ldx;
    double s = 0.0;
    for (int i = threadIdx.x; i < d.m; i += blockDim.x) s = fma(w[i], w[i], s);
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int v = 0; v < (int)(blockDim.x >> 5); ++v) t += red[v];
        la.wnorm[k] = sqrt(t);
        la.cn[k] = 0;
    }
}

// Candidate k's columns whose interval [z~ - E, z~ + E] reaches L_k, the best
// lower bound (the tiles' and the leaving column's exact z): every column
// that can be the exact (max z, min j) lies among them (one CTA per candidate).
__global__ void __launch_bounds__(256) k_la_cands(Dev d, LookaheadDev la) {
    __shared__ double red[8];
    const int k = blockIdx.x;
    const int ntile = la.nblk - 1;
    double L = la.part_z[(size_t)k * la.nblk + ntile];  // leaving column, exact (k_la_leave)
    for (int b = threadIdx.x; b < ntile; b += blockDim.x) L = fmax(L, la.part_L[(size_t)k * la.nblk + b]);
    for (int o = 16; o > 0; o >>= 1) L = fmax(L, __shfl_xor_sync(0xffffffffu, L, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = L;
    __syncthreads();
    L = red[0];
    for (int v = 1; v < 8; ++v) L = fmax(L, red[v]);
    const double uu = 1.1102230246251565e-16;
    const double cE = 3.0 * (d.m * uu / (1.0 - d.m * uu)) * (1.0 + 1e-6);
    const double wn = la.wnorm[k];
    for (int e0 = threadIdx.x; e0 < ntile * kLaTile; e0 += blockDim.x) {  // the tiles' lists
        const int b = e0 / kLaTile, c0 = e0 % kLaTile;
        if (c0 >= la.tl_n[(size_t)k * ntile + b]) continue;
        const size_t at = ((size_t)k * ntile + b) * kLaTile + c0;
        const int j = d.slot2col[la.tl_s[at]];
        const double z = la.tl_z[at];
        const double e = cE * wn * la.anorm[j] + 4.0 * uu * fabs(z) + 1e-300;
        if (z + e >= L) {
            const int c = atomicAdd(la.cn + k, 1);
            if (c >= kLaCand) {
                *la.fail = 1;
                continue;
            }
            la.cj[k * kLaCand + c] = j;
            const int p = atomicAdd(la.npairs, 1);
            if (p < kLaPairs) la.pairs[p] = k * kLaCand + c;
            else *la.fail = 1;
        }
    }
}

// The listed (k, j): exact z = dot(W'_k, a_j) - c_j, the reference's chain
// (solver.cpp:190-200), 16 per CTA through cta_batched_dot.
__global__ void __launch_bounds__(kDT) k_la_exact(Dev d, LookaheadDev la) {
    __shared__ DotSmem sm;
    const int np = min(*la.npairs, kLaPairs);
    const int p0 = blockIdx.x * kDC;
    if (p0 >= np || *la.fail) return;
    if (threadIdx.x < kDC) {
        const int p = p0 + threadIdx.x;
        const int e = p < np ? la.pairs[p] : -1;
        sm.vc[threadIdx.x] = e >= 0 ? la.cj[e] : -1;
        sm.ub[threadIdx.x] = e >= 0 ? la.Wp + (size_t)(e / kLaCand) * la.ldx : nullptr;
    }
    __syncthreads();
    const double acc = cta_batched_dot(sm, d.A_cm, d.ld_cm, d.m);
    const int p = p0 + threadIdx.x;
    if (threadIdx.x >= kDC || p >= np) return;
    const double* cost = phase_cost(d, d.ctl->phase);
    la.cz[la.pairs[p]] = dsub(acc, cost[sm.vc[threadIdx.x]]);
}

// Each candidate's exact best over its list into pricing partial 0 (the other
// tile partials are cleared; the leaving column's stays in nblk - 1).
__global__ void k_la_cands_best(Dev d, LookaheadDev la) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= la.K || *la.fail) return;
    double bz = -kInf;
    int bj = INT_MAX;
    const int n = min(la.cn[k], kLaCand);
    for (int c = 0; c < n; ++c) {
        const double z = la.cz[k * kLaCand + c];
        const int j = la.cj[k * kLaCand + c];
        if (better(z, j, bz, bj)) { bz = z; bj = j; }
    }
    for (int b = 0; b < la.nblk - 1; ++b) {
        la.part_z[(size_t)k * la.nblk + b] = b == 0 ? bz : -kInf;
        la.part_j[(size_t)k * la.nblk + b] = b == 0 ? bj : INT_MAX;
    }
}

// ---- bounded selection: select_leaving without the theta' GEMM ----------
// select_leaving keeps the FIRST survivor with the largest score (strict '>'
// from best = -1, solver.cpp:228-235). Scores are best_z * theta' with
// best_z > opt_tol, so score_k <= 0 as soon as ONE eligible row of candidate k's
// pivoted tableau has a ratio <= 0: rhs'_ik <= 0 and y'_ik > pivot_tol (theta'
// is a min). On a degenerate tie that holds for every candidate (C4: all ~1000
// scores are exactly 0), and if the first candidate's score is provably +-0
// (some ratio <= 0 and no eligible ratio < 0, i.e. no row with rhs' < 0), no
// later candidate can beat it. The probe computes y'_ik on kLaProbe rows with
// b_bar_i <= 0 for every candidate, in the reference's exact order and
// arithmetic (the same chain as k_la_gemm_theta), so each certificate is a
// fact about the reference's own values; anything unproven falls back to the
// full scoring. The decision is the reference's, bit for bit, either way.

// the first kLaProbe non-frozen rows with b_bar_i <= 0, ascending (one CTA);
// round r probes rows [64 r, 64 r + 64) of them
__global__ void __launch_bounds__(1024) k_la_probe_rows(Dev d, LookaheadDev la) {
    __shared__ int base, wcnt[32];
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const double* bcol = d.T + (size_t)d.m * d.ldT;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i0 = 0; i0 < d.m; i0 += 1024) {
        const int i = i0 + threadIdx.x;
        const bool pick = i < d.m && !d.frozen[i] && bcol[i] <= 0.0;
        const unsigned bal = __ballot_sync(0xffffffffu, pick);
        if (lane == 0) wcnt[w] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int v = 0; v < w; ++v) off += wcnt[v];
        off += __popc(bal & ((1u << lane) - 1u));
        if (pick && off < kLaProbe) la.prow[off] = i;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int v = 0; v < 32; ++v) base += wcnt[v];
        __syncthreads();
        if (base >= kLaProbe) break;
    }
    if (threadIdx.x == 0) *la.nprow = min(base, kLaProbe);
}

// Tg[j][r] = T_{prow[r], j} (j < m), zero for r >= nprow
__global__ void k_la_probe_gather(Dev d, LookaheadDev la) {
    const int np = *la.nprow;
    const size_t n = (size_t)d.m * kLaProbe;
    for (size_t e = (size_t)blockIdx.x * blockDim.x + threadIdx.x; e < n; e += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(e % kLaProbe);
        const size_t j = e / kLaProbe;
        la.Tg[e] = r < np ? d.T[j * d.ldT + la.prow[r]] : 0.0;
    }
}

// Screen inputs, any summation order: B_k = a_{b_k} gathered into W''s buffer
// (as k_la_gather) with xb = X_k . B_k, ||X_k|| and ||B_k|| on the way (blocks
// b < K, one per candidate), and ||T_i|| (j < m) of the screened probe rows
// from their gathered columns (blocks K .. K + 127).
__global__ void k_la_probe_norms(Dev d, LookaheadDev la) {
    __shared__ double red[3][32];
    const int b = blockIdx.x;
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    if (b < la.K) {
        const int c = la.bj[b];
        const double* x = la.X + (size_t)b * la.ldx;
        const double* a = c >= 0 ? d.A_cm + (size_t)c * d.ld_cm : nullptr;
        double* out = la.Wp + (size_t)b * la.ldx;
        for (int j = threadIdx.x; j < d.m; j += blockDim.x) {
            const double w = a ? a[j] : 0.0, xv = x[j];
            out[j] = w;
            s0 = fma(xv, w, s0);
            s1 = fma(xv, xv, s1);
            s2 = fma(w, w, s2);
        }
    } else {  // probe row r = b - K: ||T_row|| from its gathered column
        const int r = b - la.K;
        for (int j = threadIdx.x; j < d.m; j += blockDim.x) {
            const double v = la.Tg[(size_t)j * kLaProbe + r];
            s1 = fma(v, v, s1);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        s0 += __shfl_xor_sync(0xffffffffu, s0, o);
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) { red[0][w] = s0; red[1][w] = s1; red[2][w] = s2; }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, c = 0.0, e = 0.0;
        for (int v = 0; v < (int)(blockDim.x >> 5); ++v) { a += red[0][v]; c += red[1][v]; e += red[2][v]; }
        if (b < la.K) {
            la.pxb[b] = a;
            la.pxn[b] = sqrt(c);
            la.pbn[b] = sqrt(e);
        } else {
            la.ptn[b - la.K] = sqrt(c);
        }
    }
}

// Certificates from the screen (first kLN probe rows): y~ = yacc - y_i xb_k
// differs from the reference's y'_ik by at most
// E = (2 gamma_m + 5u)(1 + 1e-6)(||T_i|| + |y_i| ||X_k||) ||B_k|| + 2u|y~| + 1e-300
// (the elementwise T'_ij = T_ij - y_i X_kj rounding, both dots' gamma_m, the
// final subtraction; flushed subnormals in the absolute term). ok[k] = 1 when a
// row i != r_k has rhs'_ik <= 0 (exact) and y~ - E > pivot_tol.
__global__ void k_la_probe_cert(Dev d, LookaheadDev la) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    const int k = e / kLN, r = e % kLN;
    if (k >= la.K || r >= *la.nprow || la.bj[k] < 0) return;
    const int row = la.prow[r];
    if (row == la.rows[k]) return;
    const int m = d.m;
    const double uu = 1.1102230246251565e-16;
    const double gam = m * uu / (1.0 - m * uu);
    const double y = d.Y[row];
    const double yt = la.yacc[(size_t)k * kLN + r] - y * la.pxb[k];
    const double E = (2.0 * gam + 5.0 * uu) * (1.0 + 1e-6) * (la.ptn[r] + fabs(y) * la.pxn[k]) * la.pbn[k] +
                     2.0 * uu * fabs(yt) + 1e-300;
    if (!isfinite(yt) || !isfinite(E)) return;
    const double xm = la.X[(size_t)k * la.ldx + m];
    const double bi = d.T[(size_t)m * d.ldT + row];
    const double rhs = y == 0.0 ? bi : dsub(bi, dmul(y, xm));
    if (rhs <= 0.0 && yt - E > d.pivot_tol) la.ok[k] = 1;
}

// candidates with a best column and no certificate yet, ascending (one CTA)
__global__ void __launch_bounds__(1024) k_la_probe_list(LookaheadDev la) {
    __shared__ int base, wcnt[32];
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int k0 = 0; k0 < la.K; k0 += 1024) {
        const int k = k0 + threadIdx.x;
        const bool pick = k < la.K && la.bj[k] >= 0 && !la.ok[k];
        const unsigned bal = __ballot_sync(0xffffffffu, pick);
        if (lane == 0) wcnt[w] = __popc(bal);
        __syncthreads();
        int off = base;
        for (int v = 0; v < w; ++v) off += wcnt[v];
        if (pick) la.clist[off + __popc(bal & ((1u << lane) - 1u))] = k;
        __syncthreads();
        if (threadIdx.x == 0)
            for (int v = 0; v < 32; ++v) base += wcnt[v];
        __syncthreads();
    }
    if (threadIdx.x == 0) *la.ncl = base;
}

// One probe round: y'_ik for the round's kLaProbeRound probe rows x the
// unproven candidates. A CTA of 128 threads takes the 64 rows x 8 candidates,
// 2 x 2 chains per thread (rows t % 32 + {0, 32}, candidates t / 32 + {0, 4}):
// per chain step 6 shared loads feed 16 fp64 instructions, which balances the
// shared-memory wavefronts against the fp64 pipe. 16-deep chunks are
// register-staged; the chains run in the reference's order and arithmetic
// (solver.cpp:177-184, 205). ok[k] = 1 when some row i != r_k has rhs'_ik <= 0
// and y'_ik > pivot_tol.
constexpr int kPC = 16, kPKc = 8;
__global__ void __launch_bounds__(128) k_la_probe(Dev d, LookaheadDev la, int round) {
    __shared__ double Ts[kPC][kLaProbeRound];
    __shared__ double Xs[kPKc][kPC];
    __shared__ double Bs[kPKc][kPC];
    const int ncl = *la.ncl, np = *la.nprow;
    const int r0 = round * kLaProbeRound;
    if (blockIdx.x * kPKc >= ncl || r0 >= np) return;
    const int m = d.m, t = threadIdx.x, tr = t & 31, tc = t >> 5;
    int kk[2], row[2];
    double yv[2];
    bool zr[2];
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        const int ci = blockIdx.x * kPKc + tc + 4 * v;
        kk[v] = ci < ncl ? la.clist[ci] : -1;
        const int r = r0 + tr + 32 * v;
        row[v] = r < np ? la.prow[r] : -1;
        yv[v] = row[v] >= 0 ? d.Y[row[v]] : 0.0;
        zr[v] = yv[v] == 0.0;
    }
    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};  // [row][candidate]
    // chunk loads: Tg 16 j x 64 rows (8 per thread), X and Bg 8 candidates x 16 j (1 each)
    double rt[8], rx, rb;
    auto fetch = [&](int j0) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = t + 128 * q, rr = e % kLaProbeRound, jj = e / kLaProbeRound;
            rt[q] = j0 + jj < m ? la.Tg[(size_t)(j0 + jj) * kLaProbe + r0 + rr] : 0.0;
        }
        const int jj = t % kPC, cc = t / kPC;
        const int c2 = blockIdx.x * kPKc + cc;
        const int k2 = c2 < ncl ? la.clist[c2] : -1;
        const bool ok = k2 >= 0 && j0 + jj < m;
        rx = ok ? la.X[(size_t)k2 * la.ldx + j0 + jj] : 0.0;
        rb = ok ? la.Wp[(size_t)k2 * la.ldx + j0 + jj] : 0.0;
    };
    fetch(0);
    for (int j0 = 0; j0 < m; j0 += kPC) {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int e = t + 128 * q;
            Ts[e / kLaProbeRound][e % kLaProbeRound] = rt[q];
        }
        Xs[t / kPC][t % kPC] = rx;
        Bs[t / kPC][t % kPC] = rb;
        __syncthreads();
        if (j0 + kPC < m) fetch(j0 + kPC);
        auto step = [&](int jj) {
            double tv[2], xv[2], bv[2];
#pragma unroll
            for (int v = 0; v < 2; ++v) {
                tv[v] = Ts[jj][tr + 32 * v];
                xv[v] = Xs[tc + 4 * v][jj];
                bv[v] = Bs[tc + 4 * v][jj];
            }
#pragma unroll
            for (int u = 0; u < 2; ++u)
#pragma unroll
                for (int v = 0; v < 2; ++v) {
                    // rows with y_i == 0 keep T_ij (solver.cpp:177-184)
                    const double tij = zr[u] ? tv[u] : dsub(tv[u], dmul(yv[u], xv[v]));
                    acc[u][v] = dadd(acc[u][v], dmul(tij, bv[v]));
                }
        };
        if (j0 + kPC <= m) {
#pragma unroll
            for (int jj = 0; jj < kPC; ++jj) step(jj);
        } else {
            for (int jj = 0; jj < m - j0; ++jj) step(jj);
        }
        __syncthreads();
    }
    const double* bcol = d.T + (size_t)m * d.ldT;
#pragma unroll
    for (int v = 0; v < 2; ++v) {
        const int k = kk[v];
        if (k < 0) continue;
        const double xm = la.X[(size_t)k * la.ldx + m];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            if (row[u] < 0 || row[u] == la.rows[k]) continue;
            const double rhs = zr[u] ? bcol[row[u]] : dsub(bcol[row[u]], dmul(yv[u], xm));
            if (rhs <= 0.0 && acc[u][v] > d.pivot_tol) la.ok[k] = 1;
        }
    }
}

// first = every candidate is certified (score <= 0) and the first one's score
// is exactly +-0: no best column, or (certified, best_z finite, and no eligible
// row -- own row included -- with rhs' < 0, so theta'_0 = +-0).
// Not proven: first = -(1 + 2 * uncertified candidates + (first score not
// provably +-0)), for the solver's trace.
__global__ void __launch_bounds__(1024) k_la_probe_decide(Dev d, LookaheadDev la) {
    __shared__ int nbad;
    if (threadIdx.x == 0) nbad = 0;
    __syncthreads();
    for (int k = threadIdx.x; k < la.K; k += blockDim.x)
        if (la.bj[k] >= 0 && !la.ok[k]) atomicAdd(&nbad, 1);
    bool neg = false;
    if (la.bj[0] >= 0) {
        const int r0 = la.rows[0];
        const double* X0 = la.X;
        const double xm = X0[d.m];
        const double* bcol = d.T + (size_t)d.m * d.ldT;
        for (int i = threadIdx.x; i < d.m; i += blockDim.x) {
            if (d.frozen[i]) continue;
            const double y = d.Y[i];
            const double rhs = i == r0 ? xm : (y == 0.0 ? bcol[i] : dsub(bcol[i], dmul(y, xm)));
            neg |= rhs < 0.0;
        }
    }
    neg = __syncthreads_or(neg);
    if (threadIdx.x == 0) {
        const bool cert = la.bj[0] < 0 || (!neg && isfinite(la.bz[0]));
        *la.first = (nbad == 0 && cert) ? 1 : -(1 + 2 * nbad + (cert ? 0 : 1));
    }
}

__global__ void k_la_price_local(Dev d, LookaheadDev la) {
    const int k = blockIdx.x;
    if (threadIdx.x >= 32) return;
    double z = -kInf;
    int j = INT_MAX;
    for (int b = threadIdx.x; b < la.nblk; b += 32) {
        const double oz = la.part_z[(size_t)k * la.nblk + b];
        const int oj = la.part_j[(size_t)k * la.nblk + b];
        if (better(oz, oj, z, j)) { z = oz; j = oj; }
    }
    warp_argmax(z, j);
    if (threadIdx.x == 0) la.pm[k] = PriceMsg{z, j, 0};
}

// msgs: nsrc x K (shard-major); lookahead_score's "best_j" and its 0-score rule
// (solver.cpp:190-201)
__global__ void k_la_decide(Dev d, LookaheadDev la, const PriceMsg* __restrict__ msgs, int nsrc) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= la.K) return;
    double z = -kInf;
    int j = INT_MAX;
    for (int g = 0; g < nsrc; ++g) {
        const PriceMsg mm = msgs[(size_t)g * la.K + k];
        if (better(mm.z, mm.j, z, j)) { z = mm.z; j = mm.j; }
    }
    la.bz[k] = z;
    la.bj[k] = (j == INT_MAX || z <= d.opt_tol) ? -1 : j;
}

__global__ void k_la_theta_local(Dev d, LookaheadDev la) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= la.K) return;
    double t = kInf;
    if (la.bj[k] >= 0) {
        for (int b = 0; b < la.nblk_t; ++b) t = min_keep(t, la.part_t[(size_t)k * la.nblk_t + b]);
        t = min_keep(t, la.own_t[k]);
    }
    la.tl[k] = t;
}

// tl: nsrc x K local theta' (shard-major); score = best_z * theta' (solver.cpp:211-212)
__global__ void k_la_score(Dev d, LookaheadDev la, const double* __restrict__ tl, int nsrc) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= la.K) return;
    if (la.bj[k] < 0) { la.score[k] = 0.0; return; }
    double t = kInf;
    for (int g = 0; g < nsrc; ++g) t = min_keep(t, tl[(size_t)g * la.K + k]);
    la.theta[k] = t;
    la.score[k] = isinf(t) ? kInf : dmul(la.bz[k], t);
}

// ------------------------------------------------- in-process exchange ---
__global__ void k_sum_i64(const long long* __restrict__ in, int nsrc, size_t n, long long* out) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        long long v = 0;
        for (int g = 0; g < nsrc; ++g) v += in[(size_t)g * n + k];
        out[k] = v;
    }
}

__global__ void k_min_i32(const int* __restrict__ in, int nsrc, size_t n, int* out) {
    for (size_t k = blockIdx.x * (size_t)blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
        int v = INT_MAX;
        for (int g = 0; g < nsrc; ++g) v = min(v, in[(size_t)g * n + k]);
        out[k] = v;
    }
}

}  // namespace

// ------------------------------------------------------------- launchers ---
void launch_init_tableau(const Dev& d, const double* b, cudaStream_t st) {
    k_init_tableau<<<(d.mloc + 255) / 256, 256, 0, st>>>(d, b);
}

void launch_transpose(const double* A_rm, double* A_cm, int m, int n, long long ld, int* nonfinite,
                      cudaStream_t st) {
    dim3 grid((n + 31) / 32, (m + 31) / 32);
    k_transpose<<<grid, dim3(32, 8), 0, st>>>(A_rm, A_cm, m, n, ld, nonfinite);
}

void launch_build_nb_from_cm(const Dev& d, int n_scan, cudaStream_t st) {
    if (n_scan <= 0) return;
    dim3 grid((n_scan + 31) / 32, (d.m + 31) / 32);
    k_build_nb_cm<<<grid, dim3(32, 8), 0, st>>>(d, n_scan);
}

void launch_rebuild_top(const Dev& d, const double* init, double* out, cudaStream_t st) {
    k_rebuild_top<<<(d.m + 1 + 31) / 32, dim3(32, 8), 0, st>>>(d, init, out);
}

void launch_price_final(const Dev& d, cudaStream_t st) { k_price_final<<<1, 32, 0, st>>>(d); }

void launch_ratio_merge_parts(const Dev& d, const RatioMsg* msgs, const int* row0, int P, cudaStream_t st) {
    k_ratio_merge_parts<<<1, 32, 0, st>>>(d, msgs, row0, P);
}

void launch_ratio_final(const Dev& d, cudaStream_t st) { k_ratio_final<<<1, 32, 0, st>>>(d); }

namespace {
// Launch with programmatic stream serialization when d.pdl (single-GPU pivot chain).
template <class K>
void launch_chain(const Dev& d, K kernel, unsigned grid, unsigned block, size_t smem, cudaStream_t st) {
    if (!d.pdl) {
        kernel<<<grid, block, smem, st>>>(d);
        return;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(block);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, kernel, d);
}
}  // namespace

void launch_price(const Dev& d, cudaStream_t st) {
    launch_chain(d, k_price, d.price_grid, d.price_threads, d.price_smem, st);
}

void launch_update(const Dev& d, cudaStream_t st) {
    launch_chain(d, k_update, d.update_grid, d.upd_threads, d.upd_smem, st);
}

// Launch geometry of the streaming kernels and their TMA
// descriptors. Must run before the tableau is allocated: it fixes ldT.
void configure_kernels(Dev& d) {
    const int G = d.num_sms;
    // update + FTRAN: h rows per CTA (even, so the TMA box row is a 16-byte multiple)
    int h = (d.mloc + G - 1) / G;
    h = std::min(224, std::max(2, (h + 1) & ~1));  // <= 224 rows: 8 update + 7 FTRAN + 1 producer warps = 512 threads
    if (const char* e = xp_env("LPSG_UPD_H")) h = std::min(224, std::max(2, atoi(e) & ~1));  // shape experiments
    d.upd_h = h;
    d.update_grid = (d.mloc + h - 1) / h;
    // columns per stage: short row blocks (small m) take wide stages so the
    // per-stage handshakes amortise (C2 m=2000: +12 %); TMA boxes stop at 256
    d.upd_C = h <= 16 ? 128 : h <= 32 ? 64 : h <= 64 ? 32 : h <= 160 ? 16 : 8;
    if (const char* e = xp_env("LPSG_UPD_COLS")) d.upd_C = std::max(2, atoi(e)) & ~1;  // tuning experiments
    d.upd_U = 8;
    const size_t tile_el = (size_t)d.upd_C * h;
    const size_t stage = ((tile_el + 2 * (size_t)d.upd_C) * 8 + 1023) / 1024 * 1024;
    size_t s_cap = 8;
    if (const char* e = xp_env("LPSG_UPD_STAGES")) s_cap = (size_t)std::max(2, atoi(e));  // tuning experiments
    // >= 3 stages: the storer keeps 2 TMA stores in flight behind the update warps
    d.upd_S = (int)std::max<size_t>(3, std::min<size_t>(s_cap, (size_t)(200 * 1024) / stage));
    d.upd_smem = (int)(d.upd_S * stage + 3 * d.upd_S * 8);
    d.upd_threads = (d.upd_U + (h + 31) / 32 + 1) * 32;
    // pricing: one CTA per SM over contiguous slot ranges of this shard's columns
    const int ncols_local = d.col1 - d.col0;
    const PriceGeom gm = price_geom(ncols_local, G);
    d.pivot_grid = std::max(1, std::min(2 * G, (d.m + 1 + 255) / 256));
    d.price_grid = G;
    // one slot per consumer lane while 11 consumer warps cover the widest CTA
    // range, spread over at least min(4, w/8) warps (all four SM sub-partitions);
    // wider ranges (n_total > ~50k per GPU) use slot pairs
    if (gm.w <= 11 * 32 && !xp_env("LPSG_PRICE_PAIRS")) {  // env: A/B experiments
        d.price_spt = 1;
        d.price_nwc = std::max((gm.w + 31) / 32, std::min(4, (gm.w + 7) / 8));
    } else {
        d.price_spt = 2;
        d.price_nwc = (gm.w + 63) / 64;  // consumer threads own slot pairs
    }
    d.price_threads = (d.price_nwc + 1) * 32;
    d.price_stage_bytes = 0;
    for (int n = 1; n <= ncols_local; n = (n < 64 ? n + 1 : n + n / 64)) {
        const PriceGeom g = price_geom(n, G);
        const size_t st = (((size_t)g.R * g.w + g.R) * 8 + 1023) / 1024 * 1024;
        d.price_stage_bytes = std::max(d.price_stage_bytes, st);
    }
    {
        const PriceGeom g = price_geom(ncols_local, G);
        const size_t st = (((size_t)g.R * g.w + g.R) * 8 + 1023) / 1024 * 1024;
        d.price_stage_bytes = std::max(d.price_stage_bytes, st);
    }
    d.price_S = (int)std::max<size_t>(2, std::min<size_t>(6, (size_t)(192 * 1024) / d.price_stage_bytes));
    d.price_smem = (int)(d.price_S * d.price_stage_bytes + 2 * d.price_S * 8);
    cudaFuncSetAttribute(k_update, cudaFuncAttributeMaxDynamicSharedMemorySize, d.upd_smem);
    cudaFuncSetAttribute(k_price, cudaFuncAttributeMaxDynamicSharedMemorySize, d.price_smem);
    cudaFuncSetAttribute(k_la_gemm_price, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LaPriceSmem));
    cudaFuncSetAttribute(k_la_screen<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LaScreenSmem) + 1024);
    cudaFuncSetAttribute(k_la_screen<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LaScreenSmem) + 1024);
    cudaFuncSetAttribute(k_la_gemm_theta, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(LaThetaSmem));
    // One shared-memory carveout for every kernel: SMs never reconfigure the
    // L1/shared split between the streaming kernels and the small ones, and a
    // shard's spin-waiting exchange kernel can share an SM with another shard's
    // streaming CTA when shards share a GPU (a different carveout would make the
    // streaming kernel wait for the spinner to exit: deadlock).
    const void* all[] = {(const void*)k_init_tableau, (const void*)k_transpose, (const void*)k_build_nb_cm,
                         (const void*)k_rebuild_top, (const void*)k_price, (const void*)k_price_final,
                         (const void*)k_update, (const void*)k_ratio_final, (const void*)k_ratio,
                         (const void*)k_pivot_row, (const void*)k_pivot, (const void*)k_gather_row,
                         (const void*)k_drive_scan, (const void*)k_drive_red, (const void*)k_la_x,
                         (const void*)k_la_wp, (const void*)k_la_price_local,
                         (const void*)k_la_gemm_price, (const void*)k_la_screen<false>, (const void*)k_la_screen<true>, (const void*)k_la_gemm_theta, (const void*)k_la_leave,
                         (const void*)k_la_own,
                         (const void*)k_la_decide, (const void*)k_la_theta_local,
                         (const void*)k_la_score, (const void*)k_sum_i64, (const void*)k_min_i32,
                         (const void*)k_ratio_merge_parts};
    for (const void* f : all) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !p)
            return nullptr;
        fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

bool encode_2d(CUtensorMap* out, const void* base, uint64_t inner, uint64_t outer, uint64_t pitch_bytes,
               uint32_t box_inner, uint32_t box_outer, bool swizzle128 = false) {
    auto fn = get_encode();
    if (!fn) return false;
    const cuuint64_t dims[2] = {inner, outer};
    const cuuint64_t strides[1] = {pitch_bytes};
    const cuuint32_t box[2] = {box_inner, box_outer};
    const cuuint32_t estr[2] = {1, 1};
    return fn(out, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, swizzle128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// Encodes the TMA descriptors (T: one box shape; A_nb: one per slot-box width
// wbx = 8, 16, ..., 256) into device memory. Returns false on failure.
bool create_tensor_maps(Dev& d, CUtensorMap** dev_maps, int* count) {
    std::vector<CUtensorMap> maps;
    CUtensorMap mt;
    if (!encode_2d(&mt, d.T, (uint64_t)d.ldT, (uint64_t)d.m + 1, (uint64_t)d.ldT * 8, d.upd_h, d.upd_C))
        return false;
    maps.push_back(mt);
    const int nwb = 32;  // wbx = 8 .. 256
    for (int k = 1; k <= nwb; ++k) {
        const int wbx = 8 * k;
        CUtensorMap mp;
        if (!encode_2d(&mp, d.A_nb, (uint64_t)d.ld_nb, (uint64_t)d.m, (uint64_t)d.ld_nb * 8, wbx,
                       price_rows(wbx)))
            return false;
        maps.push_back(mp);
    }
    CUtensorMap* p = nullptr;
    if (cudaMalloc(&p, maps.size() * sizeof(CUtensorMap)) != cudaSuccess) return false;
    if (cudaMemcpy(p, maps.data(), maps.size() * sizeof(CUtensorMap), cudaMemcpyHostToDevice) != cudaSuccess)
        return false;
    d.tm_T = p;
    d.tm_nb = p + 1;
    *dev_maps = p;
    *count = (int)maps.size();
    return true;
}

void launch_ratio(const Dev& d, cudaStream_t st) { launch_chain(d, k_ratio, 1, 1024, 0, st); }

void launch_pivot(const Dev& d, cudaStream_t st) { launch_chain(d, k_pivot, d.pivot_grid, 256, 0, st); }

void launch_pivot_row(const Dev& d, cudaStream_t st) { k_pivot_row<<<d.pivot_grid, 256, 0, st>>>(d); }

void launch_gather_row(const Dev& d, int i, double* out, cudaStream_t st) {
    k_gather_row<<<(d.m + 1 + 255) / 256, 256, 0, st>>>(d, i, out);
}

void launch_drive_scan(const Dev& d, const double* g, cudaStream_t st) {
    k_drive_scan<<<d.price_grid, 256, 0, st>>>(d, g);
}

void launch_drive_red(const Dev& d, cudaStream_t st) { k_drive_red<<<1, 32, 0, st>>>(d); }

void launch_la_x(const Dev& d, LookaheadDev& la, cudaStream_t st) {
    k_la_x<<<dim3((d.m + 1 + 255) / 256, la.K), 256, 0, st>>>(d, la);
}

bool launch_la_price(const Dev& d, LookaheadDev& la, bool bounded, cudaStream_t st) {
    k_la_wp<<<dim3((d.m + 255) / 256, la.K), 256, 0, st>>>(d, la);
    // la.nblk = slot tiles + 1 (the last partial holds the leaving column)
    CUtensorMap tmW, tmA;
    if (la.nblk > 1 &&
        (!encode_2d(&tmW, la.Wp, (uint64_t)d.m, (uint64_t)la.K, (uint64_t)la.ldx * 8, kLC, kLK) ||
         !encode_2d(&tmA, d.A_nb, (uint64_t)d.ld_nb, (uint64_t)d.m, (uint64_t)d.ld_nb * 8, kLN, kLC)))
        return false;
    const dim3 grid(la.nblk - 1, (la.K + kLK - 1) / kLK);
    if (bounded) {
        cudaMemsetAsync(la.fail, 0, sizeof(int), st);
        cudaMemsetAsync(la.npairs, 0, sizeof(int), st);
        k_la_wnorm<<<la.K, 256, 0, st>>>(d, la);
        CUtensorMap tmWs, tmAs;
        if (la.nblk > 1 &&
            (!encode_2d(&tmWs, la.Wp, (uint64_t)d.m, (uint64_t)la.K, (uint64_t)la.ldx * 8, kLC, kLK, true) ||
             !encode_2d(&tmAs, d.A_nb, (uint64_t)d.ld_nb, (uint64_t)d.m, (uint64_t)d.ld_nb * 8, 16, kLC, true)))
            return false;
        if (la.nblk > 1) k_la_screen<false><<<grid, kLThreads, sizeof(LaScreenSmem) + 1024, st>>>(d, la, tmWs, tmAs);
        k_la_leave<<<(la.K + kDC - 1) / kDC, kDT, 0, st>>>(d, la);
        k_la_cands<<<la.K, 256, 0, st>>>(d, la);
        k_la_exact<<<kLaPairs / kDC, kDT, 0, st>>>(d, la);
        k_la_cands_best<<<(la.K + 127) / 128, 128, 0, st>>>(d, la);
        // a bound was unusable: the exact GEMM after all (its CTAs exit at once otherwise)
        if (la.nblk > 1) k_la_gemm_price<<<grid, kLThreads, sizeof(LaPriceSmem), st>>>(d, la, tmW, tmA, 1);
    } else {
        if (la.nblk > 1) k_la_gemm_price<<<grid, kLThreads, sizeof(LaPriceSmem), st>>>(d, la, tmW, tmA, 0);
        k_la_leave<<<(la.K + kDC - 1) / kDC, kDT, 0, st>>>(d, la);
    }
    k_la_price_local<<<la.K, 32, 0, st>>>(d, la);
    return true;
}

void launch_colnorm(const Dev& d, double* out, cudaStream_t st) {
    k_colnorm<<<(d.n_total + 7) / 8, 256, 0, st>>>(d, out);
}

void launch_la_decide(const Dev& d, LookaheadDev& la, const PriceMsg* msgs, int nsrc, cudaStream_t st) {
    k_la_decide<<<(la.K + 127) / 128, 128, 0, st>>>(d, la, msgs, nsrc);
}

bool launch_la_theta(const Dev& d, LookaheadDev& la, cudaStream_t st) {
    CUtensorMap tmT, tmX, tmB;
    if (!encode_2d(&tmT, d.T, (uint64_t)d.mloc, (uint64_t)d.m, (uint64_t)d.ldT * 8, kLT, kLC) ||
        !encode_2d(&tmX, la.X, (uint64_t)d.m, (uint64_t)la.K, (uint64_t)la.ldx * 8, kLC, kLT) ||
        !encode_2d(&tmB, la.Wp, (uint64_t)d.m, (uint64_t)la.K, (uint64_t)la.ldx * 8, kLC, kLT))
        return false;
    k_la_gather<<<dim3((d.m + 255) / 256, la.K), 256, 0, st>>>(d, la);
    k_la_gemm_theta<<<dim3(la.nblk_t, (la.K + kLT - 1) / kLT), 256, sizeof(LaThetaSmem), st>>>(d, la, tmT, tmX,
                                                                                                tmB);
    k_la_own<<<(la.K + kDC - 1) / kDC, kDT, 0, st>>>(d, la);
    k_la_theta_local<<<(la.K + 127) / 128, 128, 0, st>>>(d, la);
    return true;
}

bool launch_la_probe(const Dev& d, LookaheadDev& la, cudaStream_t st) {
    cudaMemsetAsync(la.ok, 0, sizeof(int) * la.K, st);
    k_la_probe_rows<<<1, 1024, 0, st>>>(d, la);
    k_la_probe_gather<<<4 * 148, 256, 0, st>>>(d, la);
    // DMMA screen of the first kLN probe rows for every candidate (split along
    // the reduction to fill the GPU), then certificates from its error bound;
    // the exact rounds below only see the candidates it leaves unproven
    CUtensorMap tmB, tmT;
    if (!encode_2d(&tmB, la.Wp, (uint64_t)d.m, (uint64_t)la.K, (uint64_t)la.ldx * 8, kLC, kLK, true) ||
        !encode_2d(&tmT, la.Tg, (uint64_t)kLaProbe, (uint64_t)d.m, (uint64_t)kLaProbe * 8, 16, kLC, true))
        return false;
    cudaMemsetAsync(la.yacc, 0, sizeof(double) * la.K * kLN, st);
    k_la_probe_norms<<<la.K + kLN, 256, 0, st>>>(d, la);
    const int ktiles = (la.K + kLK - 1) / kLK;
    const int split = std::max(1, std::min((d.m + kLC - 1) / kLC, (2 * 148 + ktiles - 1) / ktiles));
    k_la_screen<true><<<dim3(1, ktiles, split), kLThreads, sizeof(LaScreenSmem) + 1024, st>>>(d, la, tmB, tmT);
    k_la_probe_cert<<<(la.K * kLN + 255) / 256, 256, 0, st>>>(d, la);
    k_la_probe_list<<<1, 1024, 0, st>>>(la);  // la.ncl: candidates the screen left unproven
    k_la_probe_decide<<<1, 1024, 0, st>>>(d, la);
    return true;
}

// The exact rounds for the candidates the screen left unproven (the host runs
// them only when la.ncl > 0): rows [64 r, 64 r + 64) of the probe set per round.
void launch_la_probe_rounds(const Dev& d, LookaheadDev& la, cudaStream_t st) {
    for (int r = 0; r < kLaProbeRounds; ++r) {
        if (r) k_la_probe_list<<<1, 1024, 0, st>>>(la);
        k_la_probe<<<(la.K + kPKc - 1) / kPKc, 128, 0, st>>>(d, la, r);
    }
    k_la_probe_decide<<<1, 1024, 0, st>>>(d, la);
}

void launch_la_score(const Dev& d, LookaheadDev& la, const double* tl, int nsrc, cudaStream_t st) {
    k_la_score<<<(la.K + 127) / 128, 128, 0, st>>>(d, la, tl, nsrc);
}

// fp64 pipe probe: 8 independent DMUL chains and 8 DADD chains per thread
// (no FMA contraction: --fmad=false and explicit __dmul_rn/__dadd_rn).
__global__ void __launch_bounds__(256) k_fp64_probe(double* out, int iters, double a, double b) {
    double m[8], s[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        m[u] = 1.0 + 1e-9 * (threadIdx.x + u);
        s[u] = 1e-3 * (blockIdx.x + u);
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            m[u] = __dmul_rn(m[u], a);
            s[u] = __dadd_rn(s[u], b);
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u) acc += m[u] + s[u];
    if (acc == 12345.678) out[0] = acc;  // keeps the chains alive
}

double fp64_probe_tflops(cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double* out = nullptr;
    if (cudaMalloc(&out, sizeof(double)) != cudaSuccess) return 0.0;
    const int blocks = sms * 8, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k_fp64_probe<<<blocks, threads, 0, st>>>(out, iters, 0.9999999, 1e-12);  // warm-up
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0, st);
        k_fp64_probe<<<blocks, threads, 0, st>>>(out, iters, 0.9999999, 1e-12);
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        best = std::min(best, ms);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    const double flops = 16.0 * iters * (double)blocks * threads;
    return cudaGetLastError() == cudaSuccess && best > 0.f ? flops / (best * 1e-3) / 1e12 : 0.0;
}

void launch_sum_i64(const long long* in, int nsrc, size_t n, long long* out, cudaStream_t st) {
    k_sum_i64<<<(unsigned)std::min<size_t>(1024, (n + 255) / 256), 256, 0, st>>>(in, nsrc, n, out);
}

void launch_min_i32(const int* in, int nsrc, size_t n, int* out, cudaStream_t st) {
    k_min_i32<<<(unsigned)std::min<size_t>(1024, (n + 255) / 256), 256, 0, st>>>(in, nsrc, n, out);
}

}  // namespace lpsg
