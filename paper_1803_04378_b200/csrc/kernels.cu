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
__global__ void k_init_tableau(Dev d, const double* __restrict__ b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < d.m) {
        d.T[(size_t)i * d.ldT + i] = 1.0;
        d.T[(size_t)d.m * d.ldT + i] = b[i];
    }
}

// A_cm[j*m + i] = A_rm[i*n + j]  (tiled transpose through shared memory)
__global__ void k_transpose(const double* __restrict__ A_rm, double* __restrict__ A_cm, int m,
                            int n) {
    __shared__ double tile[32][33];
    const int j0 = blockIdx.x * 32, i0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int i = i0 + k, j = j0 + threadIdx.x;
        if (i < m && j < n) tile[k][threadIdx.x] = A_rm[(size_t)i * n + j];
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int j = j0 + k, i = i0 + threadIdx.x;
        if (i < m && j < n) A_cm[(size_t)j * m + i] = tile[threadIdx.x][k];
    }
}

// A_nb[i*ld_nb + s] = A_rm[i*n + slot2col[s]]
__global__ void k_build_nb(const double* __restrict__ A_rm, Dev d, int n_scan) {
    const int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= n_scan) return;
    const int j = d.slot2col[s];
    for (int i = blockIdx.y; i < d.m; i += gridDim.y)
        d.A_nb[(size_t)i * d.ld_nb + s] = A_rm[(size_t)i * d.n_total + j];
}

// ------------------------------------------------------ rebuild_top_row ---
// solver.cpp:318-329: W_j = sum_i c_B[i] * B^-1[i][j] (ascending i); obj likewise
// over b_bar (column m). One output per lane of warp 0; 32x32 tiles of T are
// staged through shared memory so the column walk stays coalesced.
__global__ void k_rebuild_top(Dev d) {
    __shared__ double tile[32][33];
    __shared__ double cb[32];
    const int j0 = blockIdx.x * 32;
    const int ncols = d.m + 1;
    const double* cost = phase_cost(d, d.ctl->phase);
    double acc = 0.0;
    for (int i0 = 0; i0 < d.m; i0 += 32) {
        __syncthreads();
        for (int k = threadIdx.y; k < 32; k += blockDim.y) {
            const int j = j0 + k, i = i0 + threadIdx.x;
            tile[k][threadIdx.x] = (j < ncols && i < d.m) ? d.T[(size_t)j * d.ldT + i] : 0.0;
        }
        if (threadIdx.y == 0) {
            const int i = i0 + threadIdx.x;
            cb[threadIdx.x] = i < d.m ? cost[d.basic[i]] : 0.0;
        }
        __syncthreads();
        if (threadIdx.y == 0) {
            const int lim = min(32, d.m - i0);
            for (int k = 0; k < lim; ++k) acc = dadd(acc, dmul(cb[k], tile[threadIdx.x][k]));
        }
    }
    if (threadIdx.y == 0) {
        const int j = j0 + threadIdx.x;
        if (j < ncols) d.top[j] = acc;
        if (j == 0) d.top[d.m + 1] = 0.0;
    }
}

// ---------------------------------------------------------------- price ---
// solver.cpp:79-129 (+ the loop-top budget check, solver.cpp:281): one thread
// per nonbasic slot, z = dot(W, a_j) - c_j with ascending i, then a grid-wide
// (max z, min j) reduction finished by the last CTA.
__global__ void __launch_bounds__(256) k_price(Dev d) {
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING) return;
    const bool budget_hit = c->total_iter >= c->budget;
    const int n_scan = c->n_scan;
    const double* cost = phase_cost(d, c->phase);
    const int m = d.m;
    const double* __restrict__ w = d.top;
    double bz = -kInf;
    int bj = INT_MAX;
    if (!budget_hit) {
        const int stride = gridDim.x * blockDim.x;
        for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_scan; s += stride) {
            const double* __restrict__ a = d.A_nb + s;
            double acc = 0.0;
            int i = 0;
            for (; i + 8 <= m; i += 8) {
                double v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = a[(size_t)(i + u) * d.ld_nb];
#pragma unroll
                for (int u = 0; u < 8; ++u) acc = dadd(acc, dmul(w[i + u], v[u]));
            }
            for (; i < m; ++i) acc = dadd(acc, dmul(w[i], a[(size_t)i * d.ld_nb]));
            const int j = d.slot2col[s];
            const double z = dsub(acc, cost[j]);
            if (better(z, j, bz, bj)) { bz = z; bj = j; }
        }
    }
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
        for (int o = 16; o > 0; o >>= 1) {
            const double oz = __shfl_down_sync(0xffffffffu, z, o);
            const int oj = __shfl_down_sync(0xffffffffu, j, o);
            if (better(oz, oj, z, j)) { z = oz; j = oj; }
        }
        if (threadIdx.x == 0) {
            c->ticket_price = 0;
            if (budget_hit) {
                c->status = ST_ITER_LIMIT;
            } else {
                c->q = j == INT_MAX ? -1 : j;
                c->d = j == INT_MAX ? 0.0 : z;
                if (j == INT_MAX || z <= d.opt_tol) c->status = ST_OPTIMAL;
            }
        }
    }
}

// --------------------------------------------------------- update+FTRAN ---
// tiled_engine.cpp:230-266 with tile_kernel's cached mode (79-106) fused with the
// NEXT pivot's compute_direction (solver.cpp:131-136), SURVEY.md Appendix B.
// Thread per row i; columns j ascending: T_ij += (-y_i) * x_j unless that
// product is 0; row r takes x. Then Y_i = sum_j T_new[i][j] * a_q[j] in order.
__global__ void __launch_bounds__(128) k_update(Dev d) {
    Ctl* c = d.ctl;
    const int status = c->status;
    const bool up = c->pending != 0;
    const bool ft = status == ST_RUNNING && !c->no_ftran && c->q >= 0;
    if (!up && !ft) return;
    const int m = d.m;
    const int r = c->upd_r;
    const double* __restrict__ x = d.xrow;
    const double* __restrict__ a = ft ? d.A_cm + (size_t)c->q * m : nullptr;
    const int stride = gridDim.x * blockDim.x;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
        const double yi = d.Y[i];
        const double ny = -yi;
        double acc = 0.0;
        double* __restrict__ col = d.T + i;
        for (int j = 0; j <= m; ++j) {
            double v = col[(size_t)j * d.ldT];
            if (up) {
                if (i == r) {
                    v = x[j];
                    col[(size_t)j * d.ldT] = v;
                } else {
                    const double p = dmul(ny, x[j]);
                    if (p != 0.0) {
                        v = dadd(v, p);
                        col[(size_t)j * d.ldT] = v;
                    }
                }
            }
            if (ft && j < m) acc = dadd(acc, dmul(v, a[j]));
        }
        if (ft) {
            d.Y[i] = acc;
        } else {
            // Reference post-pivot column m+1: row r = 1, others y + (-y)*1 (skip 0).
            if (i == r) d.Y[i] = 1.0;
            else {
                const double p = dmul(ny, x[m + 1]);
                if (p != 0.0) d.Y[i] = dadd(yi, p);
            }
        }
    }
    if (!last_block(&c->ticket_update)) return;
    if (threadIdx.x == 0) {
        c->ticket_update = 0;
        if (up) c->pending = 0;
        if (ft) d.top[m + 1] = c->d;
    }
}

// ---------------------------------------------------------------- ratio ---
// solver.cpp:138-162. One CTA: theta = min over eligible rows of b_bar_i / y_i,
// window = theta + tol * max(1, |theta|), candidates ascending via an ordered
// block compaction. One candidate (or anticycle = none) resolves on device;
// two or more under tabu hand over to the host (ST_TIE).
__global__ void __launch_bounds__(1024) k_ratio(Dev d) {
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
__global__ void __launch_bounds__(1024) k_pivot(Dev d) {
    Ctl* c = d.ctl;
    if (c->status != ST_RUNNING) return;
    const int m = d.m;
    const int r = c->r, q = c->q;
    const double yr = d.Y[r];
    if (fabs(yr) <= d.pivot_tol) {
        if (threadIdx.x == 0) c->status = ST_PIVOT_ERR;
        return;
    }
    const double dk = d.top[m + 1];
    const double ndk = -dk;
    for (int j = threadIdx.x; j <= m; j += blockDim.x) {
        const double xj = ddiv(d.T[(size_t)j * d.ldT + r], yr);
        d.xrow[j] = xj;
        const double p = dmul(ndk, xj);
        if (p != 0.0) d.top[j] = dadd(d.top[j], p);
    }
    if (threadIdx.x == 0) {
        const double xl = ddiv(yr, yr);
        d.xrow[m + 1] = xl;
        const double p = dmul(ndk, xl);
        if (p != 0.0) d.top[m + 1] = dadd(dk, p);
    }
    // nonbasic slot maintenance
    const int p_leave = d.basic[r];
    const int s_q = d.col2slot[q];
    const int n_scan = c->n_scan;
    int dst = -1, src_col = -1;
    if (p_leave < d.n_total) {
        dst = s_q >= 0 ? s_q : n_scan;  // reuse q's slot, or append
        src_col = p_leave;
    } else if (s_q >= 0 && s_q != n_scan - 1) {
        dst = s_q;                      // artificial leaves: move the last slot in
        src_col = d.slot2col[n_scan - 1];
    }
    if (dst >= 0) {
        const double* __restrict__ src = d.A_cm + (size_t)src_col * m;
        for (int i = threadIdx.x; i < m; i += blockDim.x) d.A_nb[(size_t)i * d.ld_nb + dst] = src[i];
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int ns = n_scan;
        if (p_leave < d.n_total) {
            if (s_q < 0) ++ns;
            d.slot2col[dst] = p_leave;
            d.col2slot[p_leave] = dst;
        } else if (s_q >= 0) {
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
        const int li = c->log_len;
        if (li < d.log_cap) {
            LogEntry e;
            e.iteration = c->total_iter;
            e.phase = c->phase;
            e.row = r;
            e.leaving = p_leave;
            e.entering = q;
            e.objective = d.top[m];
            d.log[li] = e;
        }
        c->log_len = li + 1;
        c->pending = 1;
        c->upd_r = r;
        c->upd_q = q;
    }
}

// --------------------------------------------------------- drive-out scan ---
// solver.cpp:295-316: first j < n_total, nonbasic, with |dot(B^-1 row i, a_j)| >
// pivot_tol (ascending i in the dot), as a min-j reduction; the last CTA also
// computes the entering reduced cost dot(W, a_j) - c_j.
__global__ void k_gather_row(Dev d, int i, double* out) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k <= d.m; k += gridDim.x * blockDim.x)
        out[k] = d.T[(size_t)k * d.ldT + i];
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
    if (!last_block(&c->ticket_misc)) return;
    if (threadIdx.x == 0) {
        c->ticket_misc = 0;
        const int j = ((volatile int*)&c->found)[0];
        if (j == INT_MAX) {
            c->found = -1;
        } else {
            const double* cost = phase_cost(d, c->phase);
            const double* __restrict__ a = d.A_cm + (size_t)j * m;
            double acc = 0.0;
            for (int i = 0; i < m; ++i) acc = dadd(acc, dmul(d.top[i], a[i]));
            c->found_red = dsub(acc, cost[j]);
        }
    }
}

// ------------------------------------------------------------ lookahead ---
// solver.cpp:164-213, batched over K candidate rows without materialising the
// K pivoted tableaus: (1) X_k = T_r / piv, W'_k = W - d*X_k; (2) pricing of
// W'_k over the nonbasic set with q removed and basic[r_k] added; (3) y'_ik =
// sum_j (T_ij - y_i X_kj) a_best[j] (ascending j) and theta'_k; (4) score.
__global__ void k_la_prep(Dev d, LookaheadDev la) {
    const int k = blockIdx.y;
    const int r = la.rows[k];
    const double piv = d.Y[r];
    const double dk = d.top[d.m + 1];
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j <= d.m; j += gridDim.x * blockDim.x) {
        const double xj = ddiv(d.T[(size_t)j * d.ldT + r], piv);
        la.X[(size_t)k * la.ldx + j] = xj;
        if (j < d.m) {
            const double w = d.top[j];
            la.Wp[(size_t)k * la.ldx + j] = dk == 0.0 ? w : dsub(w, dmul(dk, xj));
        }
    }
}

__global__ void __launch_bounds__(256) k_la_price(Dev d, LookaheadDev la) {
    const int k = blockIdx.y;
    const int n_scan = d.ctl->n_scan;
    const double* cost = phase_cost(d, d.ctl->phase);
    const double* __restrict__ w = la.Wp + (size_t)k * la.ldx;
    const int m = d.m;
    double bz = -kInf;
    int bj = INT_MAX;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < n_scan; s += gridDim.x * blockDim.x) {
        const int j = d.slot2col[s];
        if (j == la.q) continue;
        const double* __restrict__ a = d.A_nb + s;
        double acc = 0.0;
        for (int i = 0; i < m; ++i) acc = dadd(acc, dmul(w[i], a[(size_t)i * d.ld_nb]));
        const double z = dsub(acc, cost[j]);
        if (better(z, j, bz, bj)) { bz = z; bj = j; }
    }
    // the leaving variable becomes nonbasic (solver.cpp:186-188)
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const int p = d.basic[la.rows[k]];
        if (p < d.n_total && p != la.q) {
            const double* __restrict__ a = d.A_cm + (size_t)p * m;
            double acc = 0.0;
            for (int i = 0; i < m; ++i) acc = dadd(acc, dmul(w[i], a[i]));
            const double z = dsub(acc, cost[p]);
            if (better(z, p, bz, bj)) { bz = z; bj = p; }
        }
    }
    block_argmax(bz, bj);
    if (threadIdx.x == 0) {
        la.part_z[(size_t)k * la.nblk + blockIdx.x] = bz;
        la.part_j[(size_t)k * la.nblk + blockIdx.x] = bj;
    }
}

__global__ void k_la_price_final(Dev d, LookaheadDev la) {
    const int k = blockIdx.x;
    if (threadIdx.x >= 32) return;
    double z = -kInf;
    int j = INT_MAX;
    for (int b = threadIdx.x; b < la.nblk; b += 32) {
        const double oz = la.part_z[(size_t)k * la.nblk + b];
        const int oj = la.part_j[(size_t)k * la.nblk + b];
        if (better(oz, oj, z, j)) { z = oz; j = oj; }
    }
    for (int o = 16; o > 0; o >>= 1) {
        const double oz = __shfl_down_sync(0xffffffffu, z, o);
        const int oj = __shfl_down_sync(0xffffffffu, j, o);
        if (better(oz, oj, z, j)) { z = oz; j = oj; }
    }
    if (threadIdx.x == 0) {
        la.bz[k] = z;
        la.bj[k] = (j == INT_MAX || z <= d.opt_tol) ? -1 : j;
    }
}

__global__ void __launch_bounds__(128) k_la_theta(Dev d, LookaheadDev la) {
    const int k = blockIdx.y;
    const int bj = la.bj[k];
    if (bj < 0) return;
    const int m = d.m;
    const int rk = la.rows[k];
    const double* __restrict__ X = la.X + (size_t)k * la.ldx;
    const double* __restrict__ a = d.A_cm + (size_t)bj * m;
    double theta = kInf;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < m; i += gridDim.x * blockDim.x) {
        if (d.frozen[i]) continue;
        const double yi = d.Y[i];
        const double* __restrict__ col = d.T + i;
        double acc = 0.0;
        double bb;
        if (i == rk) {
            for (int j = 0; j < m; ++j) acc = dadd(acc, dmul(X[j], a[j]));
            bb = X[m];
        } else if (yi == 0.0) {
            for (int j = 0; j < m; ++j) acc = dadd(acc, dmul(col[(size_t)j * d.ldT], a[j]));
            bb = col[(size_t)m * d.ldT];
        } else {
            for (int j = 0; j < m; ++j)
                acc = dadd(acc, dmul(dsub(col[(size_t)j * d.ldT], dmul(yi, X[j])), a[j]));
            bb = dsub(col[(size_t)m * d.ldT], dmul(yi, X[m]));
        }
        if (acc <= d.pivot_tol) continue;
        theta = min_keep(theta, ddiv(bb, acc));
    }
    theta = block_min(theta);
    if (threadIdx.x == 0) la.part_t[(size_t)k * la.nblk + blockIdx.x] = theta;
}

__global__ void k_la_final(Dev d, LookaheadDev la) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= la.K) return;
    if (la.bj[k] < 0) { la.score[k] = 0.0; return; }
    double t = kInf;
    for (int b = 0; b < la.nblk; ++b) t = min_keep(t, la.part_t[(size_t)k * la.nblk + b]);
    la.theta[k] = t;
    la.score[k] = isinf(t) ? kInf : dmul(la.bz[k], t);
}

}  // namespace

// ------------------------------------------------------------- launchers ---
void launch_init_tableau(const Dev& d, const double* b, cudaStream_t st) {
    k_init_tableau<<<(d.m + 255) / 256, 256, 0, st>>>(d, b);
}

void launch_transpose(const double* A_rm, double* A_cm, int m, int n, cudaStream_t st) {
    dim3 grid((n + 31) / 32, (m + 31) / 32);
    k_transpose<<<grid, dim3(32, 8), 0, st>>>(A_rm, A_cm, m, n);
}

void launch_build_nb_from(const Dev& d, const double* A_rm, int n_scan, cudaStream_t st) {
    if (n_scan <= 0) return;
    dim3 grid((n_scan + 255) / 256, (unsigned)std::min(d.m, 1024));
    k_build_nb<<<grid, 256, 0, st>>>(A_rm, d, n_scan);
}

void launch_rebuild_top(const Dev& d, cudaStream_t st) {
    k_rebuild_top<<<(d.m + 1 + 31) / 32, dim3(32, 8), 0, st>>>(d);
}

void launch_price(const Dev& d, cudaStream_t st) { k_price<<<d.price_grid, 256, 0, st>>>(d); }

void launch_update(const Dev& d, cudaStream_t st) { k_update<<<d.update_grid, 128, 0, st>>>(d); }

void launch_ratio(const Dev& d, cudaStream_t st) { k_ratio<<<1, 1024, 0, st>>>(d); }

void launch_pivot(const Dev& d, cudaStream_t st) { k_pivot<<<1, 1024, 0, st>>>(d); }

void launch_gather_row(const Dev& d, int i, double* out, cudaStream_t st) {
    k_gather_row<<<(d.m + 1 + 255) / 256, 256, 0, st>>>(d, i, out);
}

void launch_drive_scan(const Dev& d, int row, double* scratch, cudaStream_t st) {
    launch_gather_row(d, row, scratch, st);
    k_drive_scan<<<d.price_grid, 256, 0, st>>>(d, scratch);
}

void launch_lookahead(const Dev& d, LookaheadDev& la, cudaStream_t st) {
    k_la_prep<<<dim3((d.m + 1 + 255) / 256, la.K), 256, 0, st>>>(d, la);
    k_la_price<<<dim3(la.nblk, la.K), 256, 0, st>>>(d, la);
    k_la_price_final<<<la.K, 32, 0, st>>>(d, la);
    k_la_theta<<<dim3(la.nblk, la.K), 128, 0, st>>>(d, la);
    k_la_final<<<(la.K + 127) / 128, 128, 0, st>>>(d, la);
}

}  // namespace lpsg
