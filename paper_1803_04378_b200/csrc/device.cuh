// device.cuh — device-side state and kernel launchers of the lpsg solver.
//
// HBM layout (SURVEY.md §7 "Kernel plan"):
//   T      column-major (m+1) columns x ldT rows: columns 0..m-1 = B^-1, column m = b_bar.
//          Element (i, j) of the reference's tableau row i+1 (solver.hpp:71-76) is
//          T[j*ldT + i]. Row-owner threads therefore read coalesced along i.
//   top    row 0 of the tableau: [W (m) | obj | d]  (m+2 doubles)
//   Y      the pivot column y (tableau column m+1, rows 1..m)
//   xrow   the pivot row divided by y_rk (m+2 doubles)
//   A_cm   column-major copy of A (column j contiguous, m doubles) — FTRAN operand a_q
//   A_nb   row-major m x ld_nb "nonbasic pricing matrix": slot s holds column slot2col[s];
//          slots [0, n_scan) are exactly the nonbasic non-artificial columns
//   ctl    control block; every per-pivot decision lives on the device so pivot
//          batches run without host round trips.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdint>
#include <cstdlib>

#include "peer.cuh"

// Performance experiments (memory-only / compute-only rates, kernel-shape
// overrides). Their results are NOT valid solves, so they exist only in a build
// compiled with -DLPSG_EXPERIMENTS (tools/, never the default library): there
// LPSG_XP reads the knob bits of lpsg_config.reserved[2] and xp_env the LPSG_*
// shape variables; in the default build both fold to constants.
#ifdef LPSG_EXPERIMENTS
#define LPSG_XP(d, bits) ((((d).dbg) & (bits)) != 0)
#else
#define LPSG_XP(d, bits) false
#endif

namespace lpsg {

constexpr int kLookaheadExactBit = 16;  // lpsg_config.reserved[2]: see Dev::la_exact
// lpsg_config.reserved[2]: select_leaving's bounded selection on every tie of
// >= 2 survivors (verification) / never (A/B); default from 16 survivors up
constexpr int kLookaheadBoundAllBit = 32;
constexpr int kLookaheadBoundOffBit = 64;

inline const char* xp_env(const char* name) {
#ifdef LPSG_EXPERIMENTS
    return getenv(name);
#else
    (void)name;
    return nullptr;
#endif
}

enum CtlStatus : int {
    ST_RUNNING = 0,
    ST_OPTIMAL = 1,
    ST_UNBOUNDED = 2,
    ST_TIE = 3,          // ratio test tied under tabu: host runs select_leaving
    ST_ITER_LIMIT = 4,
    ST_PIVOT_ERR = 5,    // |y_rk| <= pivot_tol
    ST_HOLD = 6,         // step API / phase boundary: kernels idle
    ST_OVERFLOW = 7      // sharded ratio test: a shard's local candidate list exceeds
                         // kRatioMsgCap; the host gathers the full lists
};

// Sharded solves (world > 1): fixed-size messages exchanged by
// all-gather after the local pricing and ratio passes.
constexpr int kRatioMsgCap = 30;
struct PriceMsg {
    double z;
    int j;
    int pad;
};
struct RatioMsg {
    double theta;   // local min ratio (valid when any)
    int any;        // any eligible local row
    int n;          // local candidates within the LOCAL window
    int rows[kRatioMsgCap];
    double ratios[kRatioMsgCap];
};
static_assert(sizeof(RatioMsg) % 8 == 0, "RatioMsg is moved as 8-byte words");
static_assert(sizeof(PriceMsg) == 16, "PriceMsg is moved as one 16-byte word");

struct LogEntry {
    long long iteration;
    int phase;
    int row;
    int leaving;
    int entering;
    double objective;
};

struct Ctl {
    int status;
    int pending;       // a pivot was committed; the tableau update is outstanding
    int q;             // entering column (last pricing result)
    int r;             // leaving row (ratio test / host)
    double d;          // reduced cost of q
    double theta;
    int ncand;
    int n_scan;        // active pricing slots
    long long total_iter;
    long long budget;
    int phase;
    int log_len;
    int no_ftran;      // update without the fused FTRAN (drive-out, step API)
    int upd_r;         // row of the pending update
    int upd_q;         // column entering in the pending update
    int any_ratio;
    unsigned int ticket_price;
    unsigned int ticket_update;
    unsigned int ticket_misc;
    unsigned int ticket_x;     // k_pivot_row's last CTA (fused P2P signal)
    int found;         // drive-out scan result
    double found_red;
    int no_ratio;      // FTRAN without the fused ratio test (drive-out, step API)
    int x_owner;       // sharded: this shard owns the current pivot row (k_pivot_row)
    unsigned long long work[4];  // launches that did their work: price, update, pivot (profiling)
};

struct Dev {
    int m, n_total, n_work;
    // sharding. Unsharded: world == 1, row0 = 0, mloc = m, col0 = 0, col1 = n_total.
    int world, rank;
    int sharded;           // 1: a communicator is attached (even with world == 1)
    int row0, mloc;        // this shard's rows of T = [B^-1 | b_bar] and of Y
    int col0, col1;        // this shard's pricing columns (original index range)
    double* xbuf;          // sharded: pivot row exchange (m+3 slots), in the transport's symmetric heap
    int xbuf_zero;         // transport sums int64 bit patterns: non-owners zero-fill xbuf
    PriceMsg* pmsg;        // world > 1: [0] local result, [1..world] gathered
    RatioMsg* rmsg;        // world > 1: [0] local result, [1..world] gathered
    // P2P transport, fused exchanges: the producing kernel's last CTA stores its
    // message into every peer's mailbox and raises the flags; the consumer
    // (k_price_final / k_ratio_final) waits and reads its own mailbox.
    int fused;
    PeerArgs px_price, px_ratio;
    int fused_x;           // P2P: k_pivot_row stores the pivot row into the peers' xbuf
    PeerArgs px_x;
    size_t xbuf_off;       // xbuf's offset in the symmetric heap
    double* cand_ratio;    // ratios of the candidates in cand (same order)
    long long ldT;
    long long ld_nb;
    double* T;
    double* top;
    double* Y;
    double* xrow;
    const double* A_cm;
    double* A_nb;
    int* slot2col;
    int* col2slot;
    int* basic;
    unsigned char* frozen;
    const double* cost_p1;
    const double* cost_true;
    Ctl* ctl;
    int* cand;
    double* pz;
    int* pj;
    LogEntry* log;
    int log_cap;
    int num_sms;
    double opt_tol, pivot_tol, feas_tol, ratio_tie_tol;
    int anticycle;
    int price_grid;
    int update_grid;
    int pivot_grid;
    // fused ratio test partials (per update CTA): local theta, candidate count
    // (-1: no eligible row), candidates (row, ratio) in row order
    double* rc_theta;
    int* rc_cnt;
    int* rc_row;
    double* rc_ratio;
    long long ld_cm;       // column pitch of A_cm (even, 16-byte aligned columns)
    // launch geometry of the streaming kernels (configure_kernels)
    int upd_h, upd_C, upd_S, upd_U, upd_smem, upd_threads;
    const CUtensorMap* tm_T;   // 2D TMA descriptor of T, box {h rows, C columns}
    const CUtensorMap* tm_nb;  // 2D TMA descriptors of A_nb, box {wbx slots, price_rows(wbx) rows}
    int price_nwc, price_S, price_smem, price_threads;
    int price_spt;             // slots per consumer thread: 1 (one chain per lane) or 2 (pairs)
    int price_pf;              // A_nb stages k_price prefetches into L2 before its PDL wait
    int dbg;               // perf-experiment knobs (cfg.reserved[2] minus bit 4); read only
                           // through LPSG_XP, i.e. only in a -DLPSG_EXPERIMENTS build
    int la_exact;          // lookahead theta' keeps the y_i == 0 select (cfg.reserved[2] bit 4):
                           // result-identical verification mode
    int fuse_pivot;        // single GPU, fused schedule: k_update's last CTA also runs pivot_update
                           // of the row its ratio test chose (no k_pivot launch on that path)
    int keep_pending;      // Case 2 (tiled): this k_update launch is not the last partition of the
                           // pass, so its last CTA leaves ctl.pending set for the next one
    int naive;             // KernelMode::naive (tiled_engine.cpp:61-77): every element is stored,
                           // no `temp != 0` skip (only zero signs differ from cached mode)
    int pdl;               // launch the pivot chain with programmatic dependent launch
    int upd_tma_store;     // k_update writes tiles back with TMA stores (else per-warp STG)
    int l2_hint;           // streaming TMA traffic carries an L2 evict-first hint
    size_t price_stage_bytes;
};

// Pricing geometry for n_scan active slots over G CTAs. The slots are dealt
// out in units of 8 so every CTA gets floor or ceil(units / G) of them (CTA b
// owns [s0, s0 + own)). The CTA loads nb TMA boxes of wbx <= 256 slots x R rows.
struct PriceGeom {
    int w, nb, wbx, R, s0, own;
};
__host__ __device__ inline int price_rows(int wbx) {
    int R = (48 * 1024) / (8 * wbx);
    R &= ~15;
    return R < 16 ? 16 : (R > 256 ? 256 : R);
}
__host__ __device__ inline PriceGeom price_geom(int n_scan, int G, int b = 0) {
    const int units = (n_scan + 7) / 8;
    const int q = units / G, rem = units % G;
    const int wu = q + (b < rem ? 1 : 0);
    PriceGeom g;
    g.own = 8 * wu;
    g.s0 = 8 * (b * q + (b < rem ? b : rem));
    int w = g.own < 8 ? 8 : g.own;
    const int nb = (w + 255) / 256;
    int wbx = (w + nb - 1) / nb;
    wbx = (wbx + 7) & ~7;
    g.nb = nb;
    g.wbx = wbx;
    g.w = nb * wbx;
    g.R = price_rows(wbx);
    return g;
}

// Lookahead (solver.cpp:164-213) batch buffers.
struct LookaheadDev {
    int K;            // candidates in this batch
    int ldx;          // row pitch of X / Wp (>= m+1)
    const int* rows;  // K candidate rows
    double* X;        // K x ldx : candidate pivot rows divided by piv (B^-1 part + b_bar)
    double* Wp;       // K x ldx : W' = W - d * X
    double* Abest;    // K x m   : a_{best_k}
    double* bz;       // K best z
    int* bj;          // K best column
    double* theta;    // K
    double* score;    // K
    double* part_z;   // partials
    int* part_j;
    double* part_t;
    PriceMsg* pm;     // K local (z, j) per candidate; world > 1: gathered into pm_all
    PriceMsg* pm_all; // world x K
    double* tl;       // K local theta'
    double* own_t;    // K theta' ratio of each candidate's own pivot row (k_la_own)
    double* tl_all;   // world x K
    int nblk;         // pricing partials per candidate (64-slot tiles + 1 leaving column)
    int nblk_t;       // theta' partials per candidate (64-row tiles)
    int q;            // entering column
    double d;         // entering reduced cost
    int* nonfinite;   // set by k_la_wp when some X_kj (j < m) is inf/NaN (host zeroes it)
    int x_owned_only; // Case 2: k_la_x writes only the rows of the resident partition (runs once
                      // per partition) instead of zero-filling the others for a sum exchange
    // bounded selection (k_la_probe*, select_leaving only): probe rows, their T
    // columns gathered [j][r], per-candidate certificates, the verdict
    int* prow;        // kLaProbe probe rows (ascending)
    int* nprow;       // how many
    double* Tg;       // m x kLaProbe
    int* ok;          // K: some probe row proves theta'_k <= 0
    int* clist;       // candidates still unproven (ascending), for the next probe round
    int* ncl;         // how many
    int* first;       // 1: the first candidate is provably chosen
    double* yacc;     // K x 128: the probe screen's y~ partial sums (atomic)
    double* pxb;      // K: X_k . B_k
    double* pxn;      // K: ||X_k||
    double* pbn;      // K: ||B_k||
    double* ptn;      // 128: ||T_i|| of the screened probe rows
    // bounded pricing (k_la_gemm_price<true> + k_la_cands/k_la_exact): z~ by
    // any-order DFMA with a rigorous error bound, exact chains only where the
    // bound cannot exclude the argmax
    const double* anorm;  // n_total: ||a_j||_2 of the original columns
    double* wnorm;    // K: ||W'_k||_2
    int* tl_s;        // K x tiles x kLaTile: slots whose interval reaches the tile's bound
    double* tl_z;     // their z~
    int* tl_n;        // K x tiles: how many
    double* part_L;   // K x nblk: per-tile max lower bound
    int* cj;          // K x kLaCand: columns whose interval reaches the best lower bound
    int* cn;          // K: how many (> kLaCand: overflow -> exact GEMM)
    double* cz;       // K x kLaCand: their exact z
    int* pairs;       // flattened k * kLaCand + e, for the exact chains
    int* npairs;
    int* fail;        // 1: some bound unusable (non-finite, list overflow): run the exact GEMM
};
constexpr int kLaCand = 8;         // exact candidates per lookahead candidate
constexpr int kLaTile = 4;         // screen survivors kept per (candidate, 128-slot tile)
constexpr int kLaPairs = 1 << 14;  // exact chains per batch
constexpr int kLaProbeRound = 64;                     // probe rows per round
constexpr int kLaProbeRounds = 6;                     // rounds before falling back to full scoring
constexpr int kLaProbe = kLaProbeRound * kLaProbeRounds;  // probe rows gathered

// ---- launchers (kernels.cu) -------------------------------------------------
void configure_kernels(Dev& d);
bool create_tensor_maps(Dev& d, CUtensorMap** dev_maps, int* count);
void launch_init_tableau(const Dev& d, const double* b, cudaStream_t st);
// rebuild_top_row over this shard's rows, continuing the ascending-i chain
// from `init` (nullptr: start at 0.0), into `out` (d.top: also zero the d slot).
void launch_rebuild_top(const Dev& d, const double* init, double* out, cudaStream_t st);
void launch_price(const Dev& d, cudaStream_t st);
void launch_price_final(const Dev& d, cudaStream_t st);       // world > 1
void launch_ratio_final(const Dev& d, cudaStream_t st);       // world > 1
void launch_pivot_row(const Dev& d, cudaStream_t st);         // world > 1
void launch_update(const Dev& d, cudaStream_t st);
void launch_ratio(const Dev& d, cudaStream_t st);
void launch_pivot(const Dev& d, cudaStream_t st);
// also sets *nonfinite (device int) to 1 when some A entry is inf/NaN
void launch_transpose(const double* A_rm, double* A_cm, int m, int n, long long ld, int* nonfinite,
                      cudaStream_t st);
// A_nb (this shard's n_scan slots, slot2col set) from d.A_cm
void launch_build_nb_from_cm(const Dev& d, int n_scan, cudaStream_t st);
// drive-out: scan this shard's slots against g = B^-1 row (m doubles) -> ctl.found
// (local min j); then, after the cross-shard min, the entering reduced cost.
void launch_drive_scan(const Dev& d, const double* g, cudaStream_t st);
void launch_drive_red(const Dev& d, cudaStream_t st);
// lookahead phases; world > 1 exchanges between them (solver.cu)
double fp64_probe_tflops(cudaStream_t st);  // k_fp64_probe, best of 5
void launch_la_x(const Dev& d, LookaheadDev& la, cudaStream_t st);
// false: TMA descriptor encode failed. bounded: the DFMA screen + exact chains
// (la.anorm ... la.fail set); else the exact GEMM over every slot.
bool launch_la_price(const Dev& d, LookaheadDev& la, bool bounded, cudaStream_t st);
void launch_colnorm(const Dev& d, double* out, cudaStream_t st);  // ||a_j||_2, j < n_total
void launch_la_decide(const Dev& d, LookaheadDev& la, const PriceMsg* msgs, int nsrc, cudaStream_t st);
bool launch_la_theta(const Dev& d, LookaheadDev& la, cudaStream_t st);
// select_leaving's bounded path (unsharded, in-core): la.first = 1 when the
// first candidate provably wins ("bounded selection")
bool launch_la_probe(const Dev& d, LookaheadDev& la, cudaStream_t st);
void launch_la_probe_rounds(const Dev& d, LookaheadDev& la, cudaStream_t st);  // when la.ncl > 0
void launch_la_score(const Dev& d, LookaheadDev& la, const double* tl, int nsrc, cudaStream_t st);
// in-process shard exchange helpers (LocalComm): out[k] = sum_g in[g*n + k] / min_g
void launch_sum_i64(const long long* in, int nsrc, size_t n, long long* out, cudaStream_t st);
void launch_min_i32(const int* in, int nsrc, size_t n, int* out, cudaStream_t st);
void launch_gather_row(const Dev& d, int i, double* out, cudaStream_t st);
// Case 2 (tiled): the ratio test over P partitions' messages (msgs[p], the
// partition's full candidate list at d.cand + row0[p]) -> ctl (r / ST_TIE /
// ST_UNBOUNDED), ascending rows in d.cand
void launch_ratio_merge_parts(const Dev& d, const RatioMsg* msgs, const int* row0, int P, cudaStream_t st);
// opt-in reinversion (reinvert.cu): column-major C = alpha A B + D (D == nullptr: + I)
void launch_dgemm_nn(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb, double* C,
                     long long ldc, double alpha, const double* D, long long ldd, cudaStream_t st);
void launch_form_basis(const Dev& d, const int* art_row, double* Bm, long long ld, cudaStream_t st);
void launch_absmax(const double* R, int m, long long ld, unsigned long long* out, cudaStream_t st);
void launch_gemv_bbar(const Dev& d, const double* b, cudaStream_t st);
void launch_probe_residual(int m, const double* Bm, long long ldb, const double* X, long long ldx, double* u,
                           double* w, unsigned long long* out, cudaStream_t st);

}  // namespace lpsg
