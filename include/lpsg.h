/* include/lpsg.h — C ABI of the B200-native dense revised simplex ("lpsg").
 *
 * This is the drop-in boundary for the reference's solver entry points
 * (/root/reference/proj/include/lps/solver.hpp). Plain pointers and sizes only;
 * no torch or C++ types cross it. Every function returns an lpsg_status code
 * (LPSG_OK on success) and leaves a thread-local message for lpsg_last_error().
 * No exceptions cross the ABI; the C++ shim (include/lpsg.hpp) rethrows them as
 * the reference's error types (errors.hpp:9-11, 58-64).
 *
 * Implementation: paper_1803_04378_b200/csrc/ (C++ host driver + sm_100a CUDA
 * kernels). There is no CPU fallback: on a machine without a usable B200 every
 * solver entry point fails with LPSG_CUDA_ERROR.
 */
#ifndef LPSG_H
#define LPSG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes. Outcomes of a solve are lpsg_solve_status, not errors. */
typedef enum {
    LPSG_OK = 0,
    LPSG_PIVOT_TOO_SMALL = 1, /* lps::PivotTooSmall (errors.hpp:58-60, solver.cpp:241-244) */
    LPSG_CUDA_ERROR = 2,
    LPSG_OUT_OF_MEMORY = 3,
    LPSG_INVALID_ARGUMENT = 4,
    LPSG_NCCL_ERROR = 5,
    LPSG_EMPTY_PROBLEM = 6,   /* lps::DegenerateSpec / EmptyProblem (errors.hpp:17-19,66-68) */
    LPSG_BUDGET_TOO_SMALL = 7 /* lps::BudgetTooSmall (tiled_engine.cpp:43-47) */
} lpsg_status;

/* lps::SolveStatus (solver.hpp:14), same order. */
typedef enum {
    LPSG_OPTIMAL = 0,
    LPSG_UNBOUNDED = 1,
    LPSG_INFEASIBLE = 2,
    LPSG_ITERATION_LIMIT = 3
} lpsg_solve_status;

/* lps::ColKind (lp_model.hpp:22). */
enum { LPSG_COL_STRUCTURAL = 0, LPSG_COL_SLACK = 1 };

/* lps::StandardFormLP (lp_model.hpp:49-60): Min c.x s.t. A x = b, b >= 0, x >= 0.
 * A is row-major m x n_total. Caller-owned; copied to the device by lpsg_create. */
typedef struct {
    int m;
    int n_total;
    const double* A;
    const double* b;
    const double* c;
    const uint8_t* col_kind;
} lpsg_problem;

/* lps::SolverConfig (solver.hpp:34-45) plus device placement. `kernel` is
 * honoured: KernelMode::cached (0, the `temp != 0` store skip) or naive (1,
 * every element stored; tiled_engine.cpp:56-111) -- they differ only in the
 * signs of zeros. `workers` selects CPU threading in the reference and is
 * ignored (its results are worker-independent, solver.cpp:99-121). */
typedef struct {
    double opt_tol;        /* 1e-7 */
    double pivot_tol;      /* 1e-9 */
    double feas_tol;       /* 1e-7 */
    double ratio_tie_tol;  /* 1e-9, relative */
    long max_iter;         /* 0 = 50 * (m + n_work)  (solver.cpp:64) */
    int anticycle;         /* 0 tabu, 1 none (solver.hpp:16) */
    int kernel;            /* 0 cached, 1 naive; anything else is LPSG_INVALID_ARGUMENT */
    int workers;           /* ignored */
    int device;            /* CUDA device ordinal, default 0 */
    int batch;             /* pivots enqueued per host check (0 = auto) */
    int reserved[6];       /* verification switches, result-identical to 0:
                              [0] bit 0: standalone ratio kernel instead of the
                                  fused epilogue;
                              [1] bit 0: attach the NCCL exchange path even for
                                  world_size 1 (exercises NCCL on one GPU);
                              [2] bit 4: lookahead theta' keeps the y_i == 0 select;
                                  bit 5: select_leaving tries the bounded selection
                                  on every tie of >= 2 survivors (default: >= 16);
                                  bit 6: never (every tie scored in full).
                              Other bits of [2] are read only by the
                              -DLPSG_EXPERIMENTS build (device.cuh). */
    /* Sharded solve over NCCL, one process (or thread) per GPU:
     * world_size > 1 makes this handle shard `rank`; every rank passes the same
     * problem, config and nccl_id (from lpsg_nccl_unique_id on rank 0) and must
     * make the same sequence of calls. world_size <= 1: single GPU. */
    int world_size;
    int rank;
    unsigned char nccl_id[128];
    /* Alternative transport: a connected P2P heap (lpsg_peer_create/connect).
     * When set, the shards exchange through device-initiated NVLink stores and
     * flags instead of NCCL (world_size/rank come from the heap). */
    struct lpsg_peer* peer;
    /* Opt-in periodic reinversion (north_star item 5; NOT the reference's
     * arithmetic, so results are no longer bit-identical to it): every
     * `reinvert_every` pivots, and before accepting an optimal or unbounded
     * phase outcome, B^-1 is rebuilt on the device from the basis columns of
     * the original A (one Newton-Schulz step from the current inverse, DFMA
     * GEMMs: csrc/reinvert.cu), then b_bar = B^-1 b and W = c_B^T B^-1.
     * 0 = off (default: the reference's drifting explicit inverse, bit for
     * bit). Single GPU only. */
    long reinvert_every;
    /* lps::SolverConfig::memory_budget (solver.hpp:41, tiled_engine.cpp:29-54):
     * device bytes for the (m+1) x (m+2) tableau. When the tableau does not fit
     * (or, with 0 = unlimited, when it does not fit the GPU's free HBM beside A)
     * the solve runs Case 2 ("tiled", report.case_used = 1): the rows of
     * [B^-1 | b_bar] live in page-locked host memory in the reference's row
     * partitions and stream through one device slab per pivot, resident
     * partition first (tiled_engine.cpp:246-263); results are bit-identical to
     * the in-core solve. A budget below two tableau rows is
     * LPSG_BUDGET_TOO_SMALL (lps::BudgetTooSmall, tiled_engine.cpp:44). Case 2
     * is single-GPU only and has no step API or reinversion. */
    unsigned long long memory_budget;
} lpsg_config;

/* lps::SolveReport (solver.hpp:47-57); x is fetched with lpsg_get_x. */
typedef struct {
    int status;             /* lpsg_solve_status */
    double objective;       /* tableau T[0][m]; -inf unbounded, NaN infeasible (solver.cpp:366-377) */
    long iterations_phase1;
    long iterations_phase2;
    double total_seconds;   /* solve() only, like solver.cpp:332,363 */
    double tpi_seconds;     /* total / max(1, iterations) (solver.cpp:387-388) */
    int case_used;          /* TileCase (tiled_engine.hpp:24): 0 in-core, 1 tiled (Case 2) */
} lpsg_report;

/* One pivot, as the reference's IterationObserver sees it (solver.hpp:21-32,
 * solver.cpp:264-275): phase, cumulative iteration, the basis row that
 * changed, the variables that left / entered, and T[0][m] after the pivot. */
typedef struct {
    long iteration;
    int phase;
    int row;
    int leaving;
    int entering;
    double objective;
} lpsg_trace;

typedef void (*lpsg_observer)(const lpsg_trace* pivot, void* user);

/* lps::MemoryCounters (tiled_engine.hpp:56-74) counterpart. The reference
 * counts the accesses of its simulated device arena; lpsg reports the real
 * traffic: host<->device bytes the library moved, kernel launches, and the
 * ALGORITHMIC HBM bytes of the pivots done (what the reference's steps must
 * touch: pricing reads A's nonbasic columns and W, the update
 * reads and writes [B^-1 | b_bar] once, the pivot row). */
typedef struct {
    uint64_t device_read_bytes;
    uint64_t device_write_bytes;
    uint64_t h2d_bytes;
    uint64_t d2h_bytes;
    uint64_t kernel_launches;
} lpsg_memory;

/* lps::IterationView (solver.hpp:21-30), handed to a view observer after
 * every pivot: phase, cumulative iteration, T[0][m] after the pivot, the whole
 * basis (`basic[i]` = variable of row i, num_rows entries; valid only during
 * the callback), the pivot itself, and the counters so far. With rows enabled
 * (lpsg_set_view_observer's with_rows) the callback may call
 * lpsg_read_row(view->solver, i, out) to read tableau row i (row_width
 * doubles) exactly as the reference's view.row(i) returns it; the solver then
 * runs one pivot per device round trip, unfused. */
typedef struct {
    int phase;
    long iteration;
    double objective;
    const int* basic;
    int num_rows;
    int row_width;
    int row, leaving, entering;
    const lpsg_memory* counters;
    struct lpsg_solver* solver;
} lpsg_iteration_view;

typedef void (*lpsg_view_observer)(const lpsg_iteration_view* view, void* user);

typedef struct lpsg_solver lpsg_solver;

/* ---- library ---------------------------------------------------------- */
const char* lpsg_last_error(void);
const char* lpsg_version(void);
/* Number of CUDA devices usable by this library (0 when none). */
int lpsg_device_count(void);
void lpsg_config_default(lpsg_config* cfg);

/* ---- solver lifecycle: replaces SimplexSolver::SimplexSolver (solver.cpp:24-77),
 *      SimplexSolver::solve (solver.cpp:331-392) and two_phase_solve
 *      (solver.hpp:173, solver.cpp:394-397). ---------------------------- */
int lpsg_create(const lpsg_problem* lp, const lpsg_config* cfg, lpsg_solver** out);
int lpsg_solve(lpsg_solver* s, lpsg_report* report);
/* Standard-form point, artificials excluded (solver.cpp:378-383); n = n_total. */
int lpsg_get_x(lpsg_solver* s, double* x, int n);
void lpsg_destroy(lpsg_solver* s);
/* One-shot: create + solve + x + destroy. x may be NULL. */
int lpsg_two_phase_solve(const lpsg_problem* lp, const lpsg_config* cfg, lpsg_report* report,
                         double* x);

/* Per-pivot trace: observer (called on the caller thread, in pivot order,
 * after each device batch) and/or a retained copy of the whole trace. */
int lpsg_set_observer(lpsg_solver* s, lpsg_observer cb, void* user);
int lpsg_keep_trace(lpsg_solver* s, int keep);
int lpsg_get_trace(lpsg_solver* s, lpsg_trace* out, long cap, long* len);
/* SolverConfig::observer with the full IterationView (solver.hpp:21-32). A
 * sharded solve calls it on every rank; with rows, every rank must read the
 * same rows in the same order (lpsg_read_row is a collective there). */
int lpsg_set_view_observer(lpsg_solver* s, lpsg_view_observer cb, void* user, int with_rows);
/* SolveReport::memory (solver.hpp:55). */
int lpsg_get_memory(lpsg_solver* s, lpsg_memory* out);
/* Reinversion mode (lpsg_config.reinvert_every): rebuilds done, Newton steps
 * taken, max |I - B X| before the last rebuild's first step and after its last
 * one, and device seconds spent rebuilding. */
int lpsg_reinvert_stats(lpsg_solver* s, long* rebuilds, long* steps, double* residual_before,
                        double* residual_after, double* seconds);
/* Batched lookaheads of >= 16 candidates. select_leaving's
 * (solver.cpp:215-238, one GPU): how many the bounded selection settled (every
 * later score provably <= the first survivor's) and how many were scored in
 * full. All of them: how many pricings the DMMA screen + exact chains settled
 * and how many needed the exact GEMM after all; probe_rounds: selections whose
 * DMMA probe screen left candidates for the exact probe rounds. Results are
 * identical either way. */
int lpsg_lookahead_stats(lpsg_solver* s, long long* bounded, long long* full, long long* price_bounded,
                         long long* price_exact, long long* probe_rounds);

/* ---- multi-GPU -------------------------
 * NCCL unique id for lpsg_config.nccl_id (rank 0 creates it, the caller
 * distributes it, e.g. over torch.distributed / MPI). */
int lpsg_nccl_unique_id(unsigned char out[128]);
/* One process, `shards` host threads: the sharded solver with in-process
 * exchanges. flags & LPSG_SHARD_SPREAD puts shard g on device
 * (cfg->device + g) % device_count (else all on cfg->device: parity testing on
 * one GPU); flags & LPSG_SHARD_P2P uses the device-initiated P2P transport
 * (else CUDA-event ordered copies with host barriers). Report, x (may be NULL) and trace (may be
 * NULL) are shard 0's; all shards reach the same decisions. */
int lpsg_solve_sharded(const lpsg_problem* lp, const lpsg_config* cfg, int shards, int flags,
                       lpsg_report* report, double* x, lpsg_trace* trace, long cap, long* len);
enum { LPSG_SHARD_SPREAD = 1, LPSG_SHARD_P2P = 2 };
/* Device-initiated P2P transport: every rank allocates a
 * symmetric heap on its GPU (heap_bytes 0 = default 96 MiB) and gets its
 * 64-byte CUDA IPC handle; the caller all-gathers the handles (rank order) and
 * connects. Pass the heap in lpsg_config.peer; destroy after the solver. */
typedef struct lpsg_peer lpsg_peer;
int lpsg_peer_create(int rank, int world, int device, size_t heap_bytes, lpsg_peer** out,
                     unsigned char handle[64]);
int lpsg_peer_connect(lpsg_peer* p, const unsigned char* handles /* world x 64 bytes */);
void lpsg_peer_destroy(lpsg_peer* p);
/* The transport a handle uses: "single", "nccl", "p2p" or "local-events". */
const char* lpsg_transport(lpsg_solver* s);
/* Shard partition used by every sharded solve: shard `rank` of `world` owns the
 * contiguous range [*lo, *hi) of n items (rows of T: n = m; pricing columns:
 * n = n_total), lo = floor(n*rank/world). Pure host arithmetic. */
int lpsg_shard_range(int n, int world, int rank, int* lo, int* hi);
/* Exchange accounting of this handle's shard: collectives issued and payload bytes. */
int lpsg_comm_stats(lpsg_solver* s, long long* calls, double* bytes);
/* Shard geometry: this handle's rows [row0, row0+rows) of T and pricing
 * columns [col0, col1). */
int lpsg_shard_info(lpsg_solver* s, int* world, int* rank, int* row0, int* rows, int* col0, int* col1);

/* ---- step API: SimplexSolver's public steps (solver.hpp:79-168) ----------
 * Single GPU only (a sharded handle returns LPSG_INVALID_ARGUMENT). */
/* price (solver.cpp:79-129) */
int lpsg_price(lpsg_solver* s, int* optimal, int* entering, double* reduced_cost);
/* compute_direction (solver.cpp:131-136) */
int lpsg_compute_direction(lpsg_solver* s, int entering, double reduced_cost);
/* ratio_test (solver.cpp:138-162); candidates ascending, *ncand may exceed cap. */
int lpsg_ratio_test(lpsg_solver* s, int* unbounded, double* theta, int* cand, int cap,
                    int* ncand);
/* select_leaving (solver.cpp:215-238), tabu + batched device lookahead. */
int lpsg_select_leaving(lpsg_solver* s, const int* cand, int ncand, int entering, int* row);
/* lookahead_score (solver.cpp:164-213) for each candidate row, batched. */
int lpsg_lookahead_scores(lpsg_solver* s, const int* rows, int k, int entering, double* scores);
/* pivot_update (solver.cpp:240-254); LPSG_PIVOT_TOO_SMALL when |y_rk| <= pivot_tol. */
int lpsg_pivot_update(lpsg_solver* s, int leaving_row, int entering);

/* Figure-1 tableau accessors (solver.hpp:139-151): row i of m+2 doubles
 * (row 0 = [W | obj | d], row i>0 = [B^-1 row i-1 | b_bar | y]). */
int lpsg_dims(lpsg_solver* s, int* m, int* n_total, int* n_work);
int lpsg_read_row(lpsg_solver* s, int i, double* out);
int lpsg_basis(lpsg_solver* s, int* basic, int m);
int lpsg_phase(lpsg_solver* s);

/* ---- measurement -------------------------------------------------------
 * Budget for the next lpsg_solve call. A solve that stopped with
 * LPSG_ITERATION_LIMIT resumes from the same state (the reference's solve() is
 * single-shot; resuming is an extension used by the benchmark). */
int lpsg_set_max_iter(lpsg_solver* s, long max_iter);

/* Per-kernel CUDA-event timing of the pivot loop (enable resets the counters).
 * algorithmic_bytes is what the reference's step must touch. */
typedef struct {
    const char* name;
    long launches;
    double milliseconds;
    double algorithmic_bytes;
} lpsg_kernel_stat;
int lpsg_profile(lpsg_solver* s, int enable);
int lpsg_profile_get(lpsg_solver* s, lpsg_kernel_stat* out, int cap, int* n);
/* CUDA-event time of the last lpsg_solve call, measured on the solver's stream. */
int lpsg_last_solve_device_ms(lpsg_solver* s, double* ms);
/* Kernel launches issued and host<->device bytes moved since creation. */
int lpsg_counters(lpsg_solver* s, long* kernel_launches, long long* h2d_bytes,
                  long long* d2h_bytes);

/* Measured fp64 SIMT throughput of this device (TFLOP/s), the roofline
 * denominator of the compute-bound batched lookahead: independent DMUL and DADD
 * chains (no FMA, like every lpsg dot) on all SMs, each instruction one flop. */
int lpsg_fp64_peak(int device, double* tflops);

/* Page-locked host buffers (cudaHostAlloc) so lpsg_create's upload of A runs at
 * full DMA bandwidth. Freed with lpsg_host_free. */
int lpsg_host_alloc(size_t bytes, void** out);
void lpsg_host_free(void* p);

/* ---- input plumbing: lps::generate (generator.cpp:35-72) plus the
 *      BASELINE.json input forms and canonicalize (lp_model.cpp:43-163) for
 *      them. form: 0 equality (verbatim), 1 le + maximize, 2 degenerate.
 *      sparsity: 0 dense, 1 S20, 2 S60. Arrays sized m x n_total etc. ----- */
int lpsg_generated_n_total(int rows, int cols, int form);
int lpsg_generate(int rows, int cols, int sparsity, uint64_t seed, int form, double* A,
                  double* b, double* c, uint8_t* col_kind);

#ifdef __cplusplus
}
#endif
#endif /* LPSG_H */
