/* oracle/lps_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement ("port") of the reference's hot path, used as the CPU
 * checker for the CUDA product and as bench.py's cpu_baseline when the
 * reference library (oracle/_ref) is unavailable. The struct layouts match
 * oracle/ref_shim.cpp so one set of ctypes structs serves both.
 *
 * Parity pin: tests/test_oracle.py checks this port pivot-for-pivot (and bit
 * for bit on objective / x) against the compiled reference (oracle/_ref) on
 * generated LPs and against the committed golden traces in tests/golden/.
 */
#ifndef LPS_ORACLE_H
#define LPS_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
    double opt_tol, pivot_tol, feas_tol, ratio_tie_tol;
    long max_iter;
    int anticycle; /* 0 tabu, 1 none */
    int workers;   /* accepted, ignored (results are worker-independent, solver.cpp:99-121) */
    int kernel;    /* 0 cached (tiled_engine.cpp:79-106), 1 naive (61-77): zero signs differ */
} lpo_config;

typedef struct {
    long iteration;
    int phase, row, leaving, entering;
    double objective;
} lpo_trace;

typedef struct {
    int status; /* 0 optimal, 1 unbounded, 2 infeasible, 3 iteration_limit, <0 error */
    double objective;
    long iterations_phase1, iterations_phase2;
    double total_seconds, tpi_seconds;
    long trace_len;
} lpo_result;

/* Column count of the standard form produced by lpo_generate. */
int lpo_generated_n_total(int rows, int cols, int form);

/* generator.cpp:35-72 + the BASELINE input forms + canonicalize (lp_model.cpp:43-163)
 * restricted to what those forms exercise. form 0 eq, 1 le+max, 2 degenerate. */
int lpo_generate(int rows, int cols, int sparsity, uint64_t seed, int form, double* A,
                 double* b, double* c, uint8_t* col_kind);

/* solver.cpp:24-397 (two_phase_solve). Returns 0, or 2 on PivotTooSmall. */
int lpo_solve(int m, int n_total, const double* A, const double* b, const double* c,
              const uint8_t* col_kind, const lpo_config* cfg, lpo_result* out, double* x,
              lpo_trace* trace, long trace_cap);

/* Test hook: the next lpo_solve calls record every tie that select_leaving
 * scores (solver.cpp:225-235): meta[4k..4k+3] = (pivots done before the tie,
 * entering column, offset into rows/scores, number of scored survivors);
 * rows/scores = the survivors and their lookahead_score values. NULL meta
 * turns it off. Not thread-safe (test infrastructure). */
void lpo_set_tie_log(long* meta, long cap_ties, int* rows, double* scores, long cap_rows);
long lpo_tie_log_len(void);

#ifdef __cplusplus
}
#endif
#endif
