/* oracle/lps_oracle.c — TEST INFRASTRUCTURE ONLY (the CPU checker; never the
 * product, never linked into paper_1803_04378_b200).
 *
 * Plain-C restatement of the reference's dense revised simplex with tabu
 * anti-cycling, /root/reference/proj. Every function cites the reference
 * lines it restates. Arithmetic contract: IEEE fp64,
 * compiled with -ffp-contract=off like the reference (CMakeLists.txt:14),
 * sequential dot products, same operation order everywhere.
 *
 * Parity pin: checked pivot-for-pivot against the compiled reference
 * (oracle/_ref/liblps_ref.so) and the golden traces in tests/golden/
 * (tests/test_oracle.py).
 */
#include "lps_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---------------------------------------------------------------- RNG --- */
/* std::mt19937_64 (the output sequence is fixed by the C++ standard;
 * generator.cpp:11-15 relies on it). */
typedef struct {
    uint64_t mt[312];
    int idx;
} mt64;

static void mt64_seed(mt64* r, uint64_t seed) {
    r->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
    r->idx = 312;
}

static uint64_t mt64_next(mt64* r) {
    if (r->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
            uint64_t v = r->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) v ^= 0xB5026F5AA96619E9ULL;
            r->mt[i] = v;
        }
        r->idx = 0;
    }
    uint64_t x = r->mt[r->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= (x >> 43);
    return x;
}

/* generator.cpp:13-15: u in (0, 1] */
static double unit_open_closed(mt64* r) { return 1.0 - (double)(mt64_next(r) >> 11) * 0x1.0p-53; }

int lpo_generated_n_total(int rows, int cols, int form) { return form == 0 ? cols : cols + rows; }

/* generator.cpp:35-72, then the input forms of SURVEY.md §8(d), then the
 * parts of canonicalize (lp_model.cpp:43-163) these forms exercise: no bounds,
 * no ranges, b >= 0 (no row negation: lp_model.cpp:118-129 only fires for
 * rhs < 0), max -> min by c = -objective (lp_model.cpp:50,70-75), +1 slack per
 * le row appended after the structurals (lp_model.cpp:150-153). */
int lpo_generate(int rows, int cols, int sparsity, uint64_t seed, int form, double* A,
                 double* b, double* c, uint8_t* col_kind) {
    if (rows <= 0 || cols <= 0) return 1;
    const int m = rows, n = cols;
    const double p_zero = sparsity == 1 ? 0.2 : sparsity == 2 ? 0.6 : 0.0;
    const int nt = lpo_generated_n_total(rows, cols, form);
    mt64* rng = (mt64*)malloc(sizeof(mt64));
    mt64_seed(rng, seed);
    double* coef = (double*)malloc(sizeof(double) * (size_t)m * n);
    double* obj = (double*)malloc(sizeof(double) * n);
    double* xh = (double*)malloc(sizeof(double) * n);
    double* rhs = (double*)malloc(sizeof(double) * m);
    for (int i = 0; i < m; ++i) {
        double* row = coef + (size_t)i * n;
        for (;;) {
            int nonzero = 0;
            for (int j = 0; j < n; ++j) {
                row[j] = 0.01 + 0.99 * unit_open_closed(rng);
                if (p_zero > 0.0 && unit_open_closed(rng) <= p_zero) row[j] = 0.0;
                else nonzero = 1;
            }
            if (nonzero) break;
        }
    }
    for (int j = 0; j < n; ++j) obj[j] = unit_open_closed(rng);
    for (int j = 0; j < n; ++j) xh[j] = unit_open_closed(rng);
    for (int i = 0; i < m; ++i) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += coef[(size_t)i * n + j] * xh[j];
        rhs[i] = acc;
    }
    if (form == 2) {
        for (int i = 0; i + 1 < m; i += 2) {
            for (int j = 0; j < n; ++j)
                coef[(size_t)i * n + j] = coef[(size_t)i * n + j] - coef[(size_t)(i + 1) * n + j];
            rhs[i] = 0.0;
        }
    }
    /* canonicalize: shifted_rhs = rhs - sum a_j * 0 (lp_model.cpp:99-100) is rhs. */
    const double sign = form == 0 ? 1.0 : -1.0;
    memset(A, 0, sizeof(double) * (size_t)m * nt);
    for (int i = 0; i < m; ++i) {
        for (int j = 0; j < n; ++j) A[(size_t)i * nt + j] = coef[(size_t)i * n + j];
        b[i] = rhs[i];
        if (form != 0) A[(size_t)i * nt + n + i] = 1.0;
    }
    for (int j = 0; j < nt; ++j) {
        c[j] = j < n ? sign * obj[j] : 0.0;
        col_kind[j] = j < n ? 0 : 1;
    }
    free(rng);
    free(coef);
    free(obj);
    free(xh);
    free(rhs);
    return 0;
}

/* ------------------------------------------------------------- solver --- */
typedef struct {
    int m, n_total, n_work, art_start, width, rows;
    lpo_config cfg;
    long max_iter;
    double* cols; /* column-major n_work x m (solver.cpp:45-47,58) */
    double* c_true;
    double* c_phase1;
    const double* cost;
    double* T; /* (m+1) x (m+2) Figure-1 tableau, row-major (solver.hpp:71-76) */
    int* basic;
    char* in_basis;
    char* frozen;
    /* TabuState (solver.hpp:66-69): banned pairs (entering, variable) */
    int* ban_k;
    int* ban_v;
    long n_ban, cap_ban;
    double last_objective;
    int phase;
    long total_iter, phase_iter[2];
    /* trace */
    lpo_trace* trace;
    long trace_cap, trace_len;
    /* scratch */
    double* scratch_T;
    char* scratch_inb;
    double* col_buf;
    double* pivot_buf;
} S;

#define ROW(s, i) ((s)->T + (size_t)(i) * (s)->width)

/* solver.cpp:16-20 */
static double dot(const double* a, const double* b, int n) {
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += a[i] * b[i];
    return acc;
}

static const double* column(const S* s, int j) { return s->cols + (size_t)j * s->m; }

/* solver.cpp:318-329 */
static void rebuild_top_row(S* s) {
    const int m = s->m;
    double* top = ROW(s, 0);
    for (int j = 0; j < m; ++j) {
        double acc = 0.0;
        for (int i = 0; i < m; ++i) acc += s->cost[s->basic[i]] * ROW(s, i + 1)[j];
        top[j] = acc;
    }
    double obj = 0.0;
    for (int i = 0; i < m; ++i) obj += s->cost[s->basic[i]] * ROW(s, i + 1)[m];
    top[m] = obj;
    top[m + 1] = 0.0;
}

/* solver.cpp:79-129 (single-chunk scan; the threaded merge is identical) */
static int price(const S* s, int* entering, double* reduced) {
    const double* w = ROW(s, 0);
    int best_j = -1;
    double best_z = 0.0;
    for (int j = 0; j < s->art_start; ++j) {
        if (s->in_basis[j]) continue;
        const double z = dot(w, column(s, j), s->m) - s->cost[j];
        if (best_j < 0 || z > best_z) {
            best_j = j;
            best_z = z;
        }
    }
    *entering = best_j;
    *reduced = best_z;
    return best_j < 0 || best_z <= s->cfg.opt_tol; /* optimal */
}

/* solver.cpp:131-136 */
static void compute_direction(S* s, int entering, double reduced) {
    const double* a = column(s, entering);
    for (int i = 0; i < s->m; ++i) ROW(s, i + 1)[s->m + 1] = dot(ROW(s, i + 1), a, s->m);
    ROW(s, 0)[s->m + 1] = reduced;
}

/* solver.cpp:138-162. Returns number of candidates (0 = unbounded). */
static int ratio_test(const S* s, int* cand) {
    const int m = s->m;
    double theta = INFINITY;
    int any = 0;
    for (int i = 0; i < m; ++i) {
        if (s->frozen[i]) continue;
        const double y = ROW(s, i + 1)[m + 1];
        if (y <= s->cfg.pivot_tol) continue;
        any = 1;
        const double r = ROW(s, i + 1)[m] / y;
        theta = (r < theta) ? r : theta; /* std::min(theta, r) */
    }
    if (!any) return 0;
    const double window = theta + s->cfg.ratio_tie_tol * fmax(1.0, fabs(theta));
    int n = 0;
    for (int i = 0; i < m; ++i) {
        if (s->frozen[i]) continue;
        const double y = ROW(s, i + 1)[m + 1];
        if (y <= s->cfg.pivot_tol) continue;
        if (ROW(s, i + 1)[m] / y <= window) cand[n++] = i;
    }
    return n;
}

/* solver.cpp:164-213 */
static double lookahead_score(S* s, int leaving_row, int entering) {
    const int width = s->width, rows = s->rows, m = s->m;
    double* t = s->scratch_T;
    memcpy(t, s->T, sizeof(double) * (size_t)rows * width);
#define TR(i) (t + (size_t)(i) * width)
    const int pr = leaving_row + 1;
    const double piv = TR(pr)[width - 1];
    if (fabs(piv) <= s->cfg.pivot_tol) return 0.0;
    for (int j = 0; j < width; ++j) TR(pr)[j] /= piv;
    for (int i = 0; i < rows; ++i) {
        if (i == pr) continue;
        const double y = TR(i)[width - 1];
        if (y == 0.0) continue;
        const double* src = TR(pr);
        double* dst = TR(i);
        for (int j = 0; j < width; ++j) dst[j] -= y * src[j];
    }
    char* inb = s->scratch_inb;
    memcpy(inb, s->in_basis, (size_t)s->n_work);
    inb[s->basic[leaving_row]] = 0;
    inb[entering] = 1;

    const double* w = TR(0);
    int best_j = -1;
    double best_z = 0.0;
    for (int j = 0; j < s->art_start; ++j) {
        if (inb[j]) continue;
        const double z = dot(w, column(s, j), m) - s->cost[j];
        if (best_j < 0 || z > best_z) {
            best_j = j;
            best_z = z;
        }
    }
    if (best_j < 0 || best_z <= s->cfg.opt_tol) return 0.0;
    double theta = INFINITY;
    const double* a = column(s, best_j);
    for (int i = 0; i < m; ++i) {
        if (s->frozen[i]) continue;
        const double y = dot(TR(i + 1), a, m);
        if (y <= s->cfg.pivot_tol) continue;
        const double r = TR(i + 1)[m] / y;
        theta = (r < theta) ? r : theta;
    }
    if (isinf(theta)) return INFINITY;
    return best_z * theta;
#undef TR
}

static int is_banned(const S* s, int k, int v) {
    for (long q = 0; q < s->n_ban; ++q)
        if (s->ban_k[q] == k && s->ban_v[q] == v) return 1;
    return 0;
}

static void ban(S* s, int k, int v) {
    if (is_banned(s, k, v)) return;
    if (s->n_ban == s->cap_ban) {
        s->cap_ban = s->cap_ban ? 2 * s->cap_ban : 64;
        s->ban_k = (int*)realloc(s->ban_k, sizeof(int) * s->cap_ban);
        s->ban_v = (int*)realloc(s->ban_v, sizeof(int) * s->cap_ban);
    }
    s->ban_k[s->n_ban] = k;
    s->ban_v[s->n_ban] = v;
    ++s->n_ban;
}

/* Optional record of every scored tie (tests/test_gpu_parity.py compares the
 * device lookahead's scores with these bit for bit): per tie, meta = (pivots
 * done before it, entering, offset into rows/scores, survivor count). */
static struct {
    long* meta;
    int* rows;
    double* scores;
    long cap_ties, cap_rows, n_ties, n_rows;
} g_tie;

void lpo_set_tie_log(long* meta, long cap_ties, int* rows, double* scores, long cap_rows) {
    g_tie.meta = meta;
    g_tie.rows = rows;
    g_tie.scores = scores;
    g_tie.cap_ties = meta ? cap_ties : 0;
    g_tie.cap_rows = cap_rows;
    g_tie.n_ties = g_tie.n_rows = 0;
}

long lpo_tie_log_len(void) { return g_tie.n_ties; }

/* solver.cpp:215-238 */
static int select_leaving(S* s, const int* cand, int n, int entering) {
    if (n == 1) return cand[0];
    if (s->cfg.anticycle == 1) return cand[0];
    int* surv = (int*)malloc(sizeof(int) * n);
    int ns = 0;
    for (int q = 0; q < n; ++q)
        if (!is_banned(s, entering, s->basic[cand[q]])) surv[ns++] = cand[q];
    if (ns == 0) {
        memcpy(surv, cand, sizeof(int) * n);
        ns = n;
    }
    int chosen = surv[0];
    if (ns > 1) {
        double best = -1.0;
        const int log = g_tie.n_ties < g_tie.cap_ties && g_tie.n_rows + ns <= g_tie.cap_rows;
        if (log) {
            long* e = g_tie.meta + 4 * g_tie.n_ties++;
            e[0] = s->total_iter;
            e[1] = entering;
            e[2] = g_tie.n_rows;
            e[3] = ns;
        }
        for (int q = 0; q < ns; ++q) {
            const double score = lookahead_score(s, surv[q], entering);
            if (log) {
                g_tie.rows[g_tie.n_rows] = surv[q];
                g_tie.scores[g_tie.n_rows++] = score;
            }
            if (score > best) {
                best = score;
                chosen = surv[q];
            }
        }
    }
    ban(s, entering, s->basic[chosen]);
    free(surv);
    return chosen;
}

/* solver.cpp:240-254 + tiled_engine.cpp:230-266 (in-core) + tile_kernel
 * cached mode (tiled_engine.cpp:79-106) or, with cfg.kernel == 1, naive mode
 * (61-77). Returns nonzero on PivotTooSmall. */
static int pivot_update(S* s, int leaving_row, int entering) {
    const int m = s->m, width = s->width, rows = s->rows;
    const double y_rk = ROW(s, leaving_row + 1)[m + 1];
    if (fabs(y_rk) <= s->cfg.pivot_tol) return 1;
    double* pr = ROW(s, leaving_row + 1);
    for (int j = 0; j < m + 2; ++j) pr[j] /= y_rk;
    /* tiled_pivot_update */
    const int prow = leaving_row + 1;
    memcpy(s->pivot_buf, ROW(s, prow), sizeof(double) * width);
    for (int i = 0; i < rows; ++i) s->col_buf[i] = ROW(s, i)[width - 1];
    s->col_buf[prow] = 0.0;
    ROW(s, prow)[width - 1] = 0.0;
    for (int i = 0; i < rows; ++i) {
        double* row = ROW(s, i);
        const double y = -s->col_buf[i];
        if (s->cfg.kernel == 1) {
            /* naive mode (tiled_engine.cpp:61-77): every element is stored */
            for (int j = 0; j < width; ++j) row[j] = y * s->pivot_buf[j] + row[j];
            continue;
        }
        for (int j = 0; j < width; ++j) {
            const double temp = y * s->pivot_buf[j];
            if (temp != 0.0) row[j] += temp;
        }
    }
    ROW(s, prow)[width - 1] = 1.0;
    /* basis swap (solver.cpp:251-253) */
    s->in_basis[s->basic[leaving_row]] = 0;
    s->basic[leaving_row] = entering;
    s->in_basis[entering] = 1;
    return 0;
}

/* solver.cpp:256-276, trace in place of the observer */
static void note_iteration(S* s, int row, int leaving, int entering) {
    ++s->total_iter;
    ++s->phase_iter[s->phase - 1];
    const double obj = ROW(s, 0)[s->m];
    if (s->last_objective - obj > s->cfg.opt_tol) s->n_ban = 0;
    s->last_objective = obj;
    if (s->trace && s->trace_len < s->trace_cap) {
        lpo_trace* t = &s->trace[s->trace_len];
        t->iteration = s->total_iter;
        t->phase = s->phase;
        t->row = row;
        t->leaving = leaving;
        t->entering = entering;
        t->objective = obj;
    }
    ++s->trace_len;
}

enum { ST_OPT = 0, ST_UNB = 1, ST_INF = 2, ST_ITL = 3, ST_PIVERR = -2 };

/* solver.cpp:278-293. Returns status. */
static int run_phase(S* s, long budget, int* cand) {
    for (;;) {
        if (s->total_iter >= budget) return ST_ITL;
        int q;
        double z;
        if (price(s, &q, &z)) return ST_OPT;
        compute_direction(s, q, z);
        const int n = ratio_test(s, cand);
        if (n == 0) return ST_UNB;
        const int r = select_leaving(s, cand, n, q);
        const int leaving = s->basic[r];
        if (pivot_update(s, r, q)) return ST_PIVERR;
        note_iteration(s, r, leaving, q);
    }
}

/* solver.cpp:295-316 */
static int drive_out_artificials(S* s) {
    const int m = s->m;
    for (int i = 0; i < m; ++i) {
        if (s->basic[i] < s->art_start) continue;
        int found = -1;
        for (int j = 0; j < s->art_start; ++j) {
            if (s->in_basis[j]) continue;
            if (fabs(dot(ROW(s, i + 1), column(s, j), m)) > s->cfg.pivot_tol) {
                found = j;
                break;
            }
        }
        if (found < 0) {
            s->frozen[i] = 1;
            continue;
        }
        const double red = dot(ROW(s, 0), column(s, found), m) - s->cost[found];
        compute_direction(s, found, red);
        const int leaving = s->basic[i];
        if (pivot_update(s, i, found)) return 1;
        note_iteration(s, i, leaving, found);
    }
    return 0;
}

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}

int lpo_solve(int m, int n_total, const double* A, const double* b, const double* c,
              const uint8_t* col_kind, const lpo_config* cfg, lpo_result* out, double* x,
              lpo_trace* trace, long trace_cap) {
    S s_;
    S* s = &s_;
    memset(s, 0, sizeof(*s));
    s->m = m;
    s->n_total = n_total;
    s->art_start = n_total;
    s->cfg = *cfg;
    s->width = m + 2;
    s->rows = m + 1;
    s->trace = trace;
    s->trace_cap = trace_cap;
    /* constructor, solver.cpp:24-77 */
    s->basic = (int*)malloc(sizeof(int) * m);
    for (int i = 0; i < m; ++i) s->basic[i] = -1;
    for (int j = 0; j < n_total; ++j) {
        if (col_kind[j] != 1) continue; /* ColKind::slack */
        for (int i = 0; i < m; ++i) {
            if (A[(size_t)i * n_total + j] == 1.0 && s->basic[i] < 0) {
                s->basic[i] = j;
                break;
            }
        }
    }
    int n_art = 0;
    for (int i = 0; i < m; ++i)
        if (s->basic[i] < 0) ++n_art;
    s->n_work = n_total + n_art;
    s->cols = (double*)calloc((size_t)(unsigned)s->n_work * (size_t)(unsigned)m, sizeof(double));
    for (int j = 0; j < n_total; ++j)
        for (int i = 0; i < m; ++i) s->cols[(size_t)j * m + i] = A[(size_t)i * n_total + j];
    s->c_true = (double*)calloc((size_t)s->n_work, sizeof(double));
    s->c_phase1 = (double*)calloc((size_t)s->n_work, sizeof(double));
    for (int j = 0; j < n_total; ++j) s->c_true[j] = c[j];
    int next = s->art_start;
    for (int i = 0; i < m; ++i) {
        if (s->basic[i] >= 0) continue;
        s->cols[(size_t)next * m + i] = 1.0;
        s->c_phase1[next] = 1.0;
        s->basic[i] = next++;
    }
    s->in_basis = (char*)calloc((size_t)s->n_work, 1);
    for (int i = 0; i < m; ++i) s->in_basis[s->basic[i]] = 1;
    s->frozen = (char*)calloc((size_t)m, 1);
    s->max_iter = cfg->max_iter > 0 ? cfg->max_iter : 50L * (m + s->n_work);
    s->T = (double*)calloc((size_t)s->rows * s->width, sizeof(double));
    for (int i = 0; i < m; ++i) {
        ROW(s, i + 1)[i] = 1.0;
        ROW(s, i + 1)[m] = b[i];
    }
    s->phase = n_art > 0 ? 1 : 2;
    s->cost = s->phase == 1 ? s->c_phase1 : s->c_true;
    rebuild_top_row(s);
    s->last_objective = ROW(s, 0)[m];
    s->scratch_T = (double*)malloc(sizeof(double) * (size_t)s->rows * s->width);
    s->scratch_inb = (char*)malloc((size_t)s->n_work);
    s->col_buf = (double*)malloc(sizeof(double) * s->rows);
    s->pivot_buf = (double*)malloc(sizeof(double) * s->width);
    int* cand = (int*)malloc(sizeof(int) * (m > 0 ? m : 1));

    /* solve, solver.cpp:331-392 */
    const double t0 = now_s();
    int status = ST_OPT, finished = 0, err = 0;
    if (s->phase == 1) {
        const int st = run_phase(s, s->max_iter, cand);
        if (st == ST_PIVERR) {
            err = 1;
            finished = 1;
        } else if (st == ST_ITL) {
            status = ST_ITL;
            finished = 1;
        } else if (st == ST_UNB || ROW(s, 0)[m] > cfg->feas_tol) {
            status = ST_INF;
            finished = 1;
        } else if (drive_out_artificials(s)) {
            err = 1;
            finished = 1;
        }
    }
    if (!finished) {
        s->phase = 2;
        s->cost = s->c_true;
        rebuild_top_row(s);
        s->n_ban = 0;
        s->last_objective = ROW(s, 0)[m];
        status = run_phase(s, s->max_iter, cand);
        if (status == ST_PIVERR) err = 1;
    }
    const double t1 = now_s();

    out->status = err ? ST_PIVERR : status;
    switch (status) {
        case ST_OPT:
        case ST_ITL: out->objective = ROW(s, 0)[m]; break;
        case ST_UNB: out->objective = -INFINITY; break;
        case ST_INF: out->objective = NAN; break;
        default: out->objective = NAN;
    }
    if (x) {
        for (int j = 0; j < n_total; ++j) x[j] = 0.0;
        if (status == ST_OPT || status == ST_ITL)
            for (int i = 0; i < m; ++i)
                if (s->basic[i] < s->art_start) x[s->basic[i]] = ROW(s, i + 1)[m];
    }
    out->iterations_phase1 = s->phase_iter[0];
    out->iterations_phase2 = s->phase_iter[1];
    out->total_seconds = t1 - t0;
    out->tpi_seconds = out->total_seconds / (double)(s->total_iter > 1 ? s->total_iter : 1);
    out->trace_len = s->trace_len;

    free(cand);
    free(s->basic);
    free(s->cols);
    free(s->c_true);
    free(s->c_phase1);
    free(s->in_basis);
    free(s->frozen);
    free(s->T);
    free(s->scratch_T);
    free(s->scratch_inb);
    free(s->col_buf);
    free(s->pivot_buf);
    free(s->ban_k);
    free(s->ban_v);
    return err ? 2 : 0;
}
