// oracle/ref_shim.cpp — TEST INFRASTRUCTURE ONLY (never linked into the product).
//
// A thin extern "C" face over the UNMODIFIED reference library `lps_core`
// (compiled from /root/reference/proj/src/*.cpp by oracle/Makefile into
// oracle/_ref/liblps_ref.so). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs load it, as the checker and
// as the CPU baseline; the product path never does.
//
// Entry points:
//   * ref_lp_generate  — lps::generate (generator.cpp:35-72) + the three input
//     forms used by BASELINE.json's configs + lps::canonicalize
//     (lp_model.cpp:43-163).
//   * ref_lp_from_mps  — lps::parse_mps_file + to_general_lp + canonicalize
//     (mps.cpp:216,227) for the Netlib fixtures.
//   * ref_mps_*        — the MPS ingestion chain on in-memory text: parse_mps +
//     to_general_lp (warnings kept) + canonicalize (+ CanonicalMap) +
//     recover_solution, write_mps and to_mps_document (mps.cpp, lp_model.cpp),
//     for the ingestion parity tests (tests/test_mps.py).
//   * ref_solve        — lps::two_phase_solve (solver.cpp:394-397) with a
//     per-pivot trace taken through SolverConfig::observer (solver.hpp:21-32,
//     solver.cpp:264-275): the changed basis row is found by diffing `basic`.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

#include "lps/errors.hpp"
#include "lps/generator.hpp"
#include "lps/lp_model.hpp"
#include "lps/mps.hpp"
#include "lps/solver.hpp"

namespace {

thread_local std::string g_err;

struct RefLP {
    lps::StandardFormLP lp;
    lps::CanonicalMap map;
    std::vector<std::string> warnings;  // parse + to_general_lp, in order
    std::string written;                // write_mps(parse_mps(text))
};

// The most derived lps error type, for the error-behaviour parity tests.
const char* error_kind(const std::exception& e) {
#define LPS_KIND(T) \
    if (dynamic_cast<const lps::T*>(&e)) return #T;
    LPS_KIND(InconsistentBounds) LPS_KIND(EmptyProblem) LPS_KIND(LengthMismatch)
    LPS_KIND(UnknownSection) LPS_KIND(UndeclaredRow) LPS_KIND(DuplicateRow)
    LPS_KIND(MissingObjectiveRow) LPS_KIND(MalformedNumber) LPS_KIND(UnsupportedBoundKind)
    LPS_KIND(Error)
#undef LPS_KIND
    return "std::exception";
}

thread_local std::string g_kind;
thread_local std::string g_text;

}  // namespace

extern "C" {

struct ref_config {
    double opt_tol, pivot_tol, feas_tol, ratio_tie_tol;
    long max_iter;
    int anticycle;  // 0 tabu, 1 none
    int workers;
    int kernel;     // 0 cached, 1 naive
};

struct ref_trace {
    long iteration;
    int phase;
    int row;        // leaving row (index into basic[])
    int leaving;    // leaving variable (column index, artificials >= n_total)
    int entering;   // entering variable
    double objective;
};

struct ref_result {
    int status;  // 0 optimal, 1 unbounded, 2 infeasible, 3 iteration_limit, -1 error
    double objective;
    long iterations_phase1, iterations_phase2;
    double total_seconds, tpi_seconds;
    long trace_len;  // pivots observed (may exceed the trace capacity)
};

const char* ref_last_error() { return g_err.c_str(); }

// form: 0 = generator verbatim (all rows eq, generator.cpp:47)
//       1 = rows le + maximize (slack start)
//       2 = degenerate recipe (1 + rows i=0,2,4..: a_i -= a_{i+1}, b_i = 0)
void* ref_lp_generate(int rows, int cols, int sparsity, std::uint64_t seed, int form) {
    try {
        lps::GenSpec spec{rows, cols, static_cast<lps::SparsityClass>(sparsity), seed};
        lps::GeneralLP g = lps::generate(spec);
        if (form >= 1) {
            for (int i = 0; i < g.num_rows; ++i) g.row_kind[i] = lps::RowKind::le;
            g.sense = lps::Sense::maximize;
        }
        if (form == 2) {
            for (int i = 0; i + 1 < g.num_rows; i += 2) {
                for (int j = 0; j < g.num_cols; ++j) g.at(i, j) = g.at(i, j) - g.at(i + 1, j);
                g.rhs[i] = 0.0;
            }
        }
        auto [lp, map] = lps::canonicalize(g);
        return new RefLP{std::move(lp), std::move(map)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void* ref_lp_from_mps(const char* path) {
    try {
        lps::GeneralLP g = lps::to_general_lp(lps::parse_mps_file(path));
        auto [lp, map] = lps::canonicalize(g);
        return new RefLP{std::move(lp), std::move(map)};
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// parse_mps(text) -> to_general_lp -> canonicalize; nullptr on error
// (ref_last_error / ref_last_error_kind).
void* ref_mps_load(const char* text) {
    try {
        auto* r = new RefLP{};
        lps::MpsDocument doc = lps::parse_mps(std::string(text));
        r->warnings = doc.warnings;
        r->written = lps::write_mps(doc);
        lps::GeneralLP g;
        try {
            g = lps::to_general_lp(doc, &r->warnings);
            auto [lp, map] = lps::canonicalize(g);
            r->lp = std::move(lp);
            r->map = std::move(map);
        } catch (...) {
            delete r;
            throw;
        }
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_kind = error_kind(e);
        return nullptr;
    }
}

const char* ref_last_error_kind() { return g_kind.c_str(); }

// Warnings joined by '\n', then the written document, as NUL-free text.
const char* ref_mps_warnings(void* h) {
    g_text.clear();
    for (const auto& w : static_cast<RefLP*>(h)->warnings) g_text += w + "\n";
    return g_text.c_str();
}

const char* ref_mps_written(void* h) { return static_cast<RefLP*>(h)->written.c_str(); }

// CanonicalMap: shift[orig_cols], negated_row[m] (0/1), split pairs (pos, neg).
void ref_mps_map(void* h, int* orig_cols, int* n_split, double* shift, std::uint8_t* negated,
                 int* split_pos, int* split_neg) {
    const lps::CanonicalMap& mp = static_cast<RefLP*>(h)->map;
    *orig_cols = mp.orig_cols;
    *n_split = int(mp.split_pairs.size());
    if (shift) std::memcpy(shift, mp.shift.data(), sizeof(double) * mp.shift.size());
    if (negated)
        for (std::size_t i = 0; i < mp.negated_row.size(); ++i) negated[i] = mp.negated_row[i] ? 1 : 0;
    for (std::size_t k = 0; k < mp.split_pairs.size(); ++k) {
        if (split_pos) split_pos[k] = mp.split_pairs[k].pos;
        if (split_neg) split_neg[k] = mp.split_pairs[k].neg;
    }
}

// recover_solution(map, x_std[n], z_std) -> x[orig_cols], *z; 1 on error.
int ref_mps_recover(void* h, const double* x_std, int n, double z_std, double* x, double* z) {
    try {
        auto [xo, zo] = lps::recover_solution(static_cast<RefLP*>(h)->map,
                                              std::vector<double>(x_std, x_std + n), z_std);
        std::memcpy(x, xo.data(), sizeof(double) * xo.size());
        *z = zo;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        g_kind = error_kind(e);
        return 1;
    }
}

// write_mps(to_mps_document(generate(spec) with the input form)): the text
// a generated instance is saved as.
const char* ref_generated_mps(int rows, int cols, int sparsity, std::uint64_t seed, int form) {
    try {
        lps::GeneralLP g = lps::generate({rows, cols, static_cast<lps::SparsityClass>(sparsity), seed});
        if (form >= 1) {
            for (int i = 0; i < g.num_rows; ++i) g.row_kind[i] = lps::RowKind::le;
            g.sense = lps::Sense::maximize;
        }
        g_text = lps::write_mps(lps::to_mps_document(g));
        return g_text.c_str();
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_lp_dims(void* h, int* m, int* n_total) {
    auto* p = static_cast<RefLP*>(h);
    *m = p->lp.m;
    *n_total = p->lp.n_total;
}

void ref_lp_copy(void* h, double* A, double* b, double* c, std::uint8_t* col_kind,
                 double* objective_sign, double* objective_constant) {
    auto* p = static_cast<RefLP*>(h);
    std::memcpy(A, p->lp.A.data(), p->lp.A.size() * sizeof(double));
    std::memcpy(b, p->lp.b.data(), p->lp.b.size() * sizeof(double));
    std::memcpy(c, p->lp.c.data(), p->lp.c.size() * sizeof(double));
    for (int j = 0; j < p->lp.n_total; ++j) col_kind[j] = static_cast<std::uint8_t>(p->lp.col_kind[j]);
    if (objective_sign) *objective_sign = p->map.objective_sign;
    if (objective_constant) *objective_constant = p->map.objective_constant;
}

void ref_lp_free(void* h) { delete static_cast<RefLP*>(h); }

// Solves the standard-form LP given by plain arrays (copied into a
// lps::StandardFormLP) with lps::two_phase_solve. `x` receives n_total values;
// `trace` receives up to trace_cap pivots.
int ref_solve(int m, int n_total, const double* A, const double* b, const double* c,
              const std::uint8_t* col_kind, const ref_config* cfg, ref_result* out,
              double* x, ref_trace* trace, long trace_cap) {
    try {
        lps::StandardFormLP lp;
        lp.m = m;
        lp.n_total = n_total;
        lp.A.assign(A, A + std::size_t(m) * n_total);
        lp.b.assign(b, b + m);
        lp.c.assign(c, c + n_total);
        lp.col_kind.resize(n_total);
        for (int j = 0; j < n_total; ++j) lp.col_kind[j] = static_cast<lps::ColKind>(col_kind[j]);

        lps::SolverConfig sc;
        sc.opt_tol = cfg->opt_tol;
        sc.pivot_tol = cfg->pivot_tol;
        sc.feas_tol = cfg->feas_tol;
        sc.ratio_tie_tol = cfg->ratio_tie_tol;
        sc.max_iter = cfg->max_iter;
        sc.anticycle = cfg->anticycle == 1 ? lps::Anticycle::none : lps::Anticycle::tabu;
        sc.workers = cfg->workers;
        sc.kernel = cfg->kernel == 1 ? lps::KernelMode::naive : lps::KernelMode::cached;

        long count = 0;
        std::vector<int> prev;
        bool have_prev = false;
        if (trace && trace_cap > 0) {
            sc.observer = [&](const lps::IterationView& v) {
                int row = -1, leaving = -1, entering = -1;
                if (have_prev) {
                    for (int i = 0; i < int(v.basic.size()); ++i)
                        if (v.basic[i] != prev[i]) {
                            row = i;
                            leaving = prev[i];
                            entering = v.basic[i];
                            break;
                        }
                }
                if (count < trace_cap) {
                    trace[count] = ref_trace{v.iteration, v.phase, row, leaving, entering, v.objective};
                }
                ++count;
                prev.assign(v.basic.begin(), v.basic.end());
            };
        }
        // The observer only sees the basis after each pivot, so the initial basis
        // is reconstructed by a throwaway solver (constructor only; solver.cpp:24-77).
        if (trace && trace_cap > 0) {
            lps::SolverConfig c0 = sc;
            c0.observer = nullptr;
            lps::SimplexSolver probe(lp, c0);
            prev = probe.basis().basic;
            have_prev = true;
        }
        const lps::SolveReport r = lps::two_phase_solve(lp, sc);
        out->status = static_cast<int>(r.status);
        out->objective = r.objective;
        out->iterations_phase1 = r.iterations_phase1;
        out->iterations_phase2 = r.iterations_phase2;
        out->total_seconds = r.total_seconds;
        out->tpi_seconds = r.tpi_seconds;
        out->trace_len = count;
        if (x) std::memcpy(x, r.x.data(), r.x.size() * sizeof(double));
        return 0;
    } catch (const lps::PivotTooSmall& e) {
        g_err = e.what();
        out->status = -2;
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        out->status = -1;
        return 1;
    }
}

// Same solve, for bench.py's reference arm: `stamps[k]` = steady_clock seconds
// at the observer call of pivot k+1 (solver.cpp:264-275, right after the
// pivot's update), and *t_return = steady_clock seconds when two_phase_solve
// returned. A pivot window [W, W+K) is then stamps[W+K-1] - stamps[W-1]; for W
// = 0 the start is t_return - total_seconds (solve()'s own clock start,
// solver.cpp:332, up to the report's construction after the clock stops).
int ref_solve_timed(int m, int n_total, const double* A, const double* b, const double* c,
                    const std::uint8_t* col_kind, const ref_config* cfg, ref_result* out,
                    double* stamps, long cap, double* t_return) {
    try {
        lps::StandardFormLP lp;
        lp.m = m;
        lp.n_total = n_total;
        lp.A.assign(A, A + std::size_t(m) * n_total);
        lp.b.assign(b, b + m);
        lp.c.assign(c, c + n_total);
        lp.col_kind.resize(n_total);
        for (int j = 0; j < n_total; ++j) lp.col_kind[j] = static_cast<lps::ColKind>(col_kind[j]);
        lps::SolverConfig sc;
        sc.opt_tol = cfg->opt_tol;
        sc.pivot_tol = cfg->pivot_tol;
        sc.feas_tol = cfg->feas_tol;
        sc.ratio_tie_tol = cfg->ratio_tie_tol;
        sc.max_iter = cfg->max_iter;
        sc.anticycle = cfg->anticycle == 1 ? lps::Anticycle::none : lps::Anticycle::tabu;
        sc.workers = cfg->workers;
        sc.kernel = cfg->kernel == 1 ? lps::KernelMode::naive : lps::KernelMode::cached;
        long count = 0;
        auto now = [] {
            return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
        };
        sc.observer = [&](const lps::IterationView&) {
            if (count < cap) stamps[count] = now();
            ++count;
        };
        const lps::SolveReport r = lps::two_phase_solve(lp, sc);
        *t_return = now();
        out->status = static_cast<int>(r.status);
        out->objective = r.objective;
        out->iterations_phase1 = r.iterations_phase1;
        out->iterations_phase2 = r.iterations_phase2;
        out->total_seconds = r.total_seconds;
        out->tpi_seconds = r.tpi_seconds;
        out->trace_len = count;
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        out->status = -1;
        return 1;
    }
}

}  // extern "C"
