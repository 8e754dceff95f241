// include/lpsg.hpp — header-only C++ shim over the lpsg C ABI (include/lpsg.h).
//
// Mirrors the reference's C++ solver API (/root/reference/proj/include/lps/
// solver.hpp) in its own namespace, so it links beside the reference in one
// binary (the benchmark and parity tools do exactly that):
//
//   lps::two_phase_solve(lp, cfg)          solver.hpp:173
//   ->  lpsg::two_phase_solve(lp, cfg)     same arguments, same report fields
//   lps::SimplexSolver (step API)          solver.hpp:79-168
//   ->  lpsg::SimplexSolver                same member names and meaning
//   lps::IterationView / observer          solver.hpp:21-32
//   ->  lpsg::IterationView                basic, row(i) (with observer_rows), counters
//
// The problem type is duck-typed: anything with the fields of
// lps::StandardFormLP (lp_model.hpp:49-60: m, n_total, A, b, c, col_kind as
// contiguous vectors) works, including lps::StandardFormLP itself. Error codes
// come back as exceptions with the reference's names (errors.hpp:9-11, 58-60);
// pass your own exception types as template arguments to rethrow the
// reference's exact classes.
#pragma once

#include <cstddef>
#include <cstdint>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lpsg.h"

namespace lpsg {

struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct PivotTooSmall : Error {
    using Error::Error;
};
struct CudaError : Error {
    using Error::Error;
};

enum class SolveStatus { optimal, unbounded, infeasible, iteration_limit };  // solver.hpp:14
enum class Anticycle { tabu, none };                                          // solver.hpp:16
enum class KernelMode { cached, naive };                                      // tiled_engine.hpp:26-29

// std::span<const int> stand-in (the shim builds as C++17).
struct IntSpan {
    const int* p = nullptr;
    std::size_t n = 0;
    const int* begin() const { return p; }
    const int* end() const { return p + n; }
    std::size_t size() const { return n; }
    int operator[](std::size_t i) const { return p[i]; }
};

// lps::MemoryCounters counterpart (include/lpsg.h lpsg_memory): real traffic.
using MemoryCounters = lpsg_memory;

struct IterationView {  // solver.hpp:21-30
    int phase = 0;
    long iteration = 0;
    double objective = 0.0;
    IntSpan basic;
    int num_rows = 0;
    int row_width = 0;
    // The i-th tableau row (row_width doubles). Valid during the callback, and
    // only when SolverConfig::observer_rows is set (else empty).
    std::function<const double*(int)> row;
    const MemoryCounters* counters = nullptr;
    int pivot_row = -1, leaving = -1, entering = -1;  // the pivot itself (lpsg addition)
};
using IterationObserver = std::function<void(const IterationView&)>;

struct SolverConfig {  // solver.hpp:34-45
    double opt_tol = 1e-7;
    double pivot_tol = 1e-9;
    double feas_tol = 1e-7;
    double ratio_tie_tol = 1e-9;
    long max_iter = 0;
    Anticycle anticycle = Anticycle::tabu;
    KernelMode kernel = KernelMode::cached;
    int workers = 1;  // accepted, ignored (results are worker-independent)
    IterationObserver observer;
    bool observer_rows = false;  // IterationView::row readable (unfused, one pivot per round trip)
    unsigned long long memory_budget = 0;  // MemoryBudget (solver.hpp:41): tableau bytes; 0 = unlimited
    long reinvert_every = 0;  // opt-in device reinversion (NOT bit-identical to the reference)
    int device = 0;
};

struct SolveReport {  // solver.hpp:47-57
    SolveStatus status = SolveStatus::iteration_limit;
    double objective = 0.0;
    std::vector<double> x;
    long iterations_phase1 = 0;
    long iterations_phase2 = 0;
    double total_seconds = 0.0;
    double tpi_seconds = 0.0;
    MemoryCounters memory{};
    int case_used = 0;  // TileCase (tiled_engine.hpp:24): 0 in-core
};

struct Basis {  // solver.hpp:59-62
    std::vector<int> basic;
    std::vector<char> in_basis;
};

namespace detail {
template <class PivotErr, class OtherErr>
inline void check(int rc) {
    if (rc == LPSG_OK) return;
    const std::string msg = lpsg_last_error();
    if (rc == LPSG_PIVOT_TOO_SMALL) throw PivotErr(msg);
    throw OtherErr(msg);
}

struct ObserverCtx {
    const IterationObserver* obs;
    bool rows;
    std::vector<double> buf;  // the row handed out by IterationView::row
};

inline void view_trampoline(const lpsg_iteration_view* v, void* user) {
    auto* ctx = static_cast<ObserverCtx*>(user);
    IterationView iv;
    iv.phase = v->phase;
    iv.iteration = v->iteration;
    iv.objective = v->objective;
    iv.basic = IntSpan{v->basic, static_cast<std::size_t>(v->num_rows)};
    iv.num_rows = v->num_rows;
    iv.row_width = v->row_width;
    iv.counters = v->counters;
    iv.pivot_row = v->row;
    iv.leaving = v->leaving;
    iv.entering = v->entering;
    if (ctx->rows) {
        lpsg_solver* h = v->solver;
        iv.row = [ctx, h](int i) -> const double* {
            if (lpsg_read_row(h, i, ctx->buf.data()) != LPSG_OK) return nullptr;
            return ctx->buf.data();
        };
    }
    (*ctx->obs)(iv);
}
}  // namespace detail

// Converts anything shaped like lps::StandardFormLP to the C-ABI view (no copy).
template <class LP>
inline lpsg_problem view(const LP& lp, std::vector<uint8_t>& kinds) {
    kinds.resize(lp.col_kind.size());
    for (size_t j = 0; j < kinds.size(); ++j) kinds[j] = static_cast<uint8_t>(lp.col_kind[j]);
    return lpsg_problem{lp.m, lp.n_total, lp.A.data(), lp.b.data(), lp.c.data(), kinds.data()};
}

inline lpsg_config to_c(const SolverConfig& cfg) {
    lpsg_config c;
    lpsg_config_default(&c);
    c.opt_tol = cfg.opt_tol;
    c.pivot_tol = cfg.pivot_tol;
    c.feas_tol = cfg.feas_tol;
    c.ratio_tie_tol = cfg.ratio_tie_tol;
    c.max_iter = cfg.max_iter;
    c.anticycle = cfg.anticycle == Anticycle::none ? 1 : 0;
    c.kernel = cfg.kernel == KernelMode::naive ? 1 : 0;
    c.workers = cfg.workers;
    c.memory_budget = cfg.memory_budget;
    c.reinvert_every = cfg.reinvert_every;
    c.device = cfg.device;
    return c;
}

// lps::SimplexSolver (solver.hpp:79-168) on one GPU: the constructor uploads
// the LP and builds the start basis; solve() runs both phases; the public
// steps are the reference's, each one device round trip.
template <class PivotErr = PivotTooSmall, class OtherErr = CudaError>
class BasicSimplexSolver {
public:
    template <class LP>
    BasicSimplexSolver(const LP& lp, const SolverConfig& cfg = {}) : cfg_(cfg), m_(lp.m), n_total_(lp.n_total) {
        std::vector<uint8_t> kinds;
        const lpsg_problem p = view(lp, kinds);
        const lpsg_config c = to_c(cfg_);
        detail::check<PivotErr, OtherErr>(lpsg_create(&p, &c, &h_));
        if (cfg_.observer) {
            ctx_.obs = &cfg_.observer;
            ctx_.rows = cfg_.observer_rows;
            ctx_.buf.assign(static_cast<std::size_t>(m_) + 2, 0.0);
            const int rc = lpsg_set_view_observer(h_, &detail::view_trampoline, &ctx_, cfg_.observer_rows ? 1 : 0);
            if (rc != LPSG_OK) {
                const std::string msg = lpsg_last_error();
                lpsg_destroy(h_);  // the destructor does not run for a throwing constructor
                throw OtherErr(msg);
            }
        }
    }
    ~BasicSimplexSolver() { lpsg_destroy(h_); }
    BasicSimplexSolver(const BasicSimplexSolver&) = delete;
    BasicSimplexSolver& operator=(const BasicSimplexSolver&) = delete;

    // solver.cpp:331-392
    SolveReport solve() {
        lpsg_report r{};
        check(lpsg_solve(h_, &r));
        SolveReport out;
        out.status = static_cast<SolveStatus>(r.status);
        out.objective = r.objective;
        out.x.assign(static_cast<std::size_t>(n_total_), 0.0);
        check(lpsg_get_x(h_, out.x.data(), n_total_));
        out.iterations_phase1 = r.iterations_phase1;
        out.iterations_phase2 = r.iterations_phase2;
        out.total_seconds = r.total_seconds;
        out.tpi_seconds = r.tpi_seconds;
        check(lpsg_get_memory(h_, &out.memory));
        out.case_used = r.case_used;
        return out;
    }

    struct Pricing {
        bool optimal = false;
        int entering = -1;
        double reduced_cost = 0.0;
    };
    Pricing price() {  // solver.cpp:79-129
        int opt = 0, q = -1;
        double z = 0.0;
        check(lpsg_price(h_, &opt, &q, &z));
        return Pricing{opt != 0, q, z};
    }
    void compute_direction(int entering, double reduced_cost) {  // solver.cpp:131-136
        check(lpsg_compute_direction(h_, entering, reduced_cost));
    }
    struct Ratio {
        bool unbounded = false;
        double theta = 0.0;
        std::vector<int> candidates;
    };
    Ratio ratio_test() const {  // solver.cpp:138-162
        int unb = 0, n = 0;
        double th = 0.0;
        std::vector<int> cand(static_cast<std::size_t>(m_ > 0 ? m_ : 1));
        check(lpsg_ratio_test(h_, &unb, &th, cand.data(), m_, &n));
        cand.resize(static_cast<std::size_t>(unb ? 0 : n));
        return Ratio{unb != 0, th, std::move(cand)};
    }
    int select_leaving(const std::vector<int>& candidates, int entering) {  // solver.cpp:215-238
        int r = -1;
        check(lpsg_select_leaving(h_, candidates.data(), static_cast<int>(candidates.size()), entering, &r));
        return r;
    }
    void pivot_update(int leaving_row, int entering) {  // solver.cpp:240-254
        check(lpsg_pivot_update(h_, leaving_row, entering));
    }

    // Figure-1 tableau accessors (solver.hpp:139-151); each reads one row.
    int m() const { return m_; }
    std::vector<double> row(int i) const {
        std::vector<double> out(static_cast<std::size_t>(m_) + 2);
        check(lpsg_read_row(h_, i, out.data()));
        return out;
    }
    double objective_value() const { return row(0)[m_]; }
    double multiplier(int j) const { return row(0)[j]; }
    double rhs_bar(int i) const { return row(i + 1)[m_]; }
    double inverse_at(int i, int j) const { return row(i + 1)[j]; }
    double entering_value(int i) const { return row(i + 1)[m_ + 1]; }
    double entering_reduced_cost() const { return row(0)[m_ + 1]; }
    Basis basis() const {
        Basis b;
        b.basic.assign(static_cast<std::size_t>(m_), -1);
        check(lpsg_basis(h_, b.basic.data(), m_));
        int n_work = 0;
        check(lpsg_dims(h_, nullptr, nullptr, &n_work));
        b.in_basis.assign(static_cast<std::size_t>(n_work), 0);
        for (int v : b.basic)
            if (v >= 0 && v < n_work) b.in_basis[static_cast<std::size_t>(v)] = 1;
        return b;
    }
    int phase() const { return lpsg_phase(h_); }
    lpsg_solver* handle() const { return h_; }

private:
    static void check(int rc) { detail::check<PivotErr, OtherErr>(rc); }
    SolverConfig cfg_;
    int m_, n_total_;
    lpsg_solver* h_ = nullptr;
    detail::ObserverCtx ctx_{};
};
using SimplexSolver = BasicSimplexSolver<>;

// Drop-in for lps::two_phase_solve (solver.hpp:173, solver.cpp:394-397).
template <class LP, class PivotErr = PivotTooSmall, class OtherErr = CudaError>
inline SolveReport two_phase_solve(const LP& lp, const SolverConfig& cfg = {}) {
    BasicSimplexSolver<PivotErr, OtherErr> s(lp, cfg);
    return s.solve();
}

}  // namespace lpsg
