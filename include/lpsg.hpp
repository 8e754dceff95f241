// include/lpsg.hpp — header-only C++ shim over the lpsg C ABI (include/lpsg.h).
//
// Mirrors the reference's C++ solver API (/root/reference/proj/include/lps/
// solver.hpp) in its own namespace, so it links beside the reference in one
// binary (the benchmark and parity tools do exactly that):
//
//   lps::two_phase_solve(lp, cfg)          solver.hpp:173
//   ->  lpsg::two_phase_solve(lp, cfg)     same arguments, same report fields
//
// The problem type is duck-typed: anything with the fields of
// lps::StandardFormLP (lp_model.hpp:49-60: m, n_total, A, b, c, col_kind as
// contiguous vectors) works, including lps::StandardFormLP itself. Error codes
// come back as exceptions with the reference's names (errors.hpp:9-11, 58-60);
// pass your own exception types as template arguments to rethrow the
// reference's exact classes.
#pragma once

#include <cstdint>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
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

struct IterationView {  // solver.hpp:21-30 without the tableau rows
    int phase = 0;
    long iteration = 0;
    double objective = 0.0;
    int row = -1, leaving = -1, entering = -1;
};
using IterationObserver = std::function<void(const IterationView&)>;

struct SolverConfig {  // solver.hpp:34-45
    double opt_tol = 1e-7;
    double pivot_tol = 1e-9;
    double feas_tol = 1e-7;
    double ratio_tie_tol = 1e-9;
    long max_iter = 0;
    Anticycle anticycle = Anticycle::tabu;
    int device = 0;
    IterationObserver observer;
};

struct SolveReport {  // solver.hpp:47-57
    SolveStatus status = SolveStatus::iteration_limit;
    double objective = 0.0;
    std::vector<double> x;
    long iterations_phase1 = 0;
    long iterations_phase2 = 0;
    double total_seconds = 0.0;
    double tpi_seconds = 0.0;
};

namespace detail {
template <class PivotErr, class OtherErr>
inline void check(int rc) {
    if (rc == LPSG_OK) return;
    const std::string msg = lpsg_last_error();
    if (rc == LPSG_PIVOT_TOO_SMALL) throw PivotErr(msg);
    throw OtherErr(msg);
}
inline void trampoline(const lpsg_trace* t, void* user) {
    const auto& obs = *static_cast<const IterationObserver*>(user);
    obs(IterationView{t->phase, t->iteration, t->objective, t->row, t->leaving, t->entering});
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
    c.device = cfg.device;
    return c;
}

// Drop-in for lps::two_phase_solve (solver.hpp:173, solver.cpp:394-397).
template <class LP, class PivotErr = PivotTooSmall, class OtherErr = CudaError>
inline SolveReport two_phase_solve(const LP& lp, const SolverConfig& cfg = {}) {
    std::vector<uint8_t> kinds;
    const lpsg_problem p = view(lp, kinds);
    const lpsg_config c = to_c(cfg);
    lpsg_solver* h = nullptr;
    detail::check<PivotErr, OtherErr>(lpsg_create(&p, &c, &h));
    struct Guard {
        lpsg_solver* h;
        ~Guard() { lpsg_destroy(h); }
    } guard{h};
    if (cfg.observer)
        detail::check<PivotErr, OtherErr>(
            lpsg_set_observer(h, &detail::trampoline, const_cast<IterationObserver*>(&cfg.observer)));
    lpsg_report r{};
    detail::check<PivotErr, OtherErr>(lpsg_solve(h, &r));
    SolveReport out;
    out.status = static_cast<SolveStatus>(r.status);
    out.objective = r.objective;
    out.x.assign(lp.n_total, 0.0);
    detail::check<PivotErr, OtherErr>(lpsg_get_x(h, out.x.data(), lp.n_total));
    out.iterations_phase1 = r.iterations_phase1;
    out.iterations_phase2 = r.iterations_phase2;
    out.total_seconds = r.total_seconds;
    out.tpi_seconds = r.tpi_seconds;
    return out;
}

}  // namespace lpsg
