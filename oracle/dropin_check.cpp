// oracle/dropin_check.cpp — TEST INFRASTRUCTURE. One binary that links the
// unmodified reference (lps_core from oracle/_ref) AND the lpsg product
// through its C++ shim (include/lpsg.hpp), feeds both the identical
// lps::StandardFormLP and compares them:
//
//   1. two_phase_solve with an observer on both sides: per pivot the phase,
//      iteration, objective bits and the WHOLE basis (IterationView::basic,
//      solver.hpp:21-30); then status, iteration counts, objective and x bits.
//   2. `rows` mode: the observer also reads tableau rows 0, 1, m/2 and m at
//      every pivot (IterationView::row, lpsg with observer_rows) and compares
//      them bit for bit.
//   3. The step API (solver.hpp:79-168) driven by hand for STEPS pivots on
//      both: price, compute_direction, ratio_test, select_leaving,
//      pivot_update, compared bit for bit after every call, plus the Figure-1
//      accessors and the basis.
//
// This is the reference-side integration shown in INTEGRATION.md, exercised
// for real.
//
//   4. `parts=P`: both libraries under a memory budget of ~P row partitions
//      (the reference's own Case 2, tiled_engine.cpp:29-54, against lpsg's),
//      `naive`: both with KernelMode::naive.
//
// usage: dropin_check ROWS COLS FORM SEED [rows] [steps=N] [parts=P] [naive]
//        (FORM 0 eq, 1 le+max, 2 degenerate)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "lpsg.hpp"
#include "lps/errors.hpp"
#include "lps/generator.hpp"
#include "lps/lp_model.hpp"
#include "lps/solver.hpp"

namespace {

struct Piv {
    long it;
    int phase;
    double obj;
    std::vector<int> basic;
    std::vector<double> rows;  // rows 0, 1, m/2, m when sampled
};

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

bool same_bits(const std::vector<double>& a, const std::vector<double>& b) {
    return a.size() == b.size() && (a.empty() || std::memcmp(a.data(), b.data(), sizeof(double) * a.size()) == 0);
}

int fails = 0;
void expect(bool ok, const std::string& what) {
    if (!ok && fails++ < 10) std::printf("  mismatch: %s\n", what.c_str());
}

template <class View>
std::vector<double> sample_rows(const View& v, int m) {
    std::vector<double> out;
    const int pick[4] = {0, 1, m / 2, m};
    for (int i : pick) {
        const double* r = v.row(i);
        if (!r) return {};
        out.insert(out.end(), r, r + m + 2);
    }
    return out;
}

}  // namespace

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s ROWS COLS FORM SEED [rows] [steps=N] [parts=P] [naive]\n", argv[0]);
        return 2;
    }
    const int rows = std::atoi(argv[1]), cols = std::atoi(argv[2]), form = std::atoi(argv[3]);
    const unsigned long long seed = std::strtoull(argv[4], nullptr, 10);
    bool with_rows = false, naive = false;
    int steps = 0, parts = 0;
    for (int a = 5; a < argc; ++a) {
        if (std::strcmp(argv[a], "rows") == 0) with_rows = true;
        if (std::strcmp(argv[a], "naive") == 0) naive = true;
        if (std::strncmp(argv[a], "steps=", 6) == 0) steps = std::atoi(argv[a] + 6);
        if (std::strncmp(argv[a], "parts=", 6) == 0) parts = std::atoi(argv[a] + 6);
    }
    lps::GeneralLP g = lps::generate({rows, cols, lps::SparsityClass::dense, seed});
    if (form >= 1) {
        for (auto& k : g.row_kind) k = lps::RowKind::le;
        g.sense = lps::Sense::maximize;
    }
    if (form == 2)
        for (int i = 0; i + 1 < g.num_rows; i += 2) {
            for (int j = 0; j < g.num_cols; ++j) g.at(i, j) = g.at(i, j) - g.at(i + 1, j);
            g.rhs[i] = 0.0;
        }
    const auto [lp, map] = lps::canonicalize(g);
    const int m = lp.m;

    // ---- 1 + 2: two_phase_solve with observers
    // parts=P: a memory budget of ~P row partitions on BOTH sides, i.e. the
    // reference's own Case 2 (tiled_engine.cpp:29-54) against lpsg's
    const unsigned long long row_bytes = 8ULL * (unsigned long long)(m + 2);
    const unsigned long long budget =
        parts > 0 ? row_bytes * (unsigned long long)((m + 1 + parts - 1) / parts + 1) : 0ULL;
    std::vector<Piv> ref_tr, gpu_tr;
    lps::SolverConfig rc;
    if (budget) rc.memory_budget = lps::MemoryBudget::of_bytes(budget);
    if (naive) rc.kernel = lps::KernelMode::naive;
    rc.observer = [&](const lps::IterationView& v) {
        Piv p{v.iteration, v.phase, v.objective, std::vector<int>(v.basic.begin(), v.basic.end()), {}};
        if (with_rows) p.rows = sample_rows(v, m);
        ref_tr.push_back(std::move(p));
    };
    const lps::SolveReport r = lps::two_phase_solve(lp, rc);

    lpsg::SolverConfig gc;
    gc.observer_rows = with_rows;
    gc.memory_budget = budget;
    if (naive) gc.kernel = lpsg::KernelMode::naive;
    gc.observer = [&](const lpsg::IterationView& v) {
        Piv p{v.iteration, v.phase, v.objective, std::vector<int>(v.basic.begin(), v.basic.end()), {}};
        if (with_rows) p.rows = sample_rows(v, m);
        gpu_tr.push_back(std::move(p));
    };
    lpsg::SolveReport q;
    try {
        q = lpsg::two_phase_solve<lps::StandardFormLP, lps::PivotTooSmall, lps::Error>(lp, gc);
    } catch (const lps::Error& e) {
        std::printf("FAIL lpsg error: %s\n", e.what());
        return 1;
    }
    expect(int(q.status) == int(r.status), "status");
    expect(q.iterations_phase1 == r.iterations_phase1 && q.iterations_phase2 == r.iterations_phase2,
           "iteration counts");
    expect(ref_tr.size() == gpu_tr.size(), "observer calls");
    for (size_t k = 0; k < std::min(ref_tr.size(), gpu_tr.size()); ++k) {
        const Piv &a = ref_tr[k], &b = gpu_tr[k];
        expect(a.it == b.it && a.phase == b.phase, "pivot " + std::to_string(k) + " iteration/phase");
        expect(same_bits(a.obj, b.obj), "pivot " + std::to_string(k) + " objective");
        expect(a.basic == b.basic, "pivot " + std::to_string(k) + " basis");
        if (with_rows) expect(!a.rows.empty() && same_bits(a.rows, b.rows), "pivot " + std::to_string(k) + " rows");
    }
    expect(same_bits(q.objective, r.objective) || (q.objective != q.objective && r.objective != r.objective),
           "objective");
    expect(same_bits(q.x, r.x), "x");
    expect(q.case_used == (r.case_used == lps::TileCase::tiled ? 1 : 0), "case_used");

    // ---- 3: the step API by hand
    int step_pivots = 0;
    if (steps > 0) {
        lps::SolverConfig c0;
        lps::SimplexSolver rs(lp, c0);
        rs.engine().begin_solve();  // in-core arena, like solve() (solver.cpp:333)
        lpsg::BasicSimplexSolver<lps::PivotTooSmall, lps::Error> gs(lp, lpsg::SolverConfig{});
        expect(rs.basis().basic == gs.basis().basic, "start basis");
        expect(rs.phase() == gs.phase(), "start phase");
        for (int t = 0; t < steps; ++t) {
            const auto pr = rs.price();
            const auto pg = gs.price();
            expect(pr.optimal == pg.optimal && pr.entering == pg.entering && same_bits(pr.reduced_cost, pg.reduced_cost),
                   "step " + std::to_string(t) + " price");
            if (pr.optimal || pr.entering != pg.entering) break;
            rs.compute_direction(pr.entering, pr.reduced_cost);
            gs.compute_direction(pg.entering, pg.reduced_cost);
            for (int i : {0, m / 2, m - 1})
                expect(same_bits(rs.entering_value(i), gs.entering_value(i)), "step " + std::to_string(t) + " y");
            expect(same_bits(rs.entering_reduced_cost(), gs.entering_reduced_cost()), "step d slot");
            const auto tr_ = rs.ratio_test();
            const auto tg = gs.ratio_test();
            expect(tr_.unbounded == tg.unbounded && same_bits(tr_.theta, tg.theta) && tr_.candidates == tg.candidates,
                   "step " + std::to_string(t) + " ratio_test");
            if (tr_.unbounded || tr_.candidates != tg.candidates) break;
            const int lr = rs.select_leaving(tr_.candidates, pr.entering);
            const int lg = gs.select_leaving(tg.candidates, pg.entering);
            expect(lr == lg, "step " + std::to_string(t) + " select_leaving");
            if (lr != lg) break;
            rs.pivot_update(lr, pr.entering);
            gs.pivot_update(lg, pg.entering);
            ++step_pivots;
            expect(rs.basis().basic == gs.basis().basic, "step " + std::to_string(t) + " basis");
            expect(same_bits(rs.objective_value(), gs.objective_value()), "step objective_value");
            for (int i : {0, lr, m - 1}) {
                expect(same_bits(rs.rhs_bar(i), gs.rhs_bar(i)), "step rhs_bar");
                expect(same_bits(rs.inverse_at(i, lr), gs.inverse_at(i, lr)), "step inverse_at");
                expect(same_bits(rs.multiplier(i), gs.multiplier(i)), "step multiplier");
            }
        }
        // a too-small pivot raises the reference's own exception type
        bool threw = false;
        try {
            gs.pivot_update(0, -1);  // bad index: LPSG_INVALID_ARGUMENT
        } catch (const lps::Error&) {
            threw = true;
        }
        expect(threw, "bad pivot_update raises lps::Error");
    }

    const bool ok = fails == 0;
    std::printf("%s %dx%d form %d seed %llu%s%s%s: %zu pivots, status %d, objective %.17g (ref %.17g), "
                "ref %.3f s, lpsg %.3f s, step-API pivots %d, lpsg device bytes %llu\n",
                ok ? "PASS" : "FAIL", rows, cols, form, seed, with_rows ? " rows" : "", naive ? " naive" : "",
                q.case_used ? " tiled" : "", gpu_tr.size(),
                int(q.status), q.objective, r.objective, r.total_seconds, q.total_seconds, step_pivots,
                (unsigned long long)(q.memory.device_read_bytes + q.memory.device_write_bytes));
    return ok ? 0 : 1;
}
