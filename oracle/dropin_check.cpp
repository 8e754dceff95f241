// oracle/dropin_check.cpp — TEST INFRASTRUCTURE. One binary that links the
// unmodified reference (lps_core from oracle/_ref) AND the lpsg product
// through its C++ shim (include/lpsg.hpp), feeds both the identical
// lps::StandardFormLP and compares them pivot for pivot (observer traces),
// status, objective bits and x bits. This is the reference-side integration
// shown in INTEGRATION.md, exercised for real.
//
// usage: dropin_check ROWS COLS FORM SEED   (FORM 0 eq, 1 le+max, 2 degenerate)
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "lpsg.hpp"
#include "lps/errors.hpp"
#include "lps/generator.hpp"
#include "lps/lp_model.hpp"
#include "lps/solver.hpp"

struct Piv {
    long it;
    int phase, entering;
    double obj;
};

int main(int argc, char** argv) {
    if (argc < 5) {
        std::fprintf(stderr, "usage: %s ROWS COLS FORM SEED\n", argv[0]);
        return 2;
    }
    const int rows = std::atoi(argv[1]), cols = std::atoi(argv[2]), form = std::atoi(argv[3]);
    const unsigned long long seed = std::strtoull(argv[4], nullptr, 10);
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

    std::vector<Piv> ref_tr, gpu_tr;
    lps::SolverConfig rc;
    rc.observer = [&](const lps::IterationView& v) {
        // entering variable: the basis entry that changed is not exposed directly;
        // record (iteration, phase, objective) plus the basis checksum via basic
        long sum = 0;
        for (int b : v.basic) sum = sum * 1000003 + b;
        ref_tr.push_back({v.iteration, v.phase, (int)(sum & 0x7fffffff), v.objective});
    };
    const lps::SolveReport r = lps::two_phase_solve(lp, rc);

    std::vector<int> basic;
    lpsg::SolverConfig gc;
    // the shim's observer reports the changed row and both variables; rebuild the
    // same basis checksum as above from them
    {
        lps::SolverConfig c0;
        lps::SimplexSolver probe(lp, c0);
        basic = probe.basis().basic;
    }
    gc.observer = [&](const lpsg::IterationView& v) {
        basic[v.row] = v.entering;
        long sum = 0;
        for (int b : basic) sum = sum * 1000003 + b;
        gpu_tr.push_back({v.iteration, v.phase, (int)(sum & 0x7fffffff), v.objective});
    };
    lpsg::SolveReport q;
    try {
        q = lpsg::two_phase_solve<lps::StandardFormLP, lps::PivotTooSmall, lps::Error>(lp, gc);
    } catch (const lps::Error& e) {
        std::printf("FAIL lpsg error: %s\n", e.what());
        return 1;
    }
    bool ok = int(q.status) == int(r.status) && ref_tr.size() == gpu_tr.size() &&
              q.iterations_phase1 == r.iterations_phase1 && q.iterations_phase2 == r.iterations_phase2;
    for (size_t k = 0; ok && k < ref_tr.size(); ++k)
        ok = ref_tr[k].it == gpu_tr[k].it && ref_tr[k].phase == gpu_tr[k].phase &&
             ref_tr[k].entering == gpu_tr[k].entering &&
             std::memcmp(&ref_tr[k].obj, &gpu_tr[k].obj, sizeof(double)) == 0;
    ok = ok && (std::memcmp(&q.objective, &r.objective, sizeof(double)) == 0 ||
                (q.objective != q.objective && r.objective != r.objective));
    ok = ok && q.x.size() == r.x.size() &&
         std::memcmp(q.x.data(), r.x.data(), sizeof(double) * r.x.size()) == 0;
    std::printf("%s %dx%d form %d seed %llu: %zu pivots, status %d, objective %.17g (ref %.17g), "
                "ref %.3f s, lpsg %.3f s\n",
                ok ? "PASS" : "FAIL", rows, cols, form, seed, gpu_tr.size(), int(q.status), q.objective,
                r.objective, r.total_seconds, q.total_seconds);
    return ok ? 0 : 1;
}
