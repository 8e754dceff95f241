// generator.cpp — input plumbing for the benchmark and tests (SURVEY.md §8(f)
// row 1 "lean LP ingestion"): lps::generate (generator.cpp:35-72) written
// straight into the standard form the solver consumes, for the input forms
// BASELINE.json's configs use, so no GeneralLP / PendingRow / cols_ copies of
// the dense matrix are made (lp_model.cpp:77-155 triple-copies it).
//
//   form 0: generator verbatim (every row eq, generator.cpp:47) -> A, b, c as drawn
//   form 1: rows le + maximize -> [A | I], c = -objective (lp_model.cpp:50,70-75,150-153)
//   form 2: form 1 with rows i = 0,2,4,.. (i+1 < m) replaced by a_i - a_{i+1}, b_i = 0
//           (the degenerate recipe of SURVEY.md §8(d), config C4)
//
// The draws are bit-identical to the reference: std::mt19937_64 is fixed by
// the C++ standard and the (0,1] mapping is generator.cpp:13-15.
#include <cstdint>
#include <cstring>
#include <random>
#include <vector>

#include "lpsg.h"

namespace {

double unit_open_closed(std::mt19937_64& rng) { return 1.0 - (rng() >> 11) * 0x1.0p-53; }

}  // namespace

extern "C" int lpsg_generated_n_total(int rows, int cols, int form) {
    return form == 0 ? cols : cols + rows;
}

extern "C" int lpsg_generate(int rows, int cols, int sparsity, uint64_t seed, int form, double* A,
                             double* b, double* c, uint8_t* col_kind) {
    if (rows <= 0 || cols <= 0) return LPSG_EMPTY_PROBLEM;
    if (!A || !b || !c || !col_kind || form < 0 || form > 2 || sparsity < 0 || sparsity > 2)
        return LPSG_INVALID_ARGUMENT;
    const int m = rows, n = cols;
    const int nt = lpsg_generated_n_total(rows, cols, form);
    const double p_zero = sparsity == 1 ? 0.2 : sparsity == 2 ? 0.6 : 0.0;
    std::mt19937_64 rng(seed);
    // Draw A directly into its standard-form rows (row pitch nt).
    for (int i = 0; i < m; ++i) {
        double* row = A + (size_t)i * nt;
        for (;;) {
            bool nonzero = false;
            for (int j = 0; j < n; ++j) {
                row[j] = 0.01 + 0.99 * unit_open_closed(rng);
                if (p_zero > 0.0 && unit_open_closed(rng) <= p_zero) row[j] = 0.0;
                else nonzero = true;
            }
            if (nonzero) break;
        }
    }
    std::vector<double> obj(n), xh(n);
    for (int j = 0; j < n; ++j) obj[j] = unit_open_closed(rng);
    for (int j = 0; j < n; ++j) xh[j] = unit_open_closed(rng);
    for (int i = 0; i < m; ++i) {
        const double* row = A + (size_t)i * nt;
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc += row[j] * xh[j];
        b[i] = acc;
    }
    if (form == 2) {
        for (int i = 0; i + 1 < m; i += 2) {
            double* ri = A + (size_t)i * nt;
            const double* rn = A + (size_t)(i + 1) * nt;
            for (int j = 0; j < n; ++j) ri[j] = ri[j] - rn[j];
            b[i] = 0.0;
        }
    }
    const double sign = form == 0 ? 1.0 : -1.0;
    if (form != 0)
        for (int i = 0; i < m; ++i) {
            double* row = A + (size_t)i * nt;
            std::memset(row + n, 0, sizeof(double) * m);
            row[n + i] = 1.0;
        }
    for (int j = 0; j < nt; ++j) {
        c[j] = j < n ? sign * obj[j] : 0.0;
        col_kind[j] = j < n ? LPSG_COL_STRUCTURAL : LPSG_COL_SLACK;
    }
    return LPSG_OK;
}
