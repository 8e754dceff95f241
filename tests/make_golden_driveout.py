"""Golden fixtures for drive_out_artificials (solver.cpp:295-316), made by the
compiled reference: equality LPs with redundant rows, so phase 1 ends with
artificial variables basic at level zero. Run in the build container:

    make -C oracle ref && python tests/make_golden_driveout.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from make_golden import save  # noqa: E402
from oracle.oracle import LP, Ref, make_config  # noqa: E402


def redundant(m, n, seed, combos, signed=False):
    """Random equality LP (A x = b with a feasible x_hat >= 0) whose rows listed
    in `combos` are linear combinations of other rows (b consistent)."""
    rng = np.random.default_rng(seed)
    A = rng.uniform(-1.0, 1.0, (m, n)) if signed else rng.uniform(0.01, 1.0, (m, n))
    for r, terms in combos.items():
        A[r] = sum(w * A[k] for k, w in terms)
    xh = rng.uniform(0.0, 1.0, n)
    b = A @ xh
    neg = b < 0
    A[neg] *= -1.0
    b[neg] *= -1.0
    c = rng.uniform(0.0, 1.0, n) if not signed else rng.uniform(-1.0, 1.0, n)
    return LP(m, n, A, b, c, np.zeros(n, np.uint8))


CASES = {
    "driveout_30x60_sum": (30, 60, 11, {29: [(0, 1.0), (1, 1.0)]}, False),
    "driveout_40x80_two": (40, 80, 12, {38: [(0, 1.0), (1, 1.0)], 39: [(5, 2.0)]}, False),
    "driveout_24x50_signed": (24, 50, 13, {23: [(2, 1.0), (3, -1.0)], 22: [(7, 0.5)]}, True),
    "driveout_64x96_many": (64, 96, 14, {60: [(0, 1.0)], 61: [(1, 1.0), (2, 1.0)],
                                          62: [(3, 2.0), (4, -1.0)], 63: [(5, 1.0), (6, 1.0), (7, 1.0)]},
                            True),
}


def main():
    ref = Ref()
    for name, (m, n, seed, combos, signed) in CASES.items():
        lp = redundant(m, n, seed, combos, signed)
        out = ref.solve(lp, make_config())
        save(name, lp, out, {})
        print(name, out.status_name, out.objective, out.iterations_phase1, out.iterations_phase2)


if __name__ == "__main__":
    main()
