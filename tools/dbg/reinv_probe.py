"""Reinversion-mode probe on one B200: GEMM rate of one rebuild, C2 / SCSD1 /
C3 solves with periodic reinversion (status, objective, residuals, time).
PYTHONPATH=. python tools/dbg/reinv_probe.py [c3]"""
import sys
import time

import numpy as np

import paper_1803_04378_b200 as P


def report(tag, lp, rep, s, t):
    x = rep.x
    res = np.abs(lp.A @ x - lp.b).max() / max(1e-300, np.abs(lp.b).max()) if rep.status == 0 else None
    cx = float(lp.c @ x)
    print(tag, rep.status.name, repr(rep.objective), "p1", rep.iterations_phase1, "p2", rep.iterations_phase2,
          "res", res, "cx-obj", (cx - rep.objective) / max(1.0, abs(rep.objective)),
          "xmin", float(x.min()), "wall", round(t, 3), s.reinvert_stats(), flush=True)


def run(tag, lp, every, **kw):
    t0 = time.perf_counter()
    with P.SimplexSolver(lp, P.SolverConfig(reinvert_every=every, **kw)) as s:
        rep = s.solve()
        report(tag, lp, rep, s, time.perf_counter() - t0)
    return rep


lp3 = P.generate(P.GenSpec(8000, 16000, seed=1))
with P.SimplexSolver(lp3, P.SolverConfig(reinvert_every=100, max_iter=101)) as s:
    s.solve()
    st = s.reinvert_stats()
    gf = 2.0 * 8000 ** 3 * (2 * st["steps"] + 1) / 1e9
    print("c3 rebuild after 100 pivots", st, "GEMM TFLOP/s ~", round(gf / st["seconds"] / 1e3, 2), flush=True)

lp2 = P.generate(P.GenSpec(2000, 4000, seed=1))
base = P.two_phase_solve(lp2)
print("c2 parity", base.status.name, repr(base.objective), base.iterations, flush=True)
for every in (500, 2000, 5000):
    r = run(f"c2 reinv {every}", lp2, every)
    print("  rel diff vs parity objective", abs(r.objective - base.objective) / abs(base.objective))
z = np.load("tests/golden/netlib_scsd1.npz")
A = np.zeros((int(z["m"]), int(z["n_total"])))
A[z["A_rows"], z["A_cols"]] = z["A_vals"]
lps = P.StandardFormLP(int(z["m"]), int(z["n_total"]), A, z["b"], z["c"], z["col_kind"])
print("scsd1 parity", P.two_phase_solve(lps).status.name, "(reference: Unbounded; Netlib optimum 8.6666667)")
for every in (100, 400):
    run(f"scsd1 reinv {every}", lps, every)
if "c3" in sys.argv[1:]:
    for every in (5000, 2000):
        run(f"c3 reinv {every}", lp3, every)
