import time, numpy as np, sys
sys.path.insert(0, '.')
import paper_1803_04378_b200 as P
lp = P.generate(P.GenSpec(8000, 16000, seed=1), pinned=True)
for every in (50000, 25000):
    t0 = time.perf_counter()
    with P.SimplexSolver(lp, P.SolverConfig(reinvert_every=every)) as s:
        rep = s.solve()
        st = s.reinvert_stats()
    t1 = time.perf_counter()
    x = rep.x
    res = np.abs(lp.A @ x - lp.b).max() / np.abs(lp.b).max()
    print(every, rep.status.name, repr(rep.objective), rep.iterations_phase1, rep.iterations_phase2, round(t1 - t0, 2), res, st, flush=True)
