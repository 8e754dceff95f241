"""Full C4 solve (BASELINE configs[3]: degenerate m=4000 n=8000, seed 1) in
parity mode: status, pivots, objective, seconds, and how the lookaheads were
settled. python tools/dbg/c4_full_solve.py [max_iter]"""
import json
import sys
import time

sys.path.insert(0, ".")
import paper_1803_04378_b200 as P

mi = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lp = P.generate(P.GenSpec(4000, 8000, P.SparsityClass.dense, 1, P.Form.degenerate), pinned=True)
t0 = time.perf_counter()
with P.SimplexSolver(lp, P.SolverConfig(max_iter=mi)) as s:
    t1 = time.perf_counter()
    rep = s.solve()
    t2 = time.perf_counter()
    st = s.lookahead_stats()
print(json.dumps(dict(status=rep.status.name, p1=rep.iterations_phase1, p2=rep.iterations_phase2,
                      objective=rep.objective, create_s=t1 - t0, solve_s=t2 - t1,
                      it_per_s=(rep.iterations_phase1 + rep.iterations_phase2) / (t2 - t1), lookahead=st)))
