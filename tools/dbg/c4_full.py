import sys, time
sys.path.insert(0, '.')
import paper_1803_04378_b200 as P
it = int(sys.argv[1]) if len(sys.argv) > 1 else 0
lp = P.generate(P.GenSpec(4000, 8000, seed=1, form=P.Form.degenerate))
t0 = time.time()
with P.SimplexSolver(lp, P.SolverConfig(max_iter=it)) as s:
    rep = s.solve()
print('c4 full' if not it else f'c4 {it}', rep.status.name, rep.objective, rep.iterations_phase1, rep.iterations_phase2,
      round(time.time() - t0, 1), 's', flush=True)
