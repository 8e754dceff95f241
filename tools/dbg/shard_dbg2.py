import sys, os, numpy as np
sys.path.insert(0, '.')
import paper_1803_04378_b200 as P
lp = P.generate(P.GenSpec(2000, 4000, seed=1))
cfg = P.SolverConfig(max_iter=12)
with P.SimplexSolver(lp, cfg) as s:
    s.keep_trace(True); r1 = s.solve(); t1 = s.trace()
for rep in range(8):
    r2, t2 = P.solve_sharded(lp, cfg, shards=2, trace=True)
    bad = [k for k in range(min(len(t1), len(t2))) if t1[k]['objective'] != t2[k]['objective']]
    print(os.environ.get('LPSG_LOCAL_SYNC'), 'run', rep, 'first bad', bad[:1], flush=True)
