import sys, numpy as np
sys.path.insert(0, '.')
import paper_1803_04378_b200 as P
def run(m, n, shards, batch=0, it=12, form=0):
    lp = P.generate(P.GenSpec(m, n, seed=1, form=P.Form(form)))
    cfg = P.SolverConfig(max_iter=it, batch=batch)
    with P.SimplexSolver(lp, cfg) as s:
        s.keep_trace(True); r1 = s.solve(); t1 = s.trace()
    r2, t2 = P.solve_sharded(lp, cfg, shards=shards, trace=True)
    bad = [k for k in range(min(len(t1), len(t2))) if tuple(t1[k])[2:5] != tuple(t2[k])[2:5] or t1[k]['objective'] != t2[k]['objective']]
    print(m, n, shards, batch, 'first bad', bad[:1], flush=True)
    if bad:
        k = bad[0]
        for kk in range(max(0, k - 2), min(len(t1), k + 3)):
            print('  1gpu', tuple(t1[kk]), '\n  shrd', tuple(t2[kk]))
for args in [(1000, 2000, 2), (2000, 4000, 2), (2000, 4000, 2, 1), (2000, 4000, 2, 64), (1500, 3000, 2), (1200, 2400, 2), (2000, 4000, 1), (4000, 8000, 2)]:
    try:
        run(*args)
    except Exception as e:
        print(args, 'ERR', e, flush=True)
