import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1803_04378_b200 as P
m = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
it = int(sys.argv[2]) if len(sys.argv) > 2 else 3
lp = P.generate(P.GenSpec(m, 2 * m, seed=1, form=P.Form.degenerate))
with P.SimplexSolver(lp, P.SolverConfig(max_iter=it)) as s:
    s.keep_trace(True)
    t0 = time.time(); rep = s.solve(); t1 = time.time()
    tr = s.trace()
print(m, it, rep.status.name, 'wall', round(t1 - t0, 3), 'dev_ms', round(s.device_ms() if False else 0, 1))
for t in tr[:10]: print(tuple(t))
np.save('gpurun_out/c4_trace_%d_%d.npy' % (m, it), tr)
