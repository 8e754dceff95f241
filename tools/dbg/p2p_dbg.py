import sys, os, faulthandler
faulthandler.dump_traceback_later(15, exit=True)
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_1803_04378_b200 as P
from conftest import Golden
name = sys.argv[1] if len(sys.argv) > 1 else 'beale_3x7'
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 2
g = Golden(name)
A, b, c, ck = g.arrays(lambda r, cc, s, f: P.generate(P.GenSpec(r, cc, seed=s, form=P.Form(f))))
lp = P.StandardFormLP(g.m, g.n_total, A, b, c, ck)
print('start', name, shards, flush=True)
batch = int(sys.argv[3]) if len(sys.argv) > 3 else 0
rep, tr = P.solve_sharded(lp, P.SolverConfig(max_iter=g.max_iter, batch=batch), shards=shards, trace=True, p2p=True)
print('done', rep.status, len(tr), g.trace_len, flush=True)
