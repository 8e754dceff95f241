"""Per-kernel times at an arbitrary (m, n) shape, e.g. the per-GPU shape of a
sharded C3 (m = 8000 rows, n/G pricing columns). Usage:
PYTHONPATH=. python tools/dbg/shape_probe.py m n [experiment]"""
import sys
import paper_1803_04378_b200 as P


def _xcfg(cfg, exp):
    cfg._experiment = exp  # knobs live only in the LPSG_EXPERIMENTS_LIB=1 build
    return cfg


m, n = int(sys.argv[1]), int(sys.argv[2])
exp = int(sys.argv[3]) if len(sys.argv) > 3 else 0
lp = P.generate(P.GenSpec(m, n, seed=1))
s = P.SimplexSolver(lp, _xcfg(P.SolverConfig(max_iter=20), exp))
s.solve()
s.set_max_iter(220)
s.profile(True)
rep = s.solve()
st = s.profile_stats()
s.close()
print(m, n, rep.iterations, {k: round(1e3 * v["ms"] / v["launches"], 2)
                             for k, v in st.items() if v["launches"] and v["ms"] > 0}, flush=True)
