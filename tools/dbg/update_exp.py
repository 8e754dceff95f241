import sys
sys.path.insert(0, '.')
import paper_1803_04378_b200 as P


def _xcfg(cfg, exp):
    cfg._experiment = exp  # knobs live only in the LPSG_EXPERIMENTS_LIB=1 build
    return cfg

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
lp = P.generate(P.GenSpec(m, 2 * m, seed=1))
for exp in (0, 4, 8, 5, 10):
    s = P.SimplexSolver(lp, _xcfg(P.SolverConfig(max_iter=10), exp))
    s.solve(); s.set_max_iter(60); s.profile(True); s.solve()
    st = s.profile_stats(); s.close()
    print(m, 'exp', exp, {k: round(1e3 * v['ms'] / v['launches'], 1) for k, v in st.items() if v['launches']}, flush=True)
