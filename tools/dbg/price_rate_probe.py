"""k_price / k_update rates with the experiment bits: 0 = production, 1 = no
math in k_price (memory-only), 2 = no loads in k_price (compute-only), 4 = no
update/FTRAN math, 8 = no update loads. Timing only (bits != 0 give invalid
pivots). Usage: PYTHONPATH=. python tools/dbg/price_rate_probe.py [m] [bits,bits,...]"""
import sys
import paper_1803_04378_b200 as P


def _xcfg(cfg, exp):
    cfg._experiment = exp  # knobs live only in the LPSG_EXPERIMENTS_LIB=1 build
    return cfg


m = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
lp = P.generate(P.GenSpec(m, 2 * m, seed=1))
for exp in [int(v) for v in (sys.argv[2].split(',') if len(sys.argv) > 2 else ['0', '1', '2', '4', '8'])]:
    s = P.SimplexSolver(lp, _xcfg(P.SolverConfig(max_iter=20), exp))
    s.solve()
    s.set_max_iter(220)
    s.profile(True)
    rep = s.solve()
    st = s.profile_stats()
    s.close()
    print(exp, rep.iterations, {k: round(1e3 * v["ms"] / v["launches"], 2)
                                for k, v in st.items() if v["launches"] and v["ms"] > 0}, flush=True)
