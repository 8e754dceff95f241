"""Per-kernel GB/s at several m (k_update grid = ceil(m / h) CTAs): is the
update bound by the number of SMs it occupies? Usage: python tools/dbg/upd_sm_probe.py"""
import sys
import paper_1803_04378_b200 as P

for m in [int(v) for v in (sys.argv[1:] or ["8000", "8288", "7992", "8400"])]:
    lp = P.generate(P.GenSpec(m, 2 * m, seed=1))
    s = P.SimplexSolver(lp, P.SolverConfig(max_iter=20))
    s.solve()
    s.set_max_iter(220)
    s.profile(True)
    s.solve()
    st = s.profile_stats()
    s.close()
    print(m, {k: (round(1e3 * v["ms"] / v["launches"], 2), round(v["bytes"] / (v["ms"] / 1e3) / 1e9))
              for k, v in st.items() if v["launches"] and v["ms"] > 0 and v["bytes"]}, flush=True)
