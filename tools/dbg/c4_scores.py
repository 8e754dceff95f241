"""Score distribution of C4's lookahead ties: for a few pivot counts, re-price,
re-run the ratio test and score every tied candidate through the step API.
Decides whether bounding theta' (score <= z * partial theta') could skip work:
that needs most candidates' scores well below the tie's best.
    python tools/dbg/c4_scores.py [m] [pivots...]"""
import sys

import time

import numpy as np

sys.path.insert(0, ".")
import paper_1803_04378_b200 as P

m = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
its = [int(x) for x in sys.argv[2:]] or [1, 2, 5, 10, 20, 40]  # max_iter = 0 means the default cap, not zero
lp = P.generate(P.GenSpec(m, 2 * m, P.SparsityClass.dense, 1, P.Form.degenerate))
for it in its:
    t0 = time.time()
    with P.SimplexSolver(lp, P.SolverConfig(max_iter=it)) as s:
        rep = s.solve()
        print("solved", it, rep.status.name, round(time.time() - t0, 2), flush=True)
        pr = s.price()
        if pr.optimal:
            print(it, "optimal")
            continue
        s.compute_direction(pr.entering, pr.reduced_cost)
        ra = s.ratio_test()
        print("ratio", len(ra.candidates), round(time.time() - t0, 2), flush=True)
        rows = ra.candidates
        sc = s.lookahead_scores(rows, pr.entering)
        pos = sc[np.isfinite(sc) & (sc > 0)]
        print(f"it {it} q {pr.entering} theta {ra.theta:.3g} K {len(rows)} zero {(sc == 0).sum()} "
              f"neg {(sc < 0).sum()} pos {len(pos)} inf {np.isinf(sc).sum()} nan {np.isnan(sc).sum()} "
              f"max {sc.max():.6g} argmax {int(np.argmax(sc))} "
              f"pos-quantiles {np.quantile(pos, [0, .5, .9, 1]) if len(pos) else []}", flush=True)
