"""compute-sanitizer target: small tie-heavy solves through every lookahead
path (bounded pricing + probe with and without exact rounds, full scoring).
    compute-sanitizer --tool memcheck python tools/dbg/sanitize_bounded.py"""
import sys

import numpy as np

sys.path.insert(0, ".")
import paper_1803_04378_b200 as P

for mode in ("always", "off"):
    for rows, cols, seed in ((40, 70, 3), (96, 160, 5)):
        lp = P.generate(P.GenSpec(rows, cols, seed=seed, form=P.Form.degenerate))
        with P.SimplexSolver(lp, P.SolverConfig(lookahead_bound=mode, max_iter=400)) as s:
            rep = s.solve()
            print(mode, rows, rep.status.name, rep.iterations_phase1 + rep.iterations_phase2, s.lookahead_stats(),
                  flush=True)
