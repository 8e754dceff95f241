#!/usr/bin/env python
"""TEST INFRASTRUCTURE: runs the compiled, unmodified reference (oracle/_ref) on a
large generated LP for a long pivot prefix (or to the end) and stores its
per-pivot trace + report, so a full-size GPU solve can be compared pivot for
pivot (tests/golden/long_*.npz, tests/test_gpu_long.py).

    python tools/ref_long_trace.py ROWS COLS FORM SEED MAX_ITER WORKERS OUT.npz
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Ref, make_config  # noqa: E402


def main():
    rows, cols, form, seed, max_iter, workers = map(int, sys.argv[1:7])
    out = sys.argv[7]
    ref = Ref()
    lp = ref.generate(rows, cols, seed=seed, form=form)
    t0 = time.time()
    res = ref.solve(lp, make_config(max_iter=max_iter, workers=workers), trace_cap=max_iter + 10)
    np.savez_compressed(out, spec=np.array([rows, cols, form, seed, 0]), m=lp.m, n_total=lp.n_total,
                        status=res.status, objective=res.objective, x=res.x,
                        iterations_phase1=res.iterations_phase1,
                        iterations_phase2=res.iterations_phase2, trace=res.trace,
                        trace_len=res.trace_len, cfg_max_iter=max_iter, wall_s=time.time() - t0,
                        total_seconds=res.total_seconds, workers=workers)
    print("done", res.status, res.objective, res.iterations_phase1, res.iterations_phase2,
          time.time() - t0, flush=True)


if __name__ == "__main__":
    main()
