"""Full-size golden fixtures from the compiled, unmodified reference (oracle/_ref),
for tests/test_gpu_large.py. Run in the build container (needs /root/reference):

    make -C oracle ref && python tests/make_large_golden.py [name ...]

Each fixture stores the generator spec + SHA-256 of the reference's arrays, the
reference's report and its full per-pivot trace (see tests/make_golden.py).
These are BASELINE.json configs at their real sizes:
  c2_full      C2 m=2000 n=4000 equality form, solved to optimality (~21.6k pivots)
  c3_p200      C3 m=8000 n=16000 equality form, first 200 pivots
  c4_p3        C4 m=4000 n=8000 degenerate form, first 3 pivots (each a ~1000-way
               ratio tie resolved by the tabu lookahead; ~10 min of reference time)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from make_golden import lp_digest  # noqa: E402
from oracle.oracle import Ref, make_config  # noqa: E402

import numpy as np  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "large")
CASES = {
    "c2_full": (2000, 4000, 0, 1, {"workers": 4}),
    "c3_p200": (8000, 16000, 0, 1, {"max_iter": 200, "workers": 4}),
    "c4_p3": (4000, 8000, 2, 1, {"max_iter": 3, "workers": 1}),
    "c5_p10": (24000, 48000, 0, 1, {"max_iter": 10, "workers": 8}),
    "c4_p20": (4000, 8000, 2, 1, {"max_iter": 20, "workers": 1}),
    "c5_p100": (24000, 48000, 0, 1, {"max_iter": 100, "workers": 8}),
    "c4_p60": (4000, 8000, 2, 1, {"max_iter": 60, "workers": 1}),
}


def main(names):
    os.makedirs(OUT, exist_ok=True)
    ref = Ref()
    for name in names or CASES:
        rows, cols, form, seed, over = CASES[name]
        lp = ref.generate(rows, cols, seed, form)
        out = ref.solve(lp, make_config(**over), trace_cap=200000)
        np.savez_compressed(
            os.path.join(OUT, name + ".npz"), spec=np.array([rows, cols, form, seed, 0], np.int64),
            m=lp.m, n_total=lp.n_total, digest=lp_digest(lp), status=out.status,
            objective=out.objective, x=out.x, iterations_phase1=out.iterations_phase1,
            iterations_phase2=out.iterations_phase2, trace=out.trace, trace_len=out.trace_len,
            cfg_max_iter=over.get("max_iter", 0), cfg_anticycle=0, cfg_pivot_tol=1e-9,
            ref_seconds=out.total_seconds, ref_workers=over.get("workers", 1))
        print(name, out.status_name, out.objective, out.iterations_phase1, out.iterations_phase2,
              round(out.total_seconds, 2), "s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
