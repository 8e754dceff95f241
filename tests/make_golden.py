"""Generates tests/golden/*.npz from the compiled, unmodified reference.

Run in the build container (it needs /root/reference and oracle/_ref):

    make -C oracle && python tests/make_golden.py

Every fixture stores the standard-form LP (dense for generated instances is
replaced by its generator spec + a SHA-256 of the reference's arrays; Netlib
and hand-built LPs are stored sparse), the reference's SolveReport fields
(status, objective, x, per-phase iteration counts) and its per-pivot trace
(iteration, phase, leaving row, leaving variable, entering variable, objective)
as seen through SolverConfig::observer (oracle/ref_shim.cpp).
"""
from __future__ import annotations

import glob
import hashlib
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import LP, Ref, make_config  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
NETLIB = "/root/reference/proj/data/netlib"

# (rows, cols, form, seed, config overrides)
GENERATED = [
    (20, 40, 0, 1, {}), (20, 40, 1, 1, {}), (20, 40, 2, 1, {}),
    (64, 128, 0, 2, {}), (64, 128, 2, 3, {}), (96, 160, 1, 4, {}),
    (128, 256, 2, 5, {}), (128, 256, 2, 5, {"anticycle": "none"}),
    (256, 512, 1, 1, {}),            # C1 (le + maximize, slack start): 824 pivots
    (256, 512, 0, 1, {}),            # C1 verbatim equality form: 1202 pivots
    (256, 512, 0, 2, {}), (256, 512, 0, 3, {}),
    (256, 512, 2, 1, {}),            # degenerate recipe: 3106 pivots, tabu ties
    (256, 512, 2, 1, {"anticycle": "none"}),
    (256, 512, 0, 1, {"max_iter": 300}),
    (1000, 2000, 0, 1, {"max_iter": 400, "workers": 8}),
    (2000, 4000, 0, 1, {"max_iter": 200, "workers": 8}),   # C2 prefix
]


def lp_digest(lp: LP) -> str:
    h = hashlib.sha256()
    for a in (lp.A, lp.b, lp.c, lp.col_kind):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def save(name: str, lp: LP, out, cfg: dict, spec=None, sparse=True) -> None:
    d = dict(m=lp.m, n_total=lp.n_total, b=lp.b, c=lp.c, col_kind=lp.col_kind,
             objective_sign=lp.objective_sign, objective_constant=lp.objective_constant,
             status=out.status, objective=out.objective, x=out.x,
             iterations_phase1=out.iterations_phase1, iterations_phase2=out.iterations_phase2,
             trace=out.trace, trace_len=out.trace_len, digest=lp_digest(lp),
             cfg_max_iter=cfg.get("max_iter", 0),
             cfg_anticycle=1 if cfg.get("anticycle") == "none" else 0,
             cfg_pivot_tol=cfg.get("pivot_tol", 1e-9),
             cfg_kernel=1 if cfg.get("kernel") == "naive" else 0)
    if spec is not None:
        d["spec"] = np.array(spec, np.int64)
    else:
        r, c = np.nonzero(lp.A)
        d.update(A_rows=r.astype(np.int32), A_cols=c.astype(np.int32), A_vals=lp.A[r, c])
    np.savez_compressed(os.path.join(GOLDEN, name + ".npz"), **d)


# KernelMode::naive (tiled_engine.cpp:61-77): every element stored, no zero
# skip. On these inputs it changes the signs of zeros in x (BOEING2: 26, E226: 1).
NAIVE_NETLIB = ["boeing2", "e226"]


def naive_fixtures(ref) -> None:
    over = {"kernel": "naive"}
    for stem in NAIVE_NETLIB:
        lp = ref.from_mps(os.path.join(NETLIB, stem + ".mps"))
        out = ref.solve(lp, make_config(**over))
        save(f"netlib_{stem}_naive", lp, out, over)
        print(f"netlib_{stem}_naive", out.status_name, out.trace_len)
    lp = ref.generate(256, 512, 1, 2)
    out = ref.solve(lp, make_config(**over))
    save("gen_256x512_f2_s1_naive", lp, out, over, spec=(256, 512, 2, 1, 0))
    print("gen_256x512_f2_s1_naive", out.status_name, out.trace_len)


def main() -> None:
    os.makedirs(GOLDEN, exist_ok=True)
    ref = Ref()
    naive_fixtures(ref)
    if sys.argv[1:] == ["naive"]:
        return
    for rows, cols, form, seed, over in GENERATED:
        lp = ref.generate(rows, cols, seed, form)
        out = ref.solve(lp, make_config(**over))
        tag = "".join(f"_{k}{v}" for k, v in sorted(over.items()) if k != "workers")
        name = f"gen_{rows}x{cols}_f{form}_s{seed}{tag}"
        save(name, lp, out, over, spec=(rows, cols, form, seed, 0))
        print(name, out.status_name, out.objective, out.iterations_phase1,
              out.iterations_phase2)
    for path in sorted(glob.glob(os.path.join(NETLIB, "*.mps"))):
        lp = ref.from_mps(path)
        for over in ({}, {"pivot_tol": 1e-7}) if "scsd1" in path else ({},):
            out = ref.solve(lp, make_config(**over))
            tag = "_ptol1e-7" if over else ""
            name = "netlib_" + os.path.splitext(os.path.basename(path))[0] + tag
            save(name, lp, out, over)
            print(name, out.status_name, lp.objective_sign * out.objective + lp.objective_constant)
    # hand-built cases: SPEC.md two_phase_solve examples + Beale's cycling LP
    hand = {
        "infeasible_2x2": LP(2, 2, np.array([[1.0, 1.0], [1.0, 1.0]]), np.array([1.0, 3.0]),
                             np.array([1.0, 0.0]), np.zeros(2, np.uint8)),
        "unbounded_1x3": LP(1, 3, np.array([[-1.0, 1.0, 1.0]]), np.array([1.0]),
                            np.array([-1.0, 0.0, 0.0]), np.array([0, 0, 1], np.uint8)),
        "beale_3x7": LP(3, 7, np.array([[0.25, -8.0, -1.0, 9.0, 1.0, 0.0, 0.0],
                                        [0.5, -12.0, -0.5, 3.0, 0.0, 1.0, 0.0],
                                        [0.0, 0.0, 1.0, 0.0, 0.0, 0.0, 1.0]]),
                        np.array([0.0, 0.0, 1.0]), np.array([-0.75, 20.0, -0.5, 6.0, 0, 0, 0]),
                        np.array([0, 0, 0, 0, 1, 1, 1], np.uint8)),
    }
    for name, lp in hand.items():
        for over in ({}, {"anticycle": "none", "max_iter": 60}):
            out = ref.solve(lp, make_config(**over))
            tag = "_none" if over else ""
            save(name + tag, lp, out, over)
            print(name + tag, out.status_name, out.objective, out.trace_len)


if __name__ == "__main__":
    main()
