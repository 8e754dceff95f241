"""Generates the MPS-ingestion fixtures from the compiled, unmodified reference.

Run in the build container (needs oracle/_ref, i.e. /root/reference):

    make -C oracle ref && python tests/make_golden_mps.py

For every tests/golden/mps/*.mps (synthetic files written for these tests) it
stores what lps::parse_mps + to_general_lp + canonicalize produce
(mps.cpp, lp_model.cpp): the standard form, the CanonicalMap, the warnings and
write_mps(doc); for the optimal ones also the reference's two_phase_solve
report and recover_solution. tests/mps_cases.py's small texts go to
cases.json (error kind and message, or the standard-form digest), and
write_mps(to_mps_document(generate(...))) of two generated instances to
generated_*.mps.txt.
"""
from __future__ import annotations

import glob
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from mps_cases import CASES  # noqa: E402
from oracle.oracle import Ref, make_config  # noqa: E402

DIR = os.path.join(ROOT, "tests", "golden", "mps")
GENERATED = [(6, 9, 3, 0, 2), (5, 7, 2, 1, 0)]  # rows, cols, seed, form, sparsity


def digest(lp) -> str:
    h = hashlib.sha256()
    for a in (lp.A, lp.b, lp.c, lp.col_kind):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.float64([lp.objective_sign, lp.objective_constant]).tobytes())
    return h.hexdigest()


def main() -> None:
    ref = Ref()
    for path in sorted(glob.glob(os.path.join(DIR, "*.mps"))):
        name = os.path.splitext(os.path.basename(path))[0]
        out = ref.mps_load(open(path, "rb").read())
        lp = out["lp"]
        d = dict(A=lp.A, b=lp.b, c=lp.c, col_kind=lp.col_kind, objective_sign=lp.objective_sign,
                 objective_constant=lp.objective_constant, shift=out["shift"],
                 negated_row=out["negated_row"], split_pos=out["split_pos"],
                 split_neg=out["split_neg"], warnings=out["warnings"], written=out["written"])
        s = ref.solve(lp, make_config())
        d.update(status=s.status, objective=s.objective, x=s.x,
                 iterations_phase1=s.iterations_phase1, iterations_phase2=s.iterations_phase2)
        if s.status in (0, 3):
            xr, zr = ref.mps_recover(out, s.x, s.objective)
            d.update(x_recovered=xr, objective_recovered=zr)
        ref.mps_free(out)
        np.savez_compressed(os.path.join(DIR, name + ".npz"), **d)
        print(name, lp.m, lp.n_total, s.status_name, s.objective)
    cases = {}
    for name, text in CASES.items():
        out = ref.mps_load(text)
        if "error_kind" in out:
            cases[name] = {"error_kind": out["error_kind"], "error": out["error"]}
        else:
            cases[name] = {"digest": digest(out["lp"]), "warnings": out["warnings"],
                           "written": out["written"], "m": out["lp"].m,
                           "n_total": out["lp"].n_total}
            ref.mps_free(out)
        print(name, cases[name].get("error_kind", "ok"))
    with open(os.path.join(DIR, "cases.json"), "w") as f:
        json.dump(cases, f, indent=1, sort_keys=True)
    for rows, cols, seed, form, sp in GENERATED:
        t = ref.generated_mps(rows, cols, seed, form, sp)
        with open(os.path.join(DIR, f"generated_{rows}x{cols}_s{seed}_f{form}_sp{sp}.mps.txt"), "w") as f:
            f.write(t)


if __name__ == "__main__":
    main()
