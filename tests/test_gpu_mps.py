"""GPU parity of the MPS solve path (the reference CLI's `solve`, lps_main.cpp:110-118).

solve_mps = parse + to_general_lp + canonicalize (host, tests/test_mps.py)
-> two_phase_solve on the B200 -> recover_solution. Against the reference's
run on the same files (tests/golden/mps/*.npz, tests/make_golden_mps.py):
status, per-phase iterations, objective and x bit for bit, and the recovered
original-space x and objective.
"""
import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR

pytestmark = pytest.mark.gpu

MPS_DIR = os.path.join(GOLDEN_DIR, "mps")
FILES = sorted(os.path.splitext(os.path.basename(p))[0]
               for p in glob.glob(os.path.join(MPS_DIR, "*.mps")))


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("name", FILES)
def test_solve_mps_matches_reference(name):
    import paper_1803_04378_b200 as P
    z = np.load(os.path.join(MPS_DIR, name + ".npz"), allow_pickle=False)
    res = P.solve_mps(os.path.join(MPS_DIR, name + ".mps"))
    rep = res.report
    assert int(rep.status) == int(z["status"]), (name, rep.status)
    assert (rep.iterations_phase1, rep.iterations_phase2) == (int(z["iterations_phase1"]),
                                                              int(z["iterations_phase2"]))
    assert _bits([rep.objective])[0] == _bits([float(z["objective"])])[0] or (
        np.isnan(rep.objective) and np.isnan(float(z["objective"])))
    assert np.array_equal(_bits(rep.x), _bits(z["x"])), name
    if "x_recovered" in z.files:
        assert np.array_equal(_bits(res.x), _bits(z["x_recovered"])), name
        assert _bits([res.objective])[0] == _bits([float(z["objective_recovered"])])[0]


@pytest.mark.parametrize("name", FILES)
def test_solve_mps_pinned_upload(name):
    """canonicalize(pinned=True) builds A straight in page-locked memory; the
    solve is the same."""
    import paper_1803_04378_b200 as P
    z = np.load(os.path.join(MPS_DIR, name + ".npz"), allow_pickle=False)
    lp, _ = P.load_mps(os.path.join(MPS_DIR, name + ".mps"), pinned=True)
    rep = P.two_phase_solve(lp)
    assert int(rep.status) == int(z["status"])
    assert np.array_equal(_bits(rep.x), _bits(z["x"])), name
