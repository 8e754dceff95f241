"""GPU tests of the opt-in periodic reinversion mode (north_star item 5,
include/lpsg.h lpsg_config.reinvert_every; csrc/reinvert.cu).

This mode deliberately leaves the reference's arithmetic (the reference never
re-factorises, solver.cpp:240-254), so it is checked against the LP itself,
not against golden traces:
  * feasibility max|A x - b| / max|b| <= 1e-9, x >= 0,
  * the reported objective equals c.x to 1e-9 relative,
  * where the parity path reaches the same optimum (C2), the objectives agree
    to 1e-9 relative; where the reference fails from inverse drift (Netlib
    SCSD1 "Unbounded", C3 "Infeasible" at pivot 67 548), reinversion reaches
    the true optimum (SCSD1: 8.6666667, Netlib / PAPER.md:456).
"""
import os

import numpy as np
import pytest

from conftest import Golden

pytestmark = pytest.mark.gpu


def _P():
    import paper_1803_04378_b200 as P
    return P


def _check_point(lp, rep, tol=1e-9):
    x = rep.x
    assert (x >= -1e-12).all(), float(x.min())
    res = np.abs(lp.A @ x - lp.b).max() / np.abs(lp.b).max()
    assert res <= tol, res
    cx = float(lp.c @ x)
    assert abs(cx - rep.objective) <= tol * max(1.0, abs(rep.objective)), (cx, rep.objective)


def test_reinversion_c2_matches_parity_optimum():
    P = _P()
    lp = P.generate(P.GenSpec(2000, 4000, seed=1))
    base = P.two_phase_solve(lp)
    assert base.status == P.SolveStatus.optimal
    with P.SimplexSolver(lp, P.SolverConfig(reinvert_every=2000)) as s:
        rep = s.solve()
        st = s.reinvert_stats()
    assert rep.status == P.SolveStatus.optimal
    assert abs(rep.objective - base.objective) <= 1e-9 * abs(base.objective)
    _check_point(lp, rep)
    assert st["rebuilds"] >= 10 and st["steps"] >= st["rebuilds"]
    assert st["residual_after"] < 1e-12, st


def test_reinversion_fixes_scsd1():
    """The reference returns Unbounded on SCSD1 with default tolerances
    (SURVEY.md §0.7); with reinversion the solve reaches the Netlib optimum."""
    P = _P()
    g = Golden("netlib_scsd1")
    A, b, c, ck = g.arrays()
    lp = P.StandardFormLP(g.m, g.n_total, A, b, c, ck)
    assert P.two_phase_solve(lp).status == P.SolveStatus.unbounded  # parity mode, like the reference
    rep = P.two_phase_solve(lp, P.SolverConfig(reinvert_every=100))
    assert rep.status == P.SolveStatus.optimal
    z = float(g.z["objective_sign"]) * rep.objective + float(g.z["objective_constant"])
    assert abs(z - 8.6666667) <= 1e-7, z
    _check_point(lp, rep)


@pytest.mark.parametrize("every", [50, 400])
def test_reinversion_generated_forms(every):
    P = _P()
    for form in (0, 1, 2):
        lp = P.generate(P.GenSpec(300, 500, seed=11 + form, form=P.Form(form)))
        base = P.two_phase_solve(lp)
        rep = P.two_phase_solve(lp, P.SolverConfig(reinvert_every=every))
        assert rep.status == base.status == P.SolveStatus.optimal, form
        assert abs(rep.objective - base.objective) <= 1e-9 * max(1.0, abs(base.objective)), form
        _check_point(lp, rep)


def test_reinversion_newton_converges_from_a_perturbed_inverse():
    """A rebuild right after a handful of pivots must leave max|I - B X| at
    rounding level even when it has to take a full Newton step."""
    P = _P()
    lp = P.generate(P.GenSpec(1000, 2000, seed=3))
    with P.SimplexSolver(lp, P.SolverConfig(reinvert_every=7, max_iter=50)) as s:
        rep = s.solve()
        st = s.reinvert_stats()
    assert rep.iterations == 50 and st["rebuilds"] >= 6
    assert st["steps"] >= st["rebuilds"] and st["residual_after"] < 1e-12, st


def test_reinversion_is_single_gpu_only():
    P = _P()
    lp = P.generate(P.GenSpec(64, 128, seed=2))
    with pytest.raises(P.Error, match="single-GPU"):
        P.solve_sharded(lp, P.SolverConfig(reinvert_every=10), shards=2)


@pytest.mark.skipif(os.environ.get("LPSG_SKIP_SLOW") == "1", reason="slow (C3 full solve, ~50 s)")
def test_reinversion_c3_reaches_optimal():
    """C3 (the headline config): the parity path ends Infeasible after 67 548
    phase-1 pivots, exactly like the reference; with reinversion the solve
    passes the phase-1 test and reaches the optimum."""
    P = _P()
    lp = P.generate(P.GenSpec(8000, 16000, seed=1))
    with P.SimplexSolver(lp, P.SolverConfig(reinvert_every=10000)) as s:
        rep = s.solve()
        st = s.reinvert_stats()
    assert rep.status == P.SolveStatus.optimal, rep.status
    assert rep.iterations_phase1 == 67548
    _check_point(lp, rep)
    # |B X 1 - 1| after the last rebuild: the two m = 8000 GEMVs of the probe
    # alone round at ~1e-12 (m eps |B| |X 1|)
    assert st["residual_after"] < 1e-10, st


def test_reinversion_with_observer_rows():
    """The unfused one-pivot-per-round-trip schedule (observer_rows) takes the
    same reinversion stops: SCSD1 still reaches the Netlib optimum, and the
    view's row 0 objective equals the report at the end."""
    P = _P()
    g = Golden("netlib_scsd1")
    A, b, c, ck = g.arrays()
    lp = P.StandardFormLP(g.m, g.n_total, A, b, c, ck)
    seen = []
    cfg = P.SolverConfig(reinvert_every=100, observer=lambda v: seen.append(v.tableau_row(0)[g.m]),
                         observer_rows=True)
    with P.SimplexSolver(lp, cfg) as s:
        rep = s.solve()
        st = s.reinvert_stats()
    assert rep.status == P.SolveStatus.optimal and st["rebuilds"] >= 2
    z = float(g.z["objective_sign"]) * rep.objective + float(g.z["objective_constant"])
    assert abs(z - 8.6666667) <= 1e-7, z
    assert len(seen) == rep.iterations
    _check_point(lp, rep)


# Published optima (PAPER.md "specifications of the Netlib benchmark" table;
# afiro / boeing2 / kb2, not in that table, are the Netlib library's values).
NETLIB_OPT = {"afiro": -464.7531429, "boeing2": -315.0187280, "kb2": -1749.900130,
              "recipe": -266.616, "e226": -18.751929, "lotfi": -25.264706, "grow7": -47787812,
              "scsd1": 8.666667, "sctap1": 1412.25, "scsd6": 50.5, "ship04s": 1798714.7}


@pytest.mark.parametrize("name", sorted(NETLIB_OPT))
def test_reinversion_netlib_reaches_published_optima(name):
    """Every shipped Netlib file in reinversion mode: Optimal at the published
    optimum (to the table's printed digits), feasible, and -- where the
    reference itself solves it (all but SCSD1) -- within 1e-9 relative of the
    reference's objective."""
    P = _P()
    g = Golden("netlib_" + name)
    A, b, c, ck = g.arrays()
    lp = P.StandardFormLP(g.m, g.n_total, A, b, c, ck)
    rep = P.two_phase_solve(lp, P.SolverConfig(reinvert_every=200))
    assert rep.status == P.SolveStatus.optimal, (name, rep.status)
    sign, const = float(g.z["objective_sign"]), float(g.z["objective_constant"])
    z = sign * rep.objective + const
    want = NETLIB_OPT[name]
    assert abs(z - want) <= 5e-7 * max(1.0, abs(want)), (name, z, want)
    _check_point(lp, rep, tol=1e-8)
    if g.status == 0:
        zr = sign * g.objective + const
        assert abs(z - zr) <= 1e-9 * max(1.0, abs(zr)), (name, z, zr)
