"""GPU parity of Case 2, the out-of-core tiled path (
/root/reference/proj/src/tiled_engine.cpp:29-54 plan, 165-184 upload /
download, 246-263 resident-partition order).

A forced-small SolverConfig.memory_budget makes the (m+1) x (m+2) tableau
"not fit": its rows then live in page-locked host memory in the reference's
row partitions and stream through one device slab per pivot. The arithmetic
is unchanged, so every golden trace must be reproduced bit for bit, with
report.case_used == "Tiled" and the partition traffic visible in the memory
counters.
"""
import numpy as np
import pytest

from conftest import Golden

pytestmark = pytest.mark.gpu


def _P():
    import paper_1803_04378_b200 as P
    return P


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def _golden_lp(g):
    P = _P()
    if g.spec is not None:
        rows, cols, form, seed, sp = g.spec
        return P.generate(P.GenSpec(rows, cols, P.SparsityClass(sp), seed, P.Form(form)))
    A, b, c, ck = g.arrays()
    return P.StandardFormLP(g.m, g.n_total, A, b, c, ck)


def budget_for(m, parts):
    """A memory_budget whose plan (tiled_engine.cpp:29-54) gives about `parts` partitions."""
    row_bytes = 8 * (m + 2)
    rpp = max(1, -(-(m + 1) // parts))
    return row_bytes * (rpp + 1)


def _run(g, budget, **kw):
    P = _P()
    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle), memory_budget=budget, **kw)
    with P.SimplexSolver(_golden_lp(g), cfg) as s:
        s.keep_trace(True)
        rep = s.solve()
        tr = s.trace()
        mem = s.memory()
    return rep, tr, mem


def _check(rep, tr, g, tag):
    ref = g.trace[: g.trace_len]
    assert int(rep.status) == g.status, (tag, rep.status, g.status)
    assert (rep.iterations_phase1, rep.iterations_phase2) == (g.p1, g.p2), tag
    assert len(tr) == len(ref), tag
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        assert np.array_equal(tr[f], ref[f]), (tag, f)
    assert np.array_equal(_bits(tr["objective"]), _bits(ref["objective"])), tag
    if np.isnan(g.objective):
        assert np.isnan(rep.objective)
    else:
        assert _bits(rep.objective) == _bits(g.objective), tag
    assert np.array_equal(_bits(rep.x), _bits(g.x)), tag


NAMES = ["gen_64x128_f0_s2", "gen_96x160_f1_s4", "gen_128x256_f2_s5", "gen_256x512_f0_s1",
         "gen_256x512_f2_s1", "gen_256x512_f2_s1_naive", "beale_3x7", "netlib_afiro", "netlib_scsd1",
         "netlib_sctap1", "driveout_64x96_many", "driveout_30x60_sum", "infeasible_2x2",
         "unbounded_1x3", "gen_2000x4000_f0_s1_max_iter200"]


@pytest.mark.parametrize("parts", [2, 5])
@pytest.mark.parametrize("name", NAMES)
def test_tiled_reproduces_golden(name, parts):
    g = Golden(name)
    if g.m + 1 < 2 * parts:
        pytest.skip("too few rows for this many partitions")
    budget = budget_for(g.m, parts)
    rep, tr, mem = _run(g, budget)
    assert rep.case_used == "Tiled", name
    _check(rep, tr, g, (name, parts))
    # every pivot moved partition payload both ways (host <-> device)
    assert mem["h2d_bytes"] > 8 * g.m * g.m and mem["d2h_bytes"] > 8 * g.m * g.m


@pytest.mark.parametrize("name", ["gen_128x256_f2_s5", "gen_256x512_f2_s1", "beale_3x7", "netlib_scsd1",
                                  "netlib_sctap1"])
def test_tiled_bounded_pricing_always(name):
    """Case 2 with the bounded pricing on every tie (the
    bounded selection itself is in-core only, so ties fall back to full
    scoring per partition): still the reference's traces, bit for bit."""
    g = Golden(name)
    if g.m + 1 < 6:
        pytest.skip("too few rows for 3 partitions")
    rep, tr, _ = _run(g, budget_for(g.m, 3), lookahead_bound="always")
    assert rep.case_used == "Tiled", name
    _check(rep, tr, g, (name, "always"))


def test_in_core_when_the_budget_fits():
    P = _P()
    g = Golden("gen_64x128_f0_s2")
    rep, tr, _ = _run(g, 8 * (g.m + 1) * (g.m + 2))
    assert rep.case_used == "InCore"
    _check(rep, tr, g, "in-core")


def test_budget_too_small_is_the_reference_error():
    """plan() needs two tableau rows (tiled_engine.cpp:43-47), same message."""
    P = _P()
    lp = P.generate(P.GenSpec(20, 40, seed=1))
    row = 8 * (lp.m + 2)
    with pytest.raises(P.BudgetTooSmall) as e:
        P.SimplexSolver(lp, P.SolverConfig(memory_budget=row + 7))
    assert str(e.value) == (f"device budget of {row + 7} bytes cannot hold one data row plus the "
                            f"pivot row (row is {row} bytes)")


def test_tiled_observer_rows_match_in_core():
    """IterationView rows read through the partitions (host or slab) equal the in-core ones."""
    P = _P()
    g = Golden("gen_96x160_f1_s4")
    out = {}
    for budget in (0, budget_for(g.m, 4)):
        seen = []

        def obs(v):
            seen.append(np.concatenate([v.tableau_row(i) for i in (0, 1, g.m // 2, g.m)]))

        cfg = P.SolverConfig(observer=obs, observer_rows=True, memory_budget=budget)
        with P.SimplexSolver(_golden_lp(g), cfg) as s:
            s.solve()
        out[budget] = np.array(seen)
    a, b = out.values()
    assert a.shape == b.shape and np.array_equal(_bits(a), _bits(b))


def test_tiled_rejects_step_api_and_reinversion():
    P = _P()
    g = Golden("gen_64x128_f0_s2")
    lp = _golden_lp(g)
    with P.SimplexSolver(lp, P.SolverConfig(memory_budget=budget_for(g.m, 3))) as s:
        with pytest.raises(P.Error, match="in-core"):
            s.price()
    with pytest.raises(P.Error, match="reinversion"):
        P.SimplexSolver(lp, P.SolverConfig(memory_budget=budget_for(g.m, 3), reinvert_every=10))
