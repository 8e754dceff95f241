"""GPU parity tests: the CUDA solver reproduces the reference pivot for pivot.

Every call goes through the C ABI (include/lpsg.h) via the Python mirror of the
reference API. The checker is (a) the committed golden traces produced by the
compiled reference (tests/golden/, made by tests/make_golden.py) and (b) the
plain-C port (oracle/lps_oracle.c) on seeded inputs beyond the fixtures.

Bar: bit-exact. Entering/leaving sequence, leaving rows, per-pivot objective,
final status, objective and x are compared as raw fp64 bits (the north_star's
1e-9 relative tolerance is implied by bit equality).
"""
import numpy as np
import pytest

from conftest import Golden, golden_names

pytestmark = pytest.mark.gpu

NAMES = golden_names()


def _P():
    import paper_1803_04378_b200 as P
    return P


def _solve_traced(lp, **cfg):
    P = _P()
    with P.SimplexSolver(lp, P.SolverConfig(**cfg)) as s:
        s.keep_trace(True)
        rep = s.solve()
        tr = s.trace()
    return rep, tr


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


def _assert_trace(tr, ref, name):
    assert len(tr) == len(ref), (name, len(tr), len(ref))
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        bad = np.nonzero(tr[f] != ref[f])[0]
        assert bad.size == 0, (name, f, int(bad[0]) if bad.size else None)
    bad = np.nonzero(_bits(tr["objective"]) != _bits(ref["objective"]))[0]
    assert bad.size == 0, (name, "objective", int(bad[0]) if bad.size else None)


def _golden_lp(g):
    P = _P()
    if g.spec is not None:
        rows, cols, form, seed, sp = g.spec
        return P.generate(P.GenSpec(rows, cols, P.SparsityClass(sp), seed, P.Form(form)))
    A, b, c, ck = g.arrays()
    return P.StandardFormLP(g.m, g.n_total, A, b, c, ck)


@pytest.mark.parametrize("name", NAMES)
def test_golden_trace_parity(name):
    P = _P()
    g = Golden(name)
    lp = _golden_lp(g)
    rep, tr = _solve_traced(lp, max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                            anticycle=P.Anticycle(g.anticycle))
    assert int(rep.status) == g.status, (name, rep.status, g.status)
    assert (rep.iterations_phase1, rep.iterations_phase2) == (g.p1, g.p2), name
    _assert_trace(tr, g.trace[: g.trace_len], name)
    if np.isnan(g.objective):
        assert np.isnan(rep.objective)
    else:
        assert _bits(rep.objective) == _bits(g.objective), (name, rep.objective, g.objective)
    assert np.array_equal(_bits(rep.x), _bits(g.x)), name


TIE_NAMES = [n for n in NAMES if "_f2_" in n or n.startswith("beale")]


@pytest.mark.parametrize("name", TIE_NAMES)
def test_lookahead_exact_select_path(name):
    """The lookahead's theta kernel drops the y_i == 0 select when every X_kj
    is finite (a zero-sign-only difference). Forcing the select
    path (lookahead_exact_select) must give the same pivots, bit for bit."""
    P = _P()
    g = Golden(name)
    rep, tr = _solve_traced(_golden_lp(g), max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                            anticycle=P.Anticycle(g.anticycle), lookahead_exact_select=True)
    assert int(rep.status) == g.status
    _assert_trace(tr, g.trace[: g.trace_len], name)
    assert np.array_equal(_bits(rep.x), _bits(g.x)), name


@pytest.mark.parametrize("name", NAMES)
def test_bounded_selection_always_same_pivots(name):
    """select_leaving's bounded selection (a probe that proves every later
    survivor's score <= the first one's +-0) tried on EVERY tie
    of >= 2 survivors instead of from 16 up: the pivots, x and objective stay
    the reference's, bit for bit, whether the probe settles a tie or falls back
    to full scoring."""
    P = _P()
    g = Golden(name)
    with P.SimplexSolver(_golden_lp(g), P.SolverConfig(
            max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
            anticycle=P.Anticycle(g.anticycle), lookahead_bound="always")) as s:
        s.keep_trace(True)
        rep = s.solve()
        tr = s.trace()
        st = s.lookahead_stats()
    assert int(rep.status) == g.status, (name, rep.status, g.status)
    _assert_trace(tr, g.trace[: g.trace_len], name)
    assert np.array_equal(_bits(rep.x), _bits(g.x)), name
    if g.anticycle == int(P.Anticycle.none):
        assert not any(st.values()), (name, st)


def test_bounded_selection_both_branches_run():
    """Across the tie fixtures the probe both settles ties and falls back, the
    bounded pricing (DFMA screen + exact chains) settles pricings (so the test
    above exercises those branches), and "off" tries neither."""
    P = _P()
    tot = dict(bounded=0, full=0, price_bounded=0, price_exact=0, probe_rounds=0)
    for name in [n for n in NAMES if "_f2_" in n or n.startswith(("beale", "netlib"))]:
        g = Golden(name)
        for mode in ("always", "off"):
            with P.SimplexSolver(_golden_lp(g), P.SolverConfig(
                    max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                    anticycle=P.Anticycle(g.anticycle), lookahead_bound=mode)) as s:
                s.solve()
                st = s.lookahead_stats()
            if mode == "off":
                assert not any(v for k, v in st.items() if k != "full"), (name, st)
            else:
                tot = {k: tot[k] + st[k] for k in tot}
    assert tot["bounded"] > 0 and tot["full"] > 0 and tot["price_bounded"] > 0, tot
    assert tot["probe_rounds"] > 0, tot  # the exact probe rounds ran somewhere too


@pytest.mark.parametrize("rows,cols,form,seed", [
    (48, 80, 0, 11), (48, 80, 1, 12), (48, 80, 2, 13), (150, 300, 0, 21), (150, 300, 2, 22),
    (333, 500, 1, 31), (300, 450, 2, 32), (513, 700, 0, 33), (1, 3, 0, 4), (2, 2, 1, 5),
    (257, 129, 0, 6), (200, 200, 2, 7)])
def test_seeded_parity_with_port(port, rows, cols, form, seed):
    """Sizes straddling warp / block boundaries, m > n, tiny and degenerate forms."""
    from oracle.oracle import LP, make_config
    P = _P()
    lp = P.generate(P.GenSpec(rows, cols, seed=seed, form=P.Form(form)))
    ref = port.solve(LP(lp.m, lp.n_total, lp.A, lp.b, lp.c, lp.col_kind), make_config())
    rep, tr = _solve_traced(lp)
    assert int(rep.status) == ref.status
    _assert_trace(tr, ref.trace, (rows, cols, form, seed))
    assert _bits(rep.objective) == _bits(ref.objective) or (np.isnan(rep.objective) and np.isnan(ref.objective))
    assert np.array_equal(_bits(rep.x), _bits(ref.x))


@pytest.mark.parametrize("mode", ["always", "auto", "off"])
def test_duplicate_columns_exact_ties_with_port(port, mode):
    """Degenerate LPs whose structural columns are duplicated: every reduced
    cost, in pricing and in each lookahead's pricing, ties exactly with its
    twin, so the bounded pricing's candidate lists carry exact ties that only
    the (max z, min j) rule on exact values resolves. Pivots, x and objective
    must equal the reference port's, bit for bit, in every lookahead_bound mode."""
    from oracle.oracle import LP, make_config
    P = _P()
    for rows, cols, seed in ((60, 90, 3), (150, 240, 22)):
        base = P.generate(P.GenSpec(rows, cols, seed=seed, form=P.Form.degenerate))
        ck = np.asarray(base.col_kind)
        ns = int(np.sum(ck == 0))
        assert np.all(ck[:ns] == 0)
        dup = np.arange(0, ns, 3)
        A = np.hstack([base.A[:, :ns], base.A[:, dup], base.A[:, ns:]])
        c = np.concatenate([base.c[:ns], base.c[dup], base.c[ns:]])
        kind = np.concatenate([ck[:ns], ck[dup], ck[ns:]]).astype(np.uint8)
        lp = P.StandardFormLP(rows, A.shape[1], np.ascontiguousarray(A), np.asarray(base.b, float), c, kind)
        ref = port.solve(LP(lp.m, lp.n_total, lp.A, lp.b, lp.c, lp.col_kind), make_config())
        rep, tr = _solve_traced(lp, lookahead_bound=mode)
        assert int(rep.status) == ref.status, (rows, mode)
        _assert_trace(tr, ref.trace, (rows, mode))
        assert np.array_equal(_bits(rep.x), _bits(ref.x)), (rows, mode)


def test_sparse_classes_parity(port):
    from oracle.oracle import LP, make_config
    P = _P()
    for sp in (1, 2):
        lp = P.generate(P.GenSpec(90, 140, P.SparsityClass(sp), 3, P.Form.equality))
        ref = port.solve(LP(lp.m, lp.n_total, lp.A, lp.b, lp.c, lp.col_kind), make_config())
        rep, tr = _solve_traced(lp)
        assert int(rep.status) == ref.status
        _assert_trace(tr, ref.trace, sp)


def test_batch_size_does_not_change_results():
    P = _P()
    lp = P.generate(P.GenSpec(128, 256, seed=5, form=P.Form.degenerate))
    runs = [_solve_traced(lp, batch=b) for b in (1, 3, 64)]
    for rep, tr in runs[1:]:
        assert rep.objective == runs[0][0].objective
        _assert_trace(tr, runs[0][1], "batch")


def test_observer_sees_every_pivot_in_order():
    P = _P()
    seen = []
    lp = P.generate(P.GenSpec(40, 60, seed=2, form=P.Form.equality))
    rep = P.two_phase_solve(lp, P.SolverConfig(observer=seen.append))
    assert len(seen) == rep.iterations
    assert [v.iteration for v in seen] == list(range(1, rep.iterations + 1))
    assert seen[-1].objective == rep.objective


@pytest.mark.parametrize("name", ["gen_128x256_f2_s5", "netlib_afiro", "netlib_scsd1", "beale_3x7",
                                  "driveout_30x60_sum", "gen_96x160_f1_s4"])
def test_observer_rows_schedule_matches_golden(name):
    """observer_rows switches to the unfused one-pivot-per-round-trip schedule
     so IterationView.row(i) reads the reference's tableau at its
    observer call: same golden trace, objective and x bits; the basis in every
    view follows the trace; row 0 column m is the view's objective."""
    P = _P()
    g = Golden(name)
    seen = []

    def obs(v):
        r0 = v.tableau_row(0)
        seen.append((v.iteration, v.row, v.entering, v.basic.copy(), r0[g.m], v.objective,
                     v.counters["device_read_bytes"]))

    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle), observer=obs, observer_rows=True)
    with P.SimplexSolver(_golden_lp(g), cfg) as s:
        s.keep_trace(True)
        rep = s.solve()
        tr = s.trace()
    _assert_trace(tr, g.trace[: g.trace_len], name)
    assert np.array_equal(_bits(rep.x), _bits(g.x)), name
    assert len(seen) == len(tr)
    for (it, row, ent, basic, obj_row, obj, rd), t in zip(seen, tr):
        assert it == t["iteration"] and row == t["row"] and ent == t["entering"]
        assert basic[row] == ent
        assert _bits(obj_row) == _bits(obj) == _bits(t["objective"])
    assert all(b[6] > a[6] for a, b in zip(seen, seen[1:]))  # counters grow
    assert rep.memory["device_read_bytes"] >= seen[-1][6] and rep.memory["kernel_launches"] > 0


def test_observer_view_carries_the_basis():
    P = _P()
    seen = []
    lp = P.generate(P.GenSpec(64, 128, seed=2, form=P.Form.equality))
    with P.SimplexSolver(lp, P.SolverConfig(observer=seen.append)) as s:
        b0 = s.basis().copy()
        rep = s.solve()
        final = s.basis()
    basis = b0
    for v in seen:
        basis[v.row] = v.entering
        assert np.array_equal(v.basic, basis)
        with pytest.raises(P.Error):
            v.tableau_row(0)  # rows need observer_rows
    assert np.array_equal(basis, final) and len(seen) == rep.iterations


# ---- step API: SPEC.md operation examples -----------------
def _lp(A, b, c, ck):
    P = _P()
    A = np.asarray(A, float)
    return P.StandardFormLP(A.shape[0], A.shape[1], A, np.asarray(b, float),
                            np.asarray(c, float), np.asarray(ck, np.uint8))


def test_step_pivot_update_spec_example():
    """m=2, B^-1 = I, b_bar = (4,6), Y = (2,3), r = 0 -> B^-1 = [[.5,0],[-1.5,1]],
    b_bar = (2,0), Y = (1,0)."""
    P = _P()
    lp = _lp([[2, 1, 0], [3, 0, 1]], [4, 6], [-1, 0, 0], [0, 1, 1])
    with P.SimplexSolver(lp) as s:
        p = s.price()
        assert not p.optimal and p.entering == 0 and p.reduced_cost == 1.0
        s.compute_direction(p.entering, p.reduced_cost)
        assert np.array_equal(s.row(1)[[0, 1, 2, 3]], [1, 0, 4, 2])
        rt = s.ratio_test()
        assert not rt.unbounded and rt.theta == 2.0 and rt.candidates == [0, 1]
        s.pivot_update(0, p.entering)
        r1, r2 = s.row(1), s.row(2)
        assert list(r1) == [0.5, 0.0, 2.0, 1.0]
        assert list(r2) == [-1.5, 1.0, 0.0, 0.0]
        assert s.objective_value() == -2.0
        assert list(s.basis()) == [0, 2]


def test_step_ratio_examples():
    """b_bar=(2,4,1), Y=(1,2,-1) -> theta=2, candidates {0,1}."""
    P = _P()
    # columns: x (Y = (1,2,-1)), slacks s0..s2; min -x
    lp = _lp([[1, 1, 0, 0], [2, 0, 1, 0], [-1, 0, 0, 1]], [2, 4, 1], [-1, 0, 0, 0],
             [0, 1, 1, 1])
    with P.SimplexSolver(lp) as s:
        p = s.price()
        s.compute_direction(p.entering, p.reduced_cost)
        rt = s.ratio_test()
        assert rt.theta == 2.0 and rt.candidates == [0, 1]
    lp = _lp([[-1, 1, 0], [-2, 0, 1]], [1, 1], [-1, 0, 0], [0, 1, 1])
    with P.SimplexSolver(lp) as s:
        p = s.price()
        s.compute_direction(p.entering, p.reduced_cost)
        assert s.ratio_test().unbounded


def test_step_price_tie_takes_lower_index():
    P = _P()
    lp = _lp([[1, 1, 1]], [1], [-3, -3, 0], [0, 0, 1])
    with P.SimplexSolver(lp) as s:
        p = s.price()
        assert p.entering == 0 and p.reduced_cost == 3.0


def test_pivot_too_small_raises():
    P = _P()
    lp = _lp([[2, 1, 0], [0, 0, 1]], [4, 6], [-1, 0, 0], [0, 1, 1])
    with P.SimplexSolver(lp) as s:
        p = s.price()
        s.compute_direction(p.entering, p.reduced_cost)
        with pytest.raises(P.PivotTooSmall):
            s.pivot_update(1, p.entering)  # y_1 = 0


@pytest.mark.parametrize("name", ["netlib_scsd1", "netlib_lotfi", "netlib_e226", "netlib_sctap1",
                                  "netlib_boeing2", "netlib_grow7"])
def test_lookahead_scores_match_port_bitwise(port, name):
    """lookahead_score (solver.cpp:164-213) values, bit for bit: the port
    records every tie select_leaving scores (pivots done, entering, survivors,
    scores; oracle/lps_oracle.c lpo_set_tie_log). For up to 8 ties with
    nonzero scores the device solver runs to the same pivot count, re-prices
    and re-runs compute_direction through the step API, and its batched
    lookahead must return the identical doubles."""
    from oracle.oracle import LP, make_config
    P = _P()
    g = Golden(name)
    A, b, c, ck = g.arrays()
    cfg = make_config(**g.config_kwargs())
    _, ties = port.solve_with_ties(LP(g.m, g.n_total, A, b, c, ck), cfg, cap_ties=4096,
                                   cap_rows=1 << 20)
    scored = [t for t in ties if np.any(t[3] != 0)]
    assert scored, name
    pick = scored[:: max(1, len(scored) // 8)][:8]
    lp = _golden_lp(g)
    for it, q, rows, want in pick:
        with P.SimplexSolver(lp, P.SolverConfig(max_iter=it, pivot_tol=g.pivot_tol)) as s:
            rep = s.solve()
            assert rep.status == P.SolveStatus.iteration_limit and rep.iterations == it
            pr = s.price()
            assert not pr.optimal and pr.entering == q, (name, it)
            s.compute_direction(pr.entering, pr.reduced_cost)
            got = s.lookahead_scores([int(r) for r in rows], q)
            assert np.array_equal(_bits(got), _bits(want)), (name, it, got, want)


def test_non_finite_costs_or_coefficients_are_rejected():
    """The (max z, min j) pricing reduction equals the reference's strict '>'
    scan only for finite reduced costs, so inf/NaN in
    A or c is refused at create with LPSG_INVALID_ARGUMENT instead of silently
    diverging."""
    P = _P()
    A = np.array([[1.0, 2.0, 1.0, 0.0], [3.0, 1.0, 0.0, 1.0]])
    b = np.array([4.0, 5.0])
    c = np.array([-1.0, -1.0, 0.0, 0.0])
    ck = np.array([0, 0, 1, 1], np.uint8)
    for bad_A, bad_c in ((np.nan, None), (np.inf, None), (None, np.inf), (None, np.nan)):
        A2, c2 = A.copy(), c.copy()
        if bad_A is not None:
            A2[1, 0] = bad_A
        if bad_c is not None:
            c2[1] = bad_c
        with pytest.raises(P.Error, match="inf/NaN"):
            P.two_phase_solve(P.StandardFormLP(2, 4, A2, b, c2, ck))


def test_rejected_create_releases_device_memory():
    """A create that fails after the device buffers exist (here: inf in A,
    found by the upload's transpose) releases every one of them:
    m = 2000 allocates ~100 MB per attempt."""
    P = _P()
    import torch
    lp = P.generate(P.GenSpec(2000, 4000, seed=1))
    A = lp.A.copy()
    A[1999, 3999] = np.inf
    bad = P.StandardFormLP(lp.m, lp.n_total, A, lp.b, lp.c, lp.col_kind)
    with pytest.raises(P.Error, match="inf/NaN"):
        P.SimplexSolver(bad)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info(0)[0]
    for _ in range(6):
        with pytest.raises(P.Error, match="inf/NaN"):
            P.SimplexSolver(bad)
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info(0)[0]
    assert free0 - free1 < 64 << 20, (free0, free1)


def test_naive_kernel_mode_changes_only_zero_signs():
    """KernelMode::naive stores every element (tiled_engine.cpp:61-77). On
    BOEING2 that turns 26 of x's -0.0 into +0.0; the naive golden fixtures
    (netlib_*_naive, made by the reference with kernel=naive) pin those bits,
    and the cached run of the same LP keeps its -0.0s."""
    P = _P()
    g = Golden("netlib_boeing2_naive")
    assert g.kernel == 1
    lp = _golden_lp(g)
    rep_n, _ = _solve_traced(lp, kernel=1)
    rep_c, _ = _solve_traced(lp, kernel=0)
    assert np.array_equal(_bits(rep_n.x), _bits(g.x))
    neg0 = lambda x: int(np.sum(np.signbit(x) & (x == 0)))  # noqa: E731
    assert neg0(rep_n.x) == 0 and neg0(rep_c.x) == 26
    with pytest.raises(P.Error, match="kernel"):
        P.SimplexSolver(lp, P.SolverConfig(kernel=2))


def test_infinite_rhs_matches_port(port):
    """A non-finite right-hand side only reaches b_bar and the ratio test,
    whose std::min / <= comparisons the kernels reproduce: accepted, and the
    pivots match the CPU restatement."""
    P = _P()
    from oracle.oracle import LP, make_config
    A = np.array([[1.0, 2.0, 1.0, 0.0, 0.0], [3.0, 1.0, 0.0, 1.0, 0.0], [1.0, 1.0, 0.0, 0.0, 1.0]])
    b = np.array([4.0, np.inf, 3.0])
    c = np.array([-1.0, -2.0, 0.0, 0.0, 0.0])
    ck = np.array([0, 0, 1, 1, 1], np.uint8)
    ref = port.solve(LP(3, 5, A, b, c, ck, 1.0, 0.0, "inf_rhs"), make_config())
    rep, tr = _solve_traced(P.StandardFormLP(3, 5, A, b, c, ck))
    assert int(rep.status) == ref.status
    want = ref.trace[: ref.trace_len]
    assert len(tr) == len(want)
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        assert np.array_equal(tr[f], want[f]), f
    # the objective is inf - inf here: NaN on both sides (a NaN's sign bit is
    # not specified by IEEE and differs between x86 and the GPU)
    o, w = tr["objective"], want["objective"]
    assert np.array_equal(np.isnan(o), np.isnan(w))
    assert np.array_equal(_bits(o[~np.isnan(o)]), _bits(w[~np.isnan(w)]))
    assert np.array_equal(_bits(rep.x), _bits(ref.x))


def test_fp64_peak_probe():
    """lpsg_fp64_peak (the lookahead's roofline denominator) measures the fp64
    SIMT pipe: B200 does ~18.5 TFLOP/s counting DMUL and DADD as one flop each."""
    P = _P()
    v = P.fp64_peak(0)
    assert 5.0 < v < 40.0, v


@pytest.mark.parametrize("nan_rows", [[0], [0, 4, 8, 148], [2, 150, 299]])
def test_nan_rhs_matches_port(port, nan_rows):
    """NaN entries of b (some at the first row of an update CTA, m = 300 gives
    4-row CTAs) make those rows' ratios NaN. std::min(theta, NaN) keeps theta
    (solver.cpp:147), so they must never win the fused ratio test's CTA
    minimum. Port pinned to the reference on these inputs in
    tests/test_oracle.py::test_port_nan_rhs_matches_reference."""
    P = _P()
    from oracle.oracle import LP, make_config
    lp = P.generate(P.GenSpec(300, 400, seed=7, form=P.Form.le_max))
    b = lp.b.copy()
    b[nan_rows] = np.nan
    ref = port.solve(LP(lp.m, lp.n_total, lp.A, b, lp.c, lp.col_kind), make_config(max_iter=200))
    rep, tr = _solve_traced(P.StandardFormLP(lp.m, lp.n_total, lp.A, b, lp.c, lp.col_kind),
                            max_iter=200)
    assert int(rep.status) == ref.status
    want = ref.trace[: ref.trace_len]
    assert len(tr) == len(want)
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        assert np.array_equal(tr[f], want[f]), f
    x, w = rep.x, ref.x
    assert np.array_equal(np.isnan(x), np.isnan(w))
    assert np.array_equal(_bits(x[~np.isnan(x)]), _bits(w[~np.isnan(w)]))
