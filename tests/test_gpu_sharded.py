"""GPU parity of the SHARDED solver.

The sharded path (rows of B^-1 split across shards, pricing columns split
across shards, pivot row / (z, j) / ratio-test messages exchanged every pivot,
the ordered rebuild_top_row chain, sharded drive-out and lookahead) runs here
as G shards on ONE B200 with in-process device-to-device exchanges
(lpsg_solve_sharded). The kernels and the host schedule are the ones an NCCL
run uses; only the transport differs. Bar: the same golden traces, bit for bit.
"""
import numpy as np
import pytest

from conftest import Golden, golden_names

pytestmark = pytest.mark.gpu

NAMES = golden_names()


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


def _check(rep, tr, g, tag):
    ref = g.trace[: g.trace_len]
    assert int(rep.status) == g.status, (tag, rep.status, g.status)
    assert (rep.iterations_phase1, rep.iterations_phase2) == (g.p1, g.p2), tag
    assert len(tr) == len(ref), (tag, len(tr), len(ref))
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        bad = np.nonzero(tr[f] != ref[f])[0]
        assert bad.size == 0, (tag, f, int(bad[0]) if bad.size else None)
    assert np.array_equal(_bits(tr["objective"]), _bits(ref["objective"])), tag
    if np.isnan(g.objective):
        assert np.isnan(rep.objective)
    else:
        assert _bits(rep.objective) == _bits(g.objective), (tag, rep.objective, g.objective)
    assert np.array_equal(_bits(rep.x), _bits(g.x)), tag


@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("name", NAMES)
def test_sharded_golden_parity(name, shards):
    P = _P()
    g = Golden(name)
    if shards > g.m:
        pytest.skip("fewer rows than shards")
    lp = _golden_lp(g)
    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle))
    rep, tr = P.solve_sharded(lp, cfg, shards=shards, trace=True)
    _check(rep, tr, g, (name, shards))


TIE_NAMES = [n for n in NAMES if "_f2_" in n or n.startswith(("beale", "netlib"))]


@pytest.mark.parametrize("shards", [2, 4])
@pytest.mark.parametrize("name", TIE_NAMES)
def test_sharded_bounded_pricing_always(name, shards):
    """The bounded pricing (DMMA screen + exact chains) on
    every tie of >= 2 candidates, per shard over its own columns, merged by the
    exact (max z, min j) exchange: the same pivots as the reference, bit for bit."""
    P = _P()
    g = Golden(name)
    if shards > g.m:
        pytest.skip("fewer rows than shards")
    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle), lookahead_bound="always")
    rep, tr = P.solve_sharded(_golden_lp(g), cfg, shards=shards, trace=True)
    _check(rep, tr, g, (name, shards, "always"))


P2P_NAMES = ["gen_256x512_f2_s1", "gen_256x512_f0_s1", "gen_1000x2000_f0_s1_max_iter400",
             "gen_2000x4000_f0_s1_max_iter200", "netlib_scsd1", "netlib_sctap1", "netlib_boeing2",
             "beale_3x7", "infeasible_2x2", "unbounded_1x3", "gen_128x256_f2_s5_anticyclenone"]


@pytest.mark.parametrize("shards", [2, 3])
@pytest.mark.parametrize("name", P2P_NAMES)
def test_sharded_p2p_golden_parity(name, shards):
    """The device-initiated P2P transport (peer stores + sequence flags, no host
    synchronisation per exchange), shards sharing one B200. Limited to 2-3
    shards: on a SHARED GPU a shard's spin-waiting exchange kernel competes for
    SMs with the other shards' streaming kernels; with one shard per GPU (the
    real deployment) it never does. A wait that cannot complete times out
    (LPSG_P2P_TIMEOUT_S) instead of hanging."""
    P = _P()
    g = Golden(name)
    if shards > g.m:
        pytest.skip("fewer rows than shards")
    lp = _golden_lp(g)
    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle))
    rep, tr = P.solve_sharded(lp, cfg, shards=shards, trace=True, p2p=True)
    _check(rep, tr, g, (name, shards, "p2p"))


@pytest.mark.parametrize("shards", [4, 8])
@pytest.mark.parametrize("name", ["gen_256x512_f2_s1", "gen_128x256_f2_s5", "netlib_scsd1",
                                  "gen_256x512_f1_s1", "beale_3x7"])
def test_sharded_more_shards(name, shards):
    """4 and 8 shards (the 8-GPU row split) on tie-heavy and structured inputs."""
    P = _P()
    g = Golden(name)
    if shards > g.m:
        pytest.skip("fewer rows than shards")
    lp = _golden_lp(g)
    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle))
    rep, tr = P.solve_sharded(lp, cfg, shards=shards, trace=True)
    _check(rep, tr, g, (name, shards))


def test_sharded_matches_single_gpu_prefix_c3():
    """C3 (m=8000, n=16000) first 60 pivots: 4 shards == single GPU, bit for bit."""
    P = _P()
    lp = P.generate(P.GenSpec(8000, 16000, seed=1))
    cfg = P.SolverConfig(max_iter=60)
    with P.SimplexSolver(lp, cfg) as s:
        s.keep_trace(True)
        rep1 = s.solve()
        tr1 = s.trace()
    for shards, p2p in ((4, False), (2, True)):
        rep4, tr4 = P.solve_sharded(lp, cfg, shards=shards, trace=True, p2p=p2p)
        assert len(tr1) == len(tr4) == 60
        for f in ("row", "leaving", "entering"):
            assert np.array_equal(tr1[f], tr4[f]), (f, p2p)
        assert np.array_equal(_bits(tr1["objective"]), _bits(tr4["objective"]))
        assert np.array_equal(_bits(rep1.x), _bits(rep4.x))
