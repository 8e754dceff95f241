"""CPU tests: the oracle is pinned to the reference, and input plumbing is bit-exact.

* The plain-C port (oracle/lps_oracle.c) reproduces every golden reference run
  pivot for pivot, with bit-identical objective and x.
* When the compiled reference (oracle/_ref) is present, it reproduces the golden
  fixtures too (the fixtures were made by it; this catches drift in the build).
* The product's generator (lpsg_generate) and the port's generator produce the
  reference's exact arrays (SHA-256 recorded in each golden fixture).
"""
import os

import numpy as np
import pytest

from conftest import Golden, ROOT, golden_names

NAMES = golden_names()
# The large prefix fixtures take a few seconds each on the port; keep the CPU suite quick.
QUICK = [n for n in NAMES if "2000x4000" not in n]


def _same_trace(a, b):
    if len(a) != len(b):
        return False
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        if not np.array_equal(a[f], b[f]):
            return False
    return np.array_equal(a["objective"].view(np.uint64), b["objective"].view(np.uint64))


def _bits_equal(x, y):
    x, y = np.asarray(x, np.float64), np.asarray(y, np.float64)
    return x.shape == y.shape and np.array_equal(x.view(np.uint64), y.view(np.uint64))


def _check_against(g, out):
    assert out.status == g.status, (g.name, out.status, g.status)
    assert out.iterations_phase1 == g.p1 and out.iterations_phase2 == g.p2, g.name
    assert out.trace_len == g.trace_len, g.name
    assert _same_trace(out.trace, g.trace), g.name
    if np.isnan(g.objective):
        assert np.isnan(out.objective)
    else:
        assert _bits_equal(out.objective, g.objective), (g.name, out.objective, g.objective)
    assert _bits_equal(out.x, g.x), g.name


@pytest.mark.parametrize("name", QUICK)
def test_port_matches_reference_golden(port, name):
    from oracle.oracle import LP, make_config
    g = Golden(name)
    A, b, c, ck = g.arrays(port.generate)
    lp = LP(g.m, g.n_total, A, b, c, ck)
    out = port.solve(lp, make_config(**g.config_kwargs()))
    _check_against(g, out)


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblps_ref.so")),
                    reason="compiled reference not present")
@pytest.mark.parametrize("name", [n for n in QUICK if n.startswith(("gen_20", "gen_64", "netlib_afiro", "beale"))])
def test_reference_build_matches_golden(name):
    from oracle.oracle import LP, Ref, make_config
    ref = Ref()
    g = Golden(name)
    A, b, c, ck = g.arrays(ref.generate)
    out = ref.solve(LP(g.m, g.n_total, A, b, c, ck), make_config(**g.config_kwargs()))
    _check_against(g, out)


def _digest(A, b, c, ck):
    import hashlib
    h = hashlib.sha256()
    for a in (A, b, c, ck):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.mark.parametrize("name", [n for n in NAMES if n.startswith("gen_") and "max_iter" not in n
                                  and "anticycle" not in n])
def test_generators_match_reference_digest(port, name):
    import paper_1803_04378_b200 as P
    g = Golden(name)
    rows, cols, form, seed, sp = g.spec
    lp = port.generate(rows, cols, seed, form)
    assert _digest(lp.A, lp.b, lp.c, lp.col_kind) == g.digest
    q = P.generate(P.GenSpec(rows, cols, P.SparsityClass(sp), seed, P.Form(form)))
    assert _digest(q.A, q.b, q.c, q.col_kind) == g.digest


def test_generator_sparsity_classes_match_port(port):
    """S20 / S60 draws (generator.cpp:55) through both restatements."""
    import paper_1803_04378_b200 as P
    for sp in (1, 2):
        for form in (0, 1, 2):
            a = port.generate(30, 50, 7, form, sparsity=sp)
            q = P.generate(P.GenSpec(30, 50, P.SparsityClass(sp), 7, P.Form(form)))
            assert _digest(a.A, a.b, a.c, a.col_kind) == _digest(q.A, q.b, q.c, q.col_kind)


def test_generator_rejects_empty_spec():
    import paper_1803_04378_b200 as P
    with pytest.raises(P.DegenerateSpec):
        P.generate(P.GenSpec(0, 5))


def test_spec_pivot_example_on_port(port):
    """SPEC.md pivot_update example through a full solve's first pivot: B^-1 = I,
    b_bar = (4, 6), Y = (2, 3) -> theta = 2 (tie of rows 0 and 1)."""
    from oracle.oracle import LP, make_config
    # Min -x0 s.t. 2 x0 + s0 = 4, 3 x0 + s1 = 6 (slack start), the reference's own
    # tie example: both ratios are 2.
    lp = LP(2, 3, np.array([[2.0, 1.0, 0.0], [3.0, 0.0, 1.0]]), np.array([4.0, 6.0]),
            np.array([-1.0, 0.0, 0.0]), np.array([0, 1, 1], np.uint8))
    out = port.solve(lp, make_config())
    assert out.status == 0 and out.objective == -2.0
    assert out.trace_len == 1
    assert out.trace[0]["entering"] == 0


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblps_ref.so")),
                    reason="compiled reference not present")
@pytest.mark.parametrize("nan_rows", [[0], [0, 4, 8, 148], [2, 150, 299]])
def test_port_nan_rhs_matches_reference(port, nan_rows):
    """Pins the port on NaN right-hand sides (the GPU test of the same inputs
    compares against the port: tests/test_gpu_parity.py::test_nan_rhs_matches_port)."""
    from oracle.oracle import LP, Ref, make_config
    ref = Ref()
    lp = ref.generate(300, 400, 7, 1)
    b = lp.b.copy()
    b[nan_rows] = np.nan
    l2 = LP(lp.m, lp.n_total, lp.A, b, lp.c, lp.col_kind)
    a = ref.solve(l2, make_config(max_iter=200))
    p = port.solve(l2, make_config(max_iter=200))
    assert a.status == p.status and a.trace_len == p.trace_len
    for f in ("iteration", "phase", "row", "leaving", "entering"):
        assert np.array_equal(a.trace[f], p.trace[f]), f
    assert np.array_equal(np.isnan(a.x), np.isnan(p.x))
    assert _bits_equal(a.x[~np.isnan(a.x)], p.x[~np.isnan(p.x)])
