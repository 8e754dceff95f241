"""CPU parity of MPS ingestion.

The checks run the product's host-side ingestion (paper_1803_04378_b200/mps.py and
lp_model.py): parse_mps, to_general_lp, canonicalize, recover_solution,
write_mps and to_mps_document. They compare it with what the unmodified
reference does on the same bytes.

* Every tests/golden/mps/*.mps gives a bit-identical standard form against the
  reference's fixture. That covers A, including negated zeros, plus b, c,
  col_kind, the objective sign and constant, the CanonicalMap, the warnings and
  write_mps. recover_solution of the reference's x is compared too.
* tests/mps_cases.py covers every error the reference raises (same lps::Error
  subtype and message) and the accepted quirks.
* write_mps(to_mps_document(...)) of generated instances is byte-identical.
* The 11 Netlib files, when /root/reference is present, reproduce the Netlib
  golden fixtures' standard forms (tests/make_golden.py). When oracle/_ref is
  built, they are also checked live against the reference.
"""
import glob
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN_DIR, ROOT
from mps_cases import CASES

import paper_1803_04378_b200 as P
from paper_1803_04378_b200 import lp_model as LM
from paper_1803_04378_b200 import mps as M

MPS_DIR = os.path.join(GOLDEN_DIR, "mps")
FILES = sorted(os.path.splitext(os.path.basename(p))[0]
               for p in glob.glob(os.path.join(MPS_DIR, "*.mps")))
NETLIB = "/root/reference/proj/data/netlib"
REF_SO = os.path.join(ROOT, "oracle", "_ref", "liblps_ref.so")


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _same(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return a.shape == b.shape and np.array_equal(_bits(a), _bits(b))


def _text(name):
    with open(os.path.join(MPS_DIR, name + ".mps"), "rb") as f:
        return f.read()


def _check_std(lp, mp, z, warnings, tag):
    assert (lp.m, lp.n_total) == z["A"].shape, tag
    assert _same(lp.A, z["A"]), tag          # bitwise: negated rows carry -0.0
    assert _same(lp.b, z["b"]), tag
    assert _same(lp.c, z["c"]), tag
    assert np.array_equal(lp.col_kind, z["col_kind"]), tag
    assert _same([lp.objective_sign, lp.objective_constant],
                 [float(z["objective_sign"]), float(z["objective_constant"])]), tag
    assert _same(mp.shift, z["shift"]), tag
    assert np.array_equal(mp.negated_row.astype(np.uint8), z["negated_row"]), tag
    assert [p for p, _ in mp.split_pairs] == list(z["split_pos"]), tag
    assert [n for _, n in mp.split_pairs] == list(z["split_neg"]), tag
    assert "".join(w + "\n" for w in warnings) == str(z["warnings"]), tag


@pytest.mark.parametrize("name", FILES)
def test_mps_fixture_standard_form(name):
    z = np.load(os.path.join(MPS_DIR, name + ".npz"), allow_pickle=False)
    warnings = []
    lp, mp = M.load_mps(_text(name), warnings)
    _check_std(lp, mp, z, warnings, name)
    assert M.write_mps(M.parse_mps(_text(name))) == str(z["written"]), name


@pytest.mark.parametrize("name", FILES)
def test_mps_recover_solution(name):
    z = np.load(os.path.join(MPS_DIR, name + ".npz"), allow_pickle=False)
    if "x_recovered" not in z.files:
        pytest.skip("the reference did not reach an optimal / iteration-limit report")
    _, mp = M.load_mps(_text(name))
    x, obj = LM.recover_solution(mp, z["x"], float(z["objective"]))
    assert _same(x, z["x_recovered"]) and _same([obj], [float(z["objective_recovered"])])
    with pytest.raises(LM.LengthMismatch):
        LM.recover_solution(mp, z["x"][:-1], 0.0)


@pytest.mark.parametrize("name", FILES)
def test_mps_write_parse_round_trip(name):
    doc = M.parse_mps(_text(name))
    again = M.parse_mps(M.write_mps(doc))
    for f in ("name", "objsense", "rows", "columns", "rhs", "ranges", "bounds"):
        assert getattr(again, f) == getattr(doc, f), (name, f)


def _cases():
    with open(os.path.join(MPS_DIR, "cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", sorted(CASES))
def test_mps_cases(name):
    want = _cases()[name]
    if "error_kind" in want:
        with pytest.raises(P.Error) as ei:
            M.load_mps(CASES[name].encode())
        kind = type(ei.value).__name__
        assert kind == want["error_kind"], (name, kind, want)
        assert str(ei.value) == want["error"], (name, str(ei.value), want["error"])
        return
    warnings = []
    lp, _ = M.load_mps(CASES[name].encode(), warnings)
    import hashlib
    h = hashlib.sha256()
    for a in (lp.A, lp.b, lp.c, lp.col_kind):
        h.update(np.ascontiguousarray(a).tobytes())
    h.update(np.float64([lp.objective_sign, lp.objective_constant]).tobytes())
    assert (lp.m, lp.n_total) == (want["m"], want["n_total"]), name
    assert h.hexdigest() == want["digest"], name
    assert "".join(w + "\n" for w in warnings) == want["warnings"], name
    assert M.write_mps(M.parse_mps(CASES[name])) == want["written"], name


def _general_from_generator(rows, cols, seed, form, sparsity):
    """The reference's GeneralLP of lps::generate (+ form 1), rebuilt from
    the product's bit-exact generator (lpsg_generate)."""
    lp = P.generate(P.GenSpec(rows, cols, P.SparsityClass(sparsity), seed, P.Form(form)))
    g = LM.GeneralLP(name="")
    g.resize(rows, cols)
    g.coeffs[:] = lp.A[:, :cols]
    g.rhs[:] = lp.b
    if form == 0:
        g.row_kind = [LM.RowKind.eq] * rows
        g.objective[:] = lp.c[:cols]
    else:
        g.sense = LM.Sense.maximize
        g.objective[:] = -lp.c[:cols]
    g.name = f"gen_{rows}x{cols}_s{seed}"  # lps::generate's naming is not part of the text below
    return g


@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(MPS_DIR, "generated_*.mps.txt"))))
def test_mps_generated_document(path):
    base = os.path.basename(path)[len("generated_"):-len(".mps.txt")]
    dims, s, f, sp = base.split("_")
    rows, cols = (int(v) for v in dims.split("x"))
    want = open(path).read()
    g = _general_from_generator(rows, cols, int(s[1:]), int(f[1:]), int(sp[2:]))
    # the reference's generate() names the LP; take the NAME line from the fixture
    g.name = want.splitlines()[0][len("NAME          "):]
    assert M.write_mps(M.to_mps_document(g)) == want
    # and the document reads back to the same standard form as the generator's
    lp, _ = M.load_mps(want)
    ref = P.generate(P.GenSpec(rows, cols, P.SparsityClass(int(sp[2:])), int(s[1:]),
                               P.Form(int(f[1:]))))
    assert _same(lp.A, ref.A) and _same(lp.b, ref.b) and _same(lp.c, ref.c)


def test_mps_number_spellings():
    pn = M._parse_number
    assert pn("1.", 1) == 1.0 and pn(".5", 1) == 0.5 and pn("-2E+3", 1) == -2000.0
    assert pn("0x1p-2", 1) == 0.25 and pn("-0x.8", 1) == -0.5 and pn("0X10", 1) == 16.0
    assert pn("inf", 1) == float("inf") and pn("-Infinity", 1) == float("-inf")
    assert np.isnan(pn("nan", 1)) and np.isnan(pn("NaN(1)", 1))
    assert pn("1e400", 1) == float("inf") and pn("1e-400", 1) == 0.0
    for bad in ("1_0", "1e", "0x", "0x1p", "infin", "--1", "1.2.3", "١", ""):
        with pytest.raises(M.MalformedNumber):
            pn(bad, 7)


def test_canonicalize_general_lp_directly():
    """A hand-built GeneralLP with a free_row and every bound shape: the
    product's canonicalize against the reference's rules (lp_model.cpp:43-163)."""
    g = LM.GeneralLP(name="hand")
    g.resize(3, 3)
    g.coeffs[:] = [[1.0, -2.0, 0.0], [0.0, 1.0, 1.0], [5.0, 5.0, 5.0]]
    g.rhs[:] = [-4.0, 3.0, 9.0]
    g.row_kind = [LM.RowKind.le, LM.RowKind.eq, LM.RowKind.free_row]
    g.objective[:] = [1.0, 2.0, -1.0]
    g.lower[:] = [-1.0, -np.inf, 0.0]
    g.upper[:] = [np.inf, 4.0, 2.0]
    lp, mp = LM.canonicalize(g)
    # rows: le (rhs -4 - (1*-1) = -3 -> negated to ge 3), eq, x2 <= 4 (split), x3 <= 2
    assert lp.m == 4 and lp.n_total == 4 + 3
    assert mp.split_pairs == [(1, 3)] and list(mp.negated_row) == [True, False, False, False]
    assert _same(lp.b, [3.0, 3.0, 4.0, 2.0])
    assert _same(lp.A[0, :4], [-1.0, 2.0, -0.0, -2.0]) and lp.A[0, 4] == -1.0
    assert _same(lp.A[2, :4], [0.0, 1.0, 0.0, -1.0]) and lp.A[2, 5] == 1.0
    assert list(lp.col_kind) == [0, 0, 0, 0, 1, 1, 1]
    with pytest.raises(LM.InconsistentBounds, match="column 0: lower 2.000000 > upper 1.000000"):
        g.lower[0], g.upper[0] = 2.0, 1.0
        LM.canonicalize(g)
    with pytest.raises(LM.EmptyProblem):
        LM.canonicalize(LM.GeneralLP())


@pytest.mark.skipif(not os.path.isdir(NETLIB), reason="/root/reference is not present")
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(NETLIB, "*.mps"))))
def test_netlib_standard_form_matches_golden(path):
    name = "netlib_" + os.path.splitext(os.path.basename(path))[0]
    z = np.load(os.path.join(GOLDEN_DIR, name + ".npz"), allow_pickle=False)
    lp, _ = M.load_mps(path)
    A = np.zeros((int(z["m"]), int(z["n_total"])))
    A[z["A_rows"], z["A_cols"]] = z["A_vals"]
    assert (lp.m, lp.n_total) == A.shape, name
    assert np.array_equal(lp.A, A), name
    nz = lp.A != 0
    assert _same(lp.A[nz], A[nz]), name
    assert _same(lp.b, z["b"]) and _same(lp.c, z["c"]), name
    assert np.array_equal(lp.col_kind, z["col_kind"]), name
    assert _same([lp.objective_sign, lp.objective_constant],
                 [float(z["objective_sign"]), float(z["objective_constant"])]), name


@pytest.mark.skipif(not (os.path.isdir(NETLIB) and os.path.exists(REF_SO)),
                    reason="needs /root/reference and oracle/_ref")
@pytest.mark.parametrize("path", sorted(glob.glob(os.path.join(NETLIB, "*.mps"))))
def test_netlib_live_against_reference(path):
    from oracle.oracle import Ref
    ref = Ref()
    data = open(path, "rb").read()
    out = ref.mps_load(data)
    warnings = []
    lp, mp = M.load_mps(data, warnings)
    z = {"A": out["lp"].A, "b": out["lp"].b, "c": out["lp"].c, "col_kind": out["lp"].col_kind,
         "objective_sign": out["lp"].objective_sign,
         "objective_constant": out["lp"].objective_constant, "shift": out["shift"],
         "negated_row": out["negated_row"], "split_pos": out["split_pos"],
         "split_neg": out["split_neg"], "warnings": out["warnings"]}
    _check_std(lp, mp, z, warnings, path)
    assert M.write_mps(M.parse_mps(data)) == out["written"]
    x_std = np.linspace(0.0, 1.0, lp.n_total)
    xr, zr = ref.mps_recover(out, x_std, -3.25)
    x, obj = LM.recover_solution(mp, x_std, -3.25)
    assert _same(x, xr) and _same([obj], [zr])
    ref.mps_free(out)
