"""General LPs and their standard form (LP ingestion).

Mirrors /root/reference/proj/include/lps/lp_model.hpp and src/lp_model.cpp, so
an MPS file (mps.py) or a hand-built model reaches the solver in exactly the
standard form the reference builds:

* ``GeneralLP`` / ``resize``                lp_model.hpp:21-43, lp_model.cpp:10-20
* ``canonicalize(p) -> (StandardFormLP, CanonicalMap)``
                                            lp_model.cpp:43-163 (same column and row
                                            order, same fp64 operation order, same errors)
* ``recover_solution(map, x_std, z_std)``   lp_model.cpp:165-177

Host-side ingestion, not the hot path. Unlike the reference it builds the
standard form in place in one dense row-major array (no PendingRow copies,
lp_model.cpp:98-146), optionally straight into pinned host memory for the
device upload (``canonicalize(..., pinned=True)``). Each fp64 result is the same
IEEE operation, in the same order, as the reference's scalar loop: numpy
elementwise ops round each element once, like the C++ statements.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from .solver import ColKind, DegenerateSpec, Error, StandardFormLP

INF = float("inf")


class InconsistentBounds(Error):
    """lps::InconsistentBounds (errors.hpp:15-17)."""


class EmptyProblem(DegenerateSpec):
    """lps::EmptyProblem (errors.hpp:19-21)."""


class LengthMismatch(Error):
    """lps::LengthMismatch (errors.hpp:23-25)."""


class Sense(enum.IntEnum):
    """lps::Sense (lp_model.hpp:14)."""
    minimize = 0
    maximize = 1


class RowKind(enum.IntEnum):
    """lps::RowKind (lp_model.hpp:18): free_row contributes no constraint."""
    eq = 0
    le = 1
    ge = 2
    free_row = 3


@dataclass
class GeneralLP:
    """lps::GeneralLP (lp_model.hpp:23-43): dense row-major coefficients.

    ``range[i]`` is None when row i has no RANGES entry (std::optional)."""
    name: str = ""
    sense: Sense = Sense.minimize
    num_rows: int = 0
    num_cols: int = 0
    row_kind: List[RowKind] = field(default_factory=list)
    coeffs: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    objective: np.ndarray = field(default_factory=lambda: np.zeros(0))
    rhs: np.ndarray = field(default_factory=lambda: np.zeros(0))
    range: List[Optional[float]] = field(default_factory=list)
    lower: np.ndarray = field(default_factory=lambda: np.zeros(0))
    upper: np.ndarray = field(default_factory=lambda: np.zeros(0))
    objective_constant: float = 0.0

    def resize(self, rows: int, cols: int) -> None:
        """lp_model.cpp:10-20: every vector sized with its default."""
        self.num_rows, self.num_cols = rows, cols
        self.row_kind = [RowKind.le] * rows
        self.coeffs = np.zeros((rows, cols))
        self.objective = np.zeros(cols)
        self.rhs = np.zeros(rows)
        self.range = [None] * rows
        self.lower = np.zeros(cols)
        self.upper = np.full(cols, INF)

    def at(self, i: int, j: int) -> float:
        return float(self.coeffs[i, j])


@dataclass
class CanonicalMap:
    """lps::CanonicalMap (lp_model.hpp:71-79)."""
    orig_cols: int = 0
    std_cols: int = 0
    shift: np.ndarray = field(default_factory=lambda: np.zeros(0))
    negated_row: np.ndarray = field(default_factory=lambda: np.zeros(0, bool))
    split_pairs: List[Tuple[int, int]] = field(default_factory=list)  # (pos, neg)
    objective_sign: float = 1.0
    objective_constant: float = 0.0


def _cxx_to_string(v: float) -> str:
    """std::to_string(double): printf("%f")."""
    return "%f" % v


def _range_interval(kind: RowKind, rhs: float, r: float) -> Tuple[float, float]:
    """lp_model.cpp:33-39 (Netlib RANGES semantics)."""
    if kind == RowKind.le:
        return rhs - abs(r), rhs
    if kind == RowKind.ge:
        return rhs, rhs + abs(r)
    return (rhs, rhs + r) if r >= 0 else (rhs + r, rhs)


def canonicalize(p: GeneralLP, pinned: bool = False) -> Tuple[StandardFormLP, CanonicalMap]:
    """lps::canonicalize (lp_model.cpp:43-163).

    Column order: originals, then the negative halves of split free columns
    (in original order), then one slack per non-equality row. Row order: the
    constraint rows (a RANGES row becomes its le row then its ge row, or one eq
    row when the interval is a point), then one x_j <= u_j row per finite upper
    bound. Rows with a negative right-hand side are negated (every structural
    coefficient, zeros included) and their relation flipped before the slacks
    are added, so b >= 0 exactly.
    """
    if p.num_rows == 0 or p.num_cols == 0:
        raise EmptyProblem("canonicalize: problem has no rows or no columns")
    n0 = p.num_cols
    lower = np.asarray(p.lower, np.float64)
    upper = np.asarray(p.upper, np.float64)
    coeffs = np.asarray(p.coeffs, np.float64).reshape(p.num_rows, n0)
    mp = CanonicalMap(orig_cols=n0, objective_sign=-1.0 if p.sense == Sense.maximize else 1.0)
    mp.shift = np.zeros(n0)

    # column plan (lp_model.cpp:54-67)
    structural = n0
    neg_col = np.full(n0, -1, np.int64)
    for j in range(n0):
        if lower[j] > upper[j]:
            raise InconsistentBounds(f"column {j}: lower {_cxx_to_string(lower[j])} > upper "
                                     f"{_cxx_to_string(upper[j])}")
        if lower[j] == -INF:
            neg_col[j] = structural
            mp.split_pairs.append((j, structural))
            structural += 1
        else:
            mp.shift[j] = lower[j]
    split = neg_col >= 0
    neg_idx = neg_col[split]

    sign = mp.objective_sign
    c_min = np.zeros(structural)
    c_min[:n0] = sign * np.asarray(p.objective, np.float64)
    c_min[neg_idx] = -c_min[:n0][split]

    # row plan (lp_model.cpp:84-115): (source row or -1, kind, rhs, upper-bound column)
    live = [i for i in range(p.num_rows) if p.row_kind[i] != RowKind.free_row]
    shifted = np.asarray(p.rhs, np.float64)[live].copy()
    if live:
        sub = coeffs[live]
        for j in range(n0):  # shifted_rhs -= a[j] * shift[j], j ascending
            shifted = shifted - sub[:, j] * mp.shift[j]
    plan = []
    for k, i in enumerate(live):
        rng = p.range[i]
        if rng is not None:
            lo, hi = _range_interval(RowKind(p.row_kind[i]), float(shifted[k]), float(rng))
            if lo == hi:
                plan.append((i, RowKind.eq, lo, -1))
            else:
                plan.append((i, RowKind.le, hi, -1))
                plan.append((i, RowKind.ge, lo, -1))
        else:
            plan.append((i, RowKind(p.row_kind[i]), float(shifted[k]), -1))
    for j in range(n0):  # upper bounds as explicit rows (lp_model.cpp:118-126)
        if upper[j] == INF:
            continue
        plan.append((-1, RowKind.le, float(upper[j] - mp.shift[j]), j))

    m = len(plan)
    n_slack = sum(1 for _, kind, _, _ in plan if kind != RowKind.eq)
    n_total = structural + n_slack
    if pinned:
        from .solver import PinnedBuffer
        A_owner = PinnedBuffer(8 * m * n_total)
        A = A_owner.array((m, n_total), np.float64)
        A[...] = 0.0
    else:
        A, A_owner = np.zeros((m, n_total)), None
    b = np.zeros(m)
    c = np.zeros(n_total)
    col_kind = np.full(n_total, int(ColKind.structural), np.uint8)
    c[:structural] = c_min
    mp.negated_row = np.zeros(m, bool)
    next_slack = structural
    for r, (i, kind, rhs, ucol) in enumerate(plan):
        row = A[r]
        if i >= 0:
            row[:n0] = coeffs[i]
            row[neg_idx] = -coeffs[i][split]
        else:
            row[ucol] = 1.0
            if neg_col[ucol] >= 0:
                row[neg_col[ucol]] = -1.0
        if rhs < 0.0:  # lp_model.cpp:129-139
            rhs = -rhs
            row[:structural] = -row[:structural]
            kind = {RowKind.le: RowKind.ge, RowKind.ge: RowKind.le}.get(kind, kind)
            mp.negated_row[r] = True
        b[r] = rhs
        if kind != RowKind.eq:
            row[next_slack] = 1.0 if kind == RowKind.le else -1.0
            col_kind[next_slack] = int(ColKind.slack)
            next_slack += 1

    mp.std_cols = n_total
    shift_cost = 0.0
    for j in range(n0):  # sequential, like lp_model.cpp:158-159
        shift_cost += float(c_min[j]) * float(mp.shift[j])
    mp.objective_constant = sign * shift_cost + float(p.objective_constant)
    lp = StandardFormLP(m, n_total, A, b, c, col_kind, name=p.name, objective_sign=sign,
                        objective_constant=mp.objective_constant)
    if A_owner is not None:
        lp._pinned = A_owner  # keeps the page-locked buffer alive with the view
    return lp, mp


def recover_solution(mp: CanonicalMap, x_std: Sequence[float], z_std: float):
    """lps::recover_solution (lp_model.cpp:165-177): (x in the original
    variables, objective in the original sense)."""
    x_std = np.asarray(x_std, np.float64)
    if x_std.shape[0] != mp.std_cols:
        raise LengthMismatch(f"recover_solution: expected {mp.std_cols} values, got "
                             f"{x_std.shape[0]}")
    x = x_std[:mp.orig_cols] + mp.shift
    for pos, neg in mp.split_pairs:
        x[pos] = x[pos] - x_std[neg]
    return x, mp.objective_sign * float(z_std) + mp.objective_constant
