"""MPS ingestion (the MPS/Netlib regression inputs).

Mirrors /root/reference/proj/include/lps/mps.hpp and src/mps.cpp:

* ``MpsDocument``, ``MpsRowKind``, ``MpsBoundKind``   mps.hpp:11-46 (file order kept,
                                                      nothing merged or defaulted)
* ``parse_mps(text)`` / ``parse_mps_file(path)``      mps.cpp:57-229 (fixed or free
                                                      format, section order enforced,
                                                      '*' comments, MARKER lines skipped,
                                                      missing ENDATA tolerated)
* ``to_general_lp(doc, warnings=None)``               mps.cpp:236-351
* ``write_mps(doc)`` (round-trip exact numbers)       mps.cpp:353-401
* ``to_mps_document(lp)`` (R1.., X1.., COST)          mps.cpp:403-427
* errors UnknownSection, UndeclaredRow, DuplicateRow, MissingObjectiveRow,
  MalformedNumber, UnsupportedBoundKind               errors.hpp:29-55

plus ``load_mps(path_or_text)`` = parse + to_general_lp + canonicalize, the
chain of the reference CLI's ``solve`` (lps_main.cpp:110-112), and
``solve_mps``, which adds the GPU solve and recover_solution
(lps_main.cpp:113-118).

Text is handled as bytes decoded latin-1 (1:1), tokens split on the C locale's
whitespace and keywords upper-cased in ASCII, like the reference's
``istringstream >>`` and ``std::toupper``. Numbers follow ``std::strtod``: the
whole token must parse (decimal, hex floats, inf/nan); Python-only spellings
such as digit underscores are rejected.
"""
from __future__ import annotations

import enum
import math
import re
from dataclasses import dataclass, field
from typing import List, Optional, Tuple

import numpy as np

from .lp_model import INF, CanonicalMap, GeneralLP, RowKind, Sense, canonicalize, recover_solution
from .solver import Error, SolveReport, SolverConfig, SolveStatus, StandardFormLP


class UnknownSection(Error):
    """lps::UnknownSection (errors.hpp:29-31)."""


class UndeclaredRow(Error):
    """lps::UndeclaredRow (errors.hpp:33-35)."""


class DuplicateRow(Error):
    """lps::DuplicateRow (errors.hpp:37-39)."""


class MissingObjectiveRow(Error):
    """lps::MissingObjectiveRow (errors.hpp:41-43)."""


class MalformedNumber(Error):
    """lps::MalformedNumber (errors.hpp:45-50)."""

    def __init__(self, token: str, line: int):
        super().__init__(f"malformed number '{token}' at line {line}")
        self.line_number = line


class UnsupportedBoundKind(Error):
    """lps::UnsupportedBoundKind (errors.hpp:52-54)."""


class MpsRowKind(enum.IntEnum):
    n = 0
    l = 1  # noqa: E741 - the MPS letter
    g = 2
    e = 3


class MpsBoundKind(enum.IntEnum):
    up = 0
    lo = 1
    fx = 2
    fr = 3
    mi = 4
    pl = 5
    bv = 6


@dataclass
class MpsRow:
    kind: MpsRowKind
    name: str


@dataclass
class MpsEntry:
    """A COLUMNS / RHS / RANGES triple (column is the set name for RHS/RANGES)."""
    column: str
    row: str
    value: float


@dataclass
class MpsBound:
    kind: MpsBoundKind
    set: str
    column: str
    value: float = 0.0  # meaningful for up/lo/fx only


@dataclass
class MpsDocument:
    """lps::MpsDocument (mps.hpp:17-46)."""
    name: str = ""
    objsense: Sense = Sense.minimize
    rows: List[MpsRow] = field(default_factory=list)
    columns: List[MpsEntry] = field(default_factory=list)
    rhs: List[MpsEntry] = field(default_factory=list)
    ranges: List[MpsEntry] = field(default_factory=list)
    bounds: List[MpsBound] = field(default_factory=list)
    warnings: List[str] = field(default_factory=list)
    missing_endata: bool = False


# section ranks (mps.cpp:19): start < name < objsense < rows < columns < rhs < ranges < bounds < endata
_START, _NAME, _OBJSENSE, _ROWS, _COLUMNS, _RHS, _RANGES, _BOUNDS, _ENDATA = range(9)
_HEADERS = {"NAME": _NAME, "OBJSENSE": _OBJSENSE, "ROWS": _ROWS, "COLUMNS": _COLUMNS,
            "RHS": _RHS, "RANGES": _RANGES, "BOUNDS": _BOUNDS}
_C_SPACE = " \t\n\v\f\r"
_SPLIT = re.compile(r"[ \t\n\v\f\r]+")
_ROW_KINDS = {"N": MpsRowKind.n, "L": MpsRowKind.l, "G": MpsRowKind.g, "E": MpsRowKind.e}
_BOUND_KINDS = {"UP": MpsBoundKind.up, "LO": MpsBoundKind.lo, "FX": MpsBoundKind.fx,
                "FR": MpsBoundKind.fr, "MI": MpsBoundKind.mi, "PL": MpsBoundKind.pl,
                "BV": MpsBoundKind.bv}
# std::strtod's accepted spellings (C locale), anchored to the whole token
_DEC = re.compile(r"[+-]?([0-9]+\.?[0-9]*|\.[0-9]+)([eE][+-]?[0-9]+)?\Z")
_HEX = re.compile(r"[+-]?0[xX]([0-9a-fA-F]+\.?[0-9a-fA-F]*|\.[0-9a-fA-F]+)([pP][+-]?[0-9]+)?\Z")
_SPECIAL = re.compile(r"([+-]?)(inf|infinity|nan(\([0-9A-Za-z_]*\))?)\Z", re.IGNORECASE)


def _upper(s: str) -> str:
    return s.translate(_UPPER)


_UPPER = str.maketrans("abcdefghijklmnopqrstuvwxyz", "ABCDEFGHIJKLMNOPQRSTUVWXYZ")


def _tokenize(line: str) -> List[str]:
    return [t for t in _SPLIT.split(line) if t]


def _parse_number(tok: str, line_no: int) -> float:
    """mps.cpp:33-39: strtod over the whole token, else MalformedNumber."""
    if _DEC.match(tok):
        return float(tok)
    if _HEX.match(tok):
        neg = tok[0] == "-"
        body = tok[1:] if tok[0] in "+-" else tok
        if "p" not in body.lower():
            body += "p0"
        v = float.fromhex(body)
        return -v if neg else v
    sp = _SPECIAL.match(tok)
    if sp:
        v = math.nan if sp.group(2).lower().startswith("nan") else INF
        return -v if sp.group(1) == "-" else v
    raise MalformedNumber(tok, line_no)


def _format_exact(v: float) -> str:
    """mps.cpp:47-55: shortest of %.15g..%.17g that reads back exactly."""
    s = ""
    for prec in (15, 16, 17):
        s = "%.*g" % (prec, v)
        if float(s) == v:
            break
    return s


def parse_mps(text) -> MpsDocument:
    """lps::parse_mps (mps.cpp:59-210). ``text``: str or bytes of the file."""
    if isinstance(text, (bytes, bytearray)):
        text = bytes(text).decode("latin-1")
    doc = MpsDocument()
    section = _START
    row_names = set()
    saw_objsense_header = False
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()  # getline yields no record after a final newline
    for line_no, raw in enumerate(lines, 1):
        if raw.endswith("\r"):
            raw = raw[:-1]
        if not raw or raw[0] == "*":
            continue
        is_header = raw[0] not in _C_SPACE
        tok = _tokenize(raw)
        if not tok:
            continue
        if is_header:
            key = _upper(tok[0])
            if key == "ENDATA":
                section = _ENDATA
                break
            if key not in _HEADERS:
                raise UnknownSection(f"unknown section '{tok[0]}' at line {line_no}")
            nxt = _HEADERS[key]
            if key == "NAME":
                if len(tok) > 1:
                    doc.name = tok[1]
            elif key == "OBJSENSE":
                saw_objsense_header = True
                if len(tok) > 1:
                    v = _upper(tok[1])
                    doc.objsense = Sense.maximize if v in ("MAX", "MAXIMIZE") else Sense.minimize
                    saw_objsense_header = False
            if nxt <= section:
                raise UnknownSection(f"section '{tok[0]}' out of order at line {line_no}")
            section = nxt
            continue

        if section == _OBJSENSE:
            if saw_objsense_header:
                v = _upper(tok[0])
                doc.objsense = Sense.maximize if v in ("MAX", "MAXIMIZE") else Sense.minimize
                saw_objsense_header = False
        elif section == _ROWS:
            if len(tok) < 2:
                raise UnknownSection(f"bad ROWS line {line_no}")
            kind = _ROW_KINDS.get(_upper(tok[0]))
            if kind is None:
                raise UnknownSection(f"unknown row kind '{tok[0]}' at line {line_no}")
            if tok[1] in row_names:
                raise DuplicateRow(f"duplicate row '{tok[1]}' at line {line_no}")
            row_names.add(tok[1])
            doc.rows.append(MpsRow(kind, tok[1]))
        elif section == _COLUMNS:
            if "MARKER" in raw:  # also catches 'MARKER' (mps.cpp:139-144)
                doc.warnings.append(f"line {line_no}: MARKER record ignored")
                continue
            if len(tok) < 3 or len(tok) % 2 == 0:
                raise MalformedNumber(raw, line_no)
            for f in range(1, len(tok) - 1, 2):
                if tok[f] not in row_names:
                    raise UndeclaredRow(f"COLUMNS entry references undeclared row '{tok[f]}' "
                                        f"at line {line_no}")
                doc.columns.append(MpsEntry(tok[0], tok[f], _parse_number(tok[f + 1], line_no)))
        elif section in (_RHS, _RANGES):
            first = 1 if len(tok) % 2 == 1 else 0  # odd count: leading set name
            set_name = tok[0] if first else ""
            if len(tok) - first < 2:
                raise MalformedNumber(raw, line_no)
            dest = doc.rhs if section == _RHS else doc.ranges
            for f in range(first, len(tok) - 1, 2):
                if tok[f] not in row_names:
                    raise UndeclaredRow(f"entry references undeclared row '{tok[f]}' at line "
                                        f"{line_no}")
                dest.append(MpsEntry(set_name, tok[f], _parse_number(tok[f + 1], line_no)))
        elif section == _BOUNDS:
            if len(tok) < 3:
                raise UnknownSection(f"bad BOUNDS line {line_no}")
            kind = _BOUND_KINDS.get(_upper(tok[0]))
            if kind is None:
                raise UnknownSection(f"unknown bound kind '{tok[0]}' at line {line_no}")
            value = 0.0
            if kind in (MpsBoundKind.up, MpsBoundKind.lo, MpsBoundKind.fx):
                if len(tok) < 4:
                    raise MalformedNumber(raw, line_no)
                value = _parse_number(tok[3], line_no)
            doc.bounds.append(MpsBound(kind, tok[1], tok[2], value))
        else:
            raise UnknownSection(f"data before any section at line {line_no}")

    if section != _ENDATA:
        doc.missing_endata = True
        doc.warnings.append("missing ENDATA; accepted input as-is")
    if not any(r.kind == MpsRowKind.n for r in doc.rows):
        raise MissingObjectiveRow(f"no N row in '{doc.name}'")
    return doc


def parse_mps_file(path: str) -> MpsDocument:
    """lps::parse_mps_file (mps.cpp:217-221)."""
    try:
        with open(path, "rb") as f:
            data = f.read()
    except OSError:
        raise Error(f"cannot open '{path}'") from None
    return parse_mps(data)


def to_general_lp(doc: MpsDocument, warnings: Optional[List[str]] = None) -> GeneralLP:
    """lps::to_general_lp (mps.cpp:228-351): the first N row is the objective
    (later N rows are dropped with a warning), columns in order of first
    appearance, duplicate (column, row) cells summed with a warning, absent
    RHS entries zero, RHS on the objective row ignored with a warning, BV
    bounds rejected."""
    def warn(msg: str) -> None:
        if warnings is not None:
            warnings.append(msg)

    obj_row = None
    row_index = {}
    dropped = set()
    constraint_rows = []
    for row in doc.rows:
        if row.kind == MpsRowKind.n:
            if obj_row is None:
                obj_row = row.name
            else:
                dropped.add(row.name)
                warn(f"extra N row '{row.name}' dropped")
            continue
        row_index.setdefault(row.name, len(constraint_rows))
        constraint_rows.append(row)

    col_index = {}
    for e in doc.columns:
        col_index.setdefault(e.column, len(col_index))

    lp = GeneralLP(name=doc.name, sense=doc.objsense)
    lp.resize(len(constraint_rows), len(col_index))
    for i, row in enumerate(constraint_rows):
        lp.row_kind[i] = {MpsRowKind.l: RowKind.le, MpsRowKind.g: RowKind.ge}.get(row.kind,
                                                                                 RowKind.eq)
    seen = set()
    # accumulate in file order (each += is one IEEE add, like mps.cpp:292-296)
    for e in doc.columns:
        j = col_index[e.column]
        if (e.column, e.row) in seen:
            warn(f"duplicate COLUMNS entry ({e.column}, {e.row}) summed")
        else:
            seen.add((e.column, e.row))
        if e.row == obj_row:
            lp.objective[j] = lp.objective[j] + e.value
        elif e.row in row_index:
            i = row_index[e.row]
            lp.coeffs[i, j] = lp.coeffs[i, j] + e.value
        # entries on dropped N rows are ignored

    for e in doc.rhs:
        if e.row == obj_row:
            warn(f"RHS entry on objective row '{e.row}' ignored")
        elif e.row in row_index:
            lp.rhs[row_index[e.row]] = e.value
        elif e.row not in dropped:
            raise UndeclaredRow(f"RHS entry for unknown row '{e.row}'")

    for e in doc.ranges:
        if e.row in row_index:
            lp.range[row_index[e.row]] = e.value
        elif e.row not in dropped and e.row != obj_row:
            raise UndeclaredRow(f"RANGES entry for unknown row '{e.row}'")

    for bd in doc.bounds:
        j = col_index.get(bd.column)
        if j is None:
            warn(f"bound on unknown column '{bd.column}' ignored")
            continue
        k = bd.kind
        if k == MpsBoundKind.up:
            lp.upper[j] = bd.value
            if bd.value < 0.0 and lp.lower[j] == 0.0:
                warn(f"negative UP bound on '{bd.column}' keeps lower bound 0")
        elif k == MpsBoundKind.lo:
            lp.lower[j] = bd.value
        elif k == MpsBoundKind.fx:
            lp.lower[j] = lp.upper[j] = bd.value
        elif k == MpsBoundKind.fr:
            lp.lower[j], lp.upper[j] = -INF, INF
        elif k == MpsBoundKind.mi:
            lp.lower[j] = -INF
        elif k == MpsBoundKind.pl:
            lp.upper[j] = INF
        else:
            raise UnsupportedBoundKind(f"BV bound on '{bd.column}': integer variables are not "
                                       f"supported")
    return lp


def _pad(s: str, w: int) -> str:
    return s + " " if len(s) >= w else s + " " * (w - len(s))


def write_mps(doc: MpsDocument) -> str:
    """lps::write_mps (mps.cpp:353-401): parse_mps(write_mps(doc)) == doc."""
    out = [f"NAME          {doc.name}\n"]
    if doc.objsense == Sense.maximize:
        out.append("OBJSENSE\n    MAX\n")
    out.append("ROWS\n")
    for r in doc.rows:
        out.append(f" {'NLGE'[int(r.kind)]}  {r.name}\n")

    def entries(header, es):
        out.append(header + "\n")
        for e in es:
            out.append("    " + _pad(e.column, 10) + _pad(e.row, 10) + _format_exact(e.value) + "\n")

    entries("COLUMNS", doc.columns)
    entries("RHS", doc.rhs)
    if doc.ranges:
        entries("RANGES", doc.ranges)
    if doc.bounds:
        out.append("BOUNDS\n")
        for bd in doc.bounds:
            line = f" {bd.kind.name.upper()} " + _pad(bd.set, 10) + _pad(bd.column, 10)
            if bd.kind in (MpsBoundKind.up, MpsBoundKind.lo, MpsBoundKind.fx):
                line += _format_exact(bd.value)
            out.append(line + "\n")
    out.append("ENDATA\n")
    return "".join(out)


def to_mps_document(lp: GeneralLP) -> MpsDocument:
    """lps::to_mps_document (mps.cpp:403-427): rows R1..Rm, columns X1..Xn,
    objective row COST; zero coefficients and default bounds omitted."""
    doc = MpsDocument(name=lp.name or "LP", objsense=lp.sense)
    doc.rows.append(MpsRow(MpsRowKind.n, "COST"))
    kinds = {RowKind.eq: MpsRowKind.e, RowKind.le: MpsRowKind.l, RowKind.ge: MpsRowKind.g}
    for i in range(lp.num_rows):
        doc.rows.append(MpsRow(kinds.get(RowKind(lp.row_kind[i]), MpsRowKind.n), f"R{i + 1}"))
    A = np.asarray(lp.coeffs, np.float64).reshape(lp.num_rows, lp.num_cols)
    for j in range(lp.num_cols):
        if lp.objective[j] != 0.0:
            doc.columns.append(MpsEntry(f"X{j + 1}", "COST", float(lp.objective[j])))
        for i in np.nonzero(A[:, j])[0]:
            doc.columns.append(MpsEntry(f"X{j + 1}", f"R{i + 1}", float(A[i, j])))
    if lp.objective_constant != 0.0:
        doc.rhs.append(MpsEntry("RHS", "COST", float(lp.objective_constant)))
    for i in range(lp.num_rows):
        if lp.rhs[i] != 0.0:
            doc.rhs.append(MpsEntry("RHS", f"R{i + 1}", float(lp.rhs[i])))
    for i in range(lp.num_rows):
        if lp.range[i] is not None:
            doc.ranges.append(MpsEntry("RNG", f"R{i + 1}", float(lp.range[i])))
    for j in range(lp.num_cols):
        lo, hi, name = float(lp.lower[j]), float(lp.upper[j]), f"X{j + 1}"
        if lo == 0.0 and hi == INF:
            continue
        if lo == hi:
            doc.bounds.append(MpsBound(MpsBoundKind.fx, "BND", name, lo))
            continue
        if lo == -INF and hi == INF:
            doc.bounds.append(MpsBound(MpsBoundKind.fr, "BND", name, 0.0))
            continue
        if lo == -INF:
            doc.bounds.append(MpsBound(MpsBoundKind.mi, "BND", name, 0.0))
        elif lo != 0.0:
            doc.bounds.append(MpsBound(MpsBoundKind.lo, "BND", name, lo))
        if hi != INF:
            doc.bounds.append(MpsBound(MpsBoundKind.up, "BND", name, hi))
    return doc


def _read(src) -> MpsDocument:
    if isinstance(src, (bytes, bytearray)) or (isinstance(src, str) and "\n" in src):
        return parse_mps(src)
    return parse_mps_file(src)


def load_mps(src, warnings: Optional[List[str]] = None,
             pinned: bool = False) -> Tuple[StandardFormLP, CanonicalMap]:
    """parse_mps(_file) + to_general_lp + canonicalize (lps_main.cpp:110-112).
    ``src``: a path, or the MPS text itself (str with newlines, or bytes)."""
    doc = _read(src)
    if warnings is not None:
        warnings.extend(doc.warnings)
    lp, mp = canonicalize(to_general_lp(doc, warnings), pinned=pinned)
    if not lp.name:
        lp.name = doc.name
    return lp, mp


@dataclass
class MpsSolveResult:
    """What the reference CLI's ``solve`` reports (lps_main.cpp:113-128)."""
    report: SolveReport
    objective: float                    # in the original sense (recovered)
    x: Optional[np.ndarray]             # original variables, when recovered
    lp: StandardFormLP
    map: CanonicalMap


def solve_mps(src, cfg: Optional[SolverConfig] = None) -> MpsSolveResult:
    """The reference CLI's solve path (lps_main.cpp:110-118) on the GPU: load,
    two_phase_solve, and recover_solution for optimal / iteration-limit
    reports (other statuses keep the solver's objective, as the CLI does)."""
    from .solver import two_phase_solve
    lp, mp = load_mps(src)
    rep = two_phase_solve(lp, cfg)
    obj, x = rep.objective, None
    if rep.status in (SolveStatus.optimal, SolveStatus.iteration_limit):
        x, obj = recover_solution(mp, rep.x, rep.objective)
    return MpsSolveResult(rep, obj, x, lp, mp)
