"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes front-end for the two CPU checkers built by oracle/Makefile:

* ``Ref``  — oracle/_ref/liblps_ref.so: the unmodified reference library
  (/root/reference/proj/src/*.cpp) behind oracle/ref_shim.cpp.
* ``Port`` — oracle/_build/liblps_port.so: our plain-C restatement
  (oracle/lps_oracle.c).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module. The product package never
does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SO = os.path.join(HERE, "_ref", "liblps_ref.so")
PORT_SO = os.path.join(HERE, "_build", "liblps_port.so")

STATUS_NAMES = {0: "Optimal", 1: "Unbounded", 2: "Infeasible", 3: "IterationLimit",
                -1: "Error", -2: "PivotTooSmall"}


class Config(C.Structure):
    _fields_ = [("opt_tol", C.c_double), ("pivot_tol", C.c_double), ("feas_tol", C.c_double),
                ("ratio_tie_tol", C.c_double), ("max_iter", C.c_long), ("anticycle", C.c_int),
                ("workers", C.c_int), ("kernel", C.c_int)]


class TraceEntry(C.Structure):
    _fields_ = [("iteration", C.c_long), ("phase", C.c_int), ("row", C.c_int),
                ("leaving", C.c_int), ("entering", C.c_int), ("objective", C.c_double)]


class Result(C.Structure):
    _fields_ = [("status", C.c_int), ("objective", C.c_double),
                ("iterations_phase1", C.c_long), ("iterations_phase2", C.c_long),
                ("total_seconds", C.c_double), ("tpi_seconds", C.c_double),
                ("trace_len", C.c_long)]


TRACE_DTYPE = np.dtype([("iteration", np.int64), ("phase", np.int32), ("row", np.int32),
                        ("leaving", np.int32), ("entering", np.int32),
                        ("objective", np.float64)])
assert TRACE_DTYPE.itemsize == C.sizeof(TraceEntry)


@dataclass
class LP:
    """Mirror of lps::StandardFormLP (lp_model.hpp:49-60)."""
    m: int
    n_total: int
    A: np.ndarray          # (m, n_total) float64, row-major
    b: np.ndarray          # (m,)
    c: np.ndarray          # (n_total,)
    col_kind: np.ndarray   # (n_total,) uint8: 0 structural, 1 slack
    objective_sign: float = 1.0
    objective_constant: float = 0.0
    name: str = ""


@dataclass
class SolveOut:
    status: int
    objective: float
    iterations_phase1: int
    iterations_phase2: int
    total_seconds: float
    tpi_seconds: float
    x: np.ndarray
    trace: np.ndarray = field(default_factory=lambda: np.zeros(0, TRACE_DTYPE))
    trace_len: int = 0

    @property
    def status_name(self) -> str:
        return STATUS_NAMES.get(self.status, str(self.status))


def make_config(opt_tol=1e-7, pivot_tol=1e-9, feas_tol=1e-7, ratio_tie_tol=1e-9, max_iter=0,
                anticycle="tabu", workers=1, kernel="cached") -> Config:
    return Config(opt_tol, pivot_tol, feas_tol, ratio_tie_tol, int(max_iter),
                  1 if anticycle == "none" else 0, int(workers), 1 if kernel == "naive" else 0)


def build(ref: bool = True) -> None:
    """Builds the checkers (make; the reference half only if its sources exist)."""
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


def _ptr(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class _Lib:
    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        self.prefix = prefix
        solve = getattr(self.lib, prefix + "solve")
        solve.restype = C.c_int
        solve.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                          C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.POINTER(Config),
                          C.POINTER(Result), C.POINTER(C.c_double), C.c_void_p, C.c_long]
        self._solve = solve

    def solve(self, lp: LP, cfg: Config | None = None, trace_cap: int = 1 << 20,
              **kw) -> SolveOut:
        cfg = cfg or make_config(**kw)
        A = np.ascontiguousarray(lp.A, dtype=np.float64)
        b = np.ascontiguousarray(lp.b, dtype=np.float64)
        c = np.ascontiguousarray(lp.c, dtype=np.float64)
        ck = np.ascontiguousarray(lp.col_kind, dtype=np.uint8)
        x = np.zeros(lp.n_total, np.float64)
        tr = np.zeros(max(trace_cap, 0), TRACE_DTYPE)
        res = Result()
        rc = self._solve(lp.m, lp.n_total, _ptr(A, C.c_double), _ptr(b, C.c_double),
                         _ptr(c, C.c_double), _ptr(ck, C.c_uint8), C.byref(cfg), C.byref(res),
                         _ptr(x, C.c_double), tr.ctypes.data if trace_cap > 0 else None,
                         trace_cap)
        if rc == 1:
            raise RuntimeError(self.last_error())
        n = min(res.trace_len, trace_cap)
        return SolveOut(res.status, res.objective, res.iterations_phase1, res.iterations_phase2,
                        res.total_seconds, res.tpi_seconds, x, tr[:n].copy(), res.trace_len)

    def last_error(self) -> str:
        return ""


class Ref(_Lib):
    """The compiled, unmodified reference (oracle/_ref)."""

    def __init__(self, path: str = REF_SO):
        super().__init__(path, "ref_")
        L = self.lib
        L.ref_lp_generate.restype = C.c_void_p
        L.ref_lp_generate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int]
        L.ref_lp_from_mps.restype = C.c_void_p
        L.ref_lp_from_mps.argtypes = [C.c_char_p]
        L.ref_lp_dims.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_lp_copy.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                  C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_lp_free.argtypes = [C.c_void_p]
        L.ref_last_error.restype = C.c_char_p

    def last_error(self) -> str:
        return self.lib.ref_last_error().decode()

    def solve_window(self, lp: LP, cfg: Config, warmup: int, steps: int):
        """bench.py's reference arm: two_phase_solve with max_iter = warmup +
        steps and per-pivot timestamps (ref_solve_timed); returns (seconds of
        pivots [warmup, warmup + steps), pivots done in that window, SolveOut-ish
        dict)."""
        L = self.lib
        L.ref_solve_timed.restype = C.c_int
        L.ref_solve_timed.argtypes = [C.c_int, C.c_int, C.POINTER(C.c_double), C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_uint8), C.POINTER(Config),
                                      C.POINTER(Result), C.POINTER(C.c_double), C.c_long,
                                      C.POINTER(C.c_double)]
        cfg.max_iter = int(warmup + steps)
        A = np.ascontiguousarray(lp.A, dtype=np.float64)
        b = np.ascontiguousarray(lp.b, dtype=np.float64)
        c = np.ascontiguousarray(lp.c, dtype=np.float64)
        ck = np.ascontiguousarray(lp.col_kind, dtype=np.uint8)
        stamps = np.zeros(warmup + steps + 1)
        res = Result()
        t_ret = C.c_double()
        rc = L.ref_solve_timed(lp.m, lp.n_total, _ptr(A, C.c_double), _ptr(b, C.c_double),
                               _ptr(c, C.c_double), _ptr(ck, C.c_uint8), C.byref(cfg), C.byref(res),
                               _ptr(stamps, C.c_double), len(stamps), C.byref(t_ret))
        if rc != 0:
            raise RuntimeError(self.last_error())
        n = int(res.trace_len)
        done = max(0, min(n, warmup + steps) - warmup)
        if done == 0:
            return 0.0, 0, res
        t0 = stamps[warmup - 1] if warmup > 0 else t_ret.value - res.total_seconds
        return float(stamps[warmup + done - 1] - t0), done, res

    def _take(self, h, name="") -> LP:
        if not h:
            raise RuntimeError(self.last_error())
        m, n = C.c_int(), C.c_int()
        self.lib.ref_lp_dims(h, C.byref(m), C.byref(n))
        m, n = m.value, n.value
        A = np.zeros((m, n)); b = np.zeros(m); c = np.zeros(n)
        ck = np.zeros(n, np.uint8)
        sgn, const = C.c_double(), C.c_double()
        self.lib.ref_lp_copy(h, _ptr(A, C.c_double), _ptr(b, C.c_double), _ptr(c, C.c_double),
                             _ptr(ck, C.c_uint8), C.byref(sgn), C.byref(const))
        self.lib.ref_lp_free(h)
        return LP(m, n, A, b, c, ck, sgn.value, const.value, name)

    def generate(self, rows: int, cols: int, seed: int = 1, form: int = 0,
                 sparsity: int = 0) -> LP:
        return self._take(self.lib.ref_lp_generate(rows, cols, sparsity, seed, form),
                          f"{rows}_{cols}_f{form}_s{seed}")

    # ---- MPS ingestion chain on in-memory text (ref_shim.cpp ref_mps_*) ----
    def _mps_sigs(self):
        L = self.lib
        if getattr(self, "_mps_ready", False):
            return L
        L.ref_mps_load.restype = C.c_void_p
        L.ref_mps_load.argtypes = [C.c_char_p]
        L.ref_last_error_kind.restype = C.c_char_p
        L.ref_mps_warnings.restype = C.c_char_p
        L.ref_mps_warnings.argtypes = [C.c_void_p]
        L.ref_mps_written.restype = C.c_char_p
        L.ref_mps_written.argtypes = [C.c_void_p]
        L.ref_mps_map.argtypes = [C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                  C.POINTER(C.c_double), C.POINTER(C.c_uint8),
                                  C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_mps_recover.restype = C.c_int
        L.ref_mps_recover.argtypes = [C.c_void_p, C.POINTER(C.c_double), C.c_int, C.c_double,
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]
        L.ref_generated_mps.restype = C.c_char_p
        L.ref_generated_mps.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int]
        self._mps_ready = True
        return L

    def mps_load(self, text) -> dict:
        """parse_mps + to_general_lp + canonicalize on `text`. Returns the
        standard form, the CanonicalMap, the warnings and write_mps(doc), or
        {"error_kind", "error"} when the reference throws."""
        L = self._mps_sigs()
        data = text.encode("latin-1") if isinstance(text, str) else bytes(text)
        h = L.ref_mps_load(data)
        if not h:
            return {"error_kind": L.ref_last_error_kind().decode(), "error": self.last_error()}
        m, n = C.c_int(), C.c_int()
        L.ref_lp_dims(h, C.byref(m), C.byref(n))
        m, n = m.value, n.value
        oc, ns = C.c_int(), C.c_int()
        L.ref_mps_map(h, C.byref(oc), C.byref(ns), None, None, None, None)
        shift = np.zeros(oc.value); neg = np.zeros(m, np.uint8)
        sp = np.zeros(max(ns.value, 1), np.int32); sn = np.zeros(max(ns.value, 1), np.int32)
        L.ref_mps_map(h, C.byref(oc), C.byref(ns), _ptr(shift, C.c_double), _ptr(neg, C.c_uint8),
                      _ptr(sp, C.c_int), _ptr(sn, C.c_int))
        out = {"warnings": L.ref_mps_warnings(h).decode("latin-1"),
               "written": L.ref_mps_written(h).decode("latin-1"),
               "shift": shift, "negated_row": neg, "split_pos": sp[:ns.value],
               "split_neg": sn[:ns.value], "_h": h}
        A = np.zeros((m, n)); b = np.zeros(m); c = np.zeros(n)
        ck = np.zeros(n, np.uint8)
        sgn, const = C.c_double(), C.c_double()
        L.ref_lp_copy(h, _ptr(A, C.c_double), _ptr(b, C.c_double), _ptr(c, C.c_double),
                      _ptr(ck, C.c_uint8), C.byref(sgn), C.byref(const))
        out["lp"] = LP(m, n, A, b, c, ck, sgn.value, const.value, "")
        return out

    def mps_recover(self, loaded: dict, x_std, z_std: float):
        L = self._mps_sigs()
        x_std = np.ascontiguousarray(x_std, np.float64)
        x = np.zeros(len(loaded["shift"])); z = C.c_double()
        if L.ref_mps_recover(loaded["_h"], _ptr(x_std, C.c_double), len(x_std), float(z_std),
                             _ptr(x, C.c_double), C.byref(z)):
            raise RuntimeError(L.ref_last_error_kind().decode() + ": " + self.last_error())
        return x, z.value

    def mps_free(self, loaded: dict) -> None:
        if loaded.get("_h"):
            self.lib.ref_lp_free(loaded.pop("_h"))

    def generated_mps(self, rows: int, cols: int, seed: int = 1, form: int = 0,
                      sparsity: int = 0) -> str:
        L = self._mps_sigs()
        t = L.ref_generated_mps(rows, cols, sparsity, seed, form)
        if t is None:
            raise RuntimeError(self.last_error())
        return t.decode("latin-1")

    def from_mps(self, path: str) -> LP:
        return self._take(self.lib.ref_lp_from_mps(path.encode()),
                          os.path.splitext(os.path.basename(path))[0])


class Port(_Lib):
    """Our plain-C restatement (oracle/lps_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        super().__init__(path, "lpo_")
        L = self.lib
        L.lpo_generate.restype = C.c_int
        L.lpo_generate.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int,
                                   C.POINTER(C.c_double), C.POINTER(C.c_double),
                                   C.POINTER(C.c_double), C.POINTER(C.c_uint8)]
        L.lpo_generated_n_total.restype = C.c_int
        L.lpo_generated_n_total.argtypes = [C.c_int, C.c_int, C.c_int]

    def solve_with_ties(self, lp: LP, cfg: Config, cap_ties: int = 64, cap_rows: int = 1 << 16):
        """solve() plus the lookahead scores of every scored tie (lpo_set_tie_log):
        returns (SolveOut, [(pivots_before, entering, rows, scores), ...])."""
        L = self.lib
        L.lpo_set_tie_log.argtypes = [C.c_void_p, C.c_long, C.c_void_p, C.c_void_p, C.c_long]
        L.lpo_tie_log_len.restype = C.c_long
        meta = np.zeros(4 * cap_ties, np.int64)
        rows = np.zeros(cap_rows, np.int32)
        scores = np.zeros(cap_rows, np.float64)
        L.lpo_set_tie_log(meta.ctypes.data, cap_ties, rows.ctypes.data, scores.ctypes.data, cap_rows)
        try:
            out = self.solve(lp, cfg)
            n = L.lpo_tie_log_len()
        finally:
            L.lpo_set_tie_log(None, 0, None, None, 0)
        ties = []
        for k in range(n):
            it, q, off, cnt = (int(v) for v in meta[4 * k: 4 * k + 4])
            ties.append((it, q, rows[off: off + cnt].copy(), scores[off: off + cnt].copy()))
        return out, ties

    def generate(self, rows: int, cols: int, seed: int = 1, form: int = 0,
                 sparsity: int = 0) -> LP:
        n = self.lib.lpo_generated_n_total(rows, cols, form)
        A = np.zeros((rows, n)); b = np.zeros(rows); c = np.zeros(n)
        ck = np.zeros(n, np.uint8)
        rc = self.lib.lpo_generate(rows, cols, sparsity, seed, form, _ptr(A, C.c_double),
                                   _ptr(b, C.c_double), _ptr(c, C.c_double), _ptr(ck, C.c_uint8))
        if rc:
            raise ValueError("lpo_generate: rows and cols must be positive")
        return LP(rows, n, A, b, c, ck, -1.0 if form else 1.0, 0.0,
                  f"{rows}_{cols}_f{form}_s{seed}")


def save_lp(path: str, lp: LP) -> None:
    np.savez_compressed(path, m=lp.m, n_total=lp.n_total, A=lp.A, b=lp.b, c=lp.c,
                        col_kind=lp.col_kind, objective_sign=lp.objective_sign,
                        objective_constant=lp.objective_constant, name=lp.name)


def load_lp(path: str) -> LP:
    z = np.load(path, allow_pickle=False)
    return LP(int(z["m"]), int(z["n_total"]), z["A"], z["b"], z["c"], z["col_kind"],
              float(z["objective_sign"]), float(z["objective_constant"]), str(z["name"]))
