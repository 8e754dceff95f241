"""Benchmark-harness compatibility with the reference.

Mirrors /root/reference/proj/include/lps/bench.hpp so reference tooling can
read lpsg results unchanged:

* ``speedup`` / ``tpi``                       bench.cpp:14-25 (same errors)
* ``status_name`` / ``case_name``             bench.cpp:27-38
* ``BenchRow`` + ``CSV_HEADER``               bench.hpp:24-44 (the CSV schema, field for field)
* ``write_csv`` / ``read_csv``                bench.hpp:46-49 (reals as ``%.6g``; read(write(x)) == x)
* ``timed_solve`` (median of ``runs``)        bench.cpp:137-151
* ``run_suite``                               bench.cpp:155-215 (one row per instance; failures
                                              become ``ParseError`` rows and never abort)

The reference's ``device_reads``/``device_writes`` are simulated access
counters of its fake device; here they are the algorithmic HBM bytes the
solve's kernels had to read / write, and ``h2d_bytes`` /
``d2h_bytes`` are the real transfer counters of the C ABI.
"""
from __future__ import annotations

import statistics
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

from .lp_model import _cxx_to_string
from .solver import (Error, GenSpec, SimplexSolver, SolverConfig, SolveStatus, StandardFormLP,
                     generate)

# bench.hpp:40-43
CSV_HEADER = ("instance,status,objective,iterations_p1,iterations_p2,total_seconds,"
              "tpi_seconds,case,device_reads,device_writes,h2d_bytes,d2h_bytes,"
              "reference_seconds,speedup")


class NonPositiveTime(Error):
    """lps::NonPositiveTime (errors.hpp)."""


class ZeroIterations(Error):
    """lps::ZeroIterations (errors.hpp)."""


def speedup(t_ref: float, t_par: float) -> float:
    if t_par <= 0.0:
        raise NonPositiveTime(f"speedup: t_par must be positive, got {_cxx_to_string(t_par)}")
    return t_ref / t_par


def tpi(total_seconds: float, iterations: int) -> float:
    if iterations < 1:
        raise ZeroIterations("tpi: iteration count must be at least 1")
    return total_seconds / float(iterations)


def status_name(s: SolveStatus) -> str:
    return {SolveStatus.optimal: "Optimal", SolveStatus.unbounded: "Unbounded",
            SolveStatus.infeasible: "Infeasible"}.get(SolveStatus(s), "IterationLimit")


def case_name(in_core: bool = True) -> str:
    return "InCore" if in_core else "Tiled"


@dataclass
class BenchRow:
    """lps::BenchRow (bench.hpp:24-38)."""
    instance: str
    status: str
    objective: float = 0.0
    iterations_p1: int = 0
    iterations_p2: int = 0
    total_seconds: float = 0.0
    tpi_seconds: float = 0.0
    case_used: str = ""
    device_reads: int = 0
    device_writes: int = 0
    h2d_bytes: int = 0
    d2h_bytes: int = 0
    reference_seconds: Optional[float] = None
    speedup: Optional[float] = None


def _fmt6(v: float) -> str:
    return "%.6g" % v


def write_csv(rows: Sequence[BenchRow]) -> str:
    out = [CSV_HEADER]
    for r in rows:
        out.append(",".join([
            r.instance, r.status, _fmt6(r.objective), str(r.iterations_p1), str(r.iterations_p2),
            _fmt6(r.total_seconds), _fmt6(r.tpi_seconds), r.case_used, str(r.device_reads),
            str(r.device_writes), str(r.h2d_bytes), str(r.d2h_bytes),
            "" if r.reference_seconds is None else _fmt6(r.reference_seconds),
            "" if r.speedup is None else _fmt6(r.speedup)]))
    return "\n".join(out) + "\n"


def read_csv(text: str) -> List[BenchRow]:
    lines = [ln for ln in text.splitlines() if ln]
    if not lines or lines[0] != CSV_HEADER:
        raise Error("read_csv: missing or unexpected header")
    rows = []
    for ln in lines[1:]:
        f = ln.split(",")
        if len(f) != 14:
            raise Error(f"read_csv: expected 14 fields, got {len(f)}")
        rows.append(BenchRow(f[0], f[1], float(f[2]), int(f[3]), int(f[4]), float(f[5]),
                             float(f[6]), f[7], int(f[8]), int(f[9]), int(f[10]), int(f[11]),
                             float(f[12]) if f[12] else None, float(f[13]) if f[13] else None))
    return rows


def _algorithmic_bytes(lp: StandardFormLP, iterations: int):
    """(reads, writes) of the fused pivot schedule: pricing reads the
    nonbasic A (bounded by m x n_total), the update+FTRAN reads and writes B^-1|b."""
    m, n = lp.m, lp.n_total
    reads = iterations * 8 * (m * n + (m + 1) * (m + 1))
    writes = iterations * 8 * (m + 1) * (m + 1)
    return int(reads), int(writes)


def timed_solve(lp: StandardFormLP, cfg: Optional[SolverConfig] = None, runs: int = 1):
    """bench.cpp:137-151: median total_seconds over `runs` solves; the last
    report carries the other fields, tpi recomputed from the median."""
    times, rep, counters = [], None, None
    for _ in range(max(1, runs)):
        with SimplexSolver(lp, cfg) as s:
            rep = s.solve()
            counters = s.counters()
        times.append(rep.total_seconds)
    rep.total_seconds = statistics.median(times)
    rep.tpi_seconds = rep.total_seconds / max(1, rep.iterations)
    return rep, counters


def run_suite(instances: Sequence, cfg: Optional[SolverConfig] = None, runs: int = 1,
              reference: Optional[Callable[[StandardFormLP], float]] = None) -> List[BenchRow]:
    """bench.cpp:155-215. `instances`: (label, StandardFormLP | GenSpec | MPS path)
    pairs; an MPS file goes through parse + to_general_lp + canonicalize
    (mps.py) like the reference's suite loader (bench.cpp:160-166).
    `reference(lp)`, when given, returns the reference run's seconds (the
    reference harness uses a single-worker naive-kernel solve, 174-181)."""
    rows = []
    for label, inst in instances:
        mp = None
        try:
            if isinstance(inst, GenSpec):
                lp = generate(inst)
            elif isinstance(inst, str):
                from .mps import load_mps
                lp, mp = load_mps(inst)
            else:
                lp = inst
        except Exception:  # noqa: BLE001 - a ParseError row, like load_instance (bench.cpp:119-131)
            rows.append(BenchRow(label, "ParseError", objective=float("nan")))
            continue
        rep, cnt = timed_solve(lp, cfg, runs)
        it = rep.iterations
        rd, wr = _algorithmic_bytes(lp, it)
        obj = rep.objective
        if rep.status in (SolveStatus.optimal, SolveStatus.iteration_limit):
            # recover_solution's objective (bench.cpp:191-195); generated
            # instances carry only the sign and constant of their map
            if mp is not None:
                from .lp_model import recover_solution
                obj = recover_solution(mp, rep.x, rep.objective)[1]
            else:
                obj = lp.objective_sign * rep.objective + lp.objective_constant
        row = BenchRow(label, status_name(rep.status), obj, rep.iterations_phase1,
                       rep.iterations_phase2, rep.total_seconds, rep.tpi_seconds, case_name(True),
                       rd, wr, int(cnt["h2d_bytes"]), int(cnt["d2h_bytes"]))
        if reference is not None and rep.total_seconds > 0.0:
            row.reference_seconds = float(reference(lp))
            row.speedup = speedup(row.reference_seconds, row.total_seconds)
        rows.append(row)
    return rows
