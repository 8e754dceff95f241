"""Python mirror of the reference solver API (/root/reference/proj/include/lps/solver.hpp).

Same names, argument meaning and error behaviour as the reference:

* ``two_phase_solve(lp, cfg)``          solver.hpp:173 / solver.cpp:394-397
* ``SimplexSolver`` step API             solver.hpp:79-168
* ``SolverConfig`` / ``SolveReport``     solver.hpp:34-57
* ``StandardFormLP``                     lp_model.hpp:49-60
* ``generate(GenSpec)`` (+ input forms)  generator.cpp:35-72
* errors ``PivotTooSmall`` etc.          errors.hpp

Every call goes through the C ABI of the CUDA library (include/lpsg.h); there
is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import numpy as np

from . import _lib as L


# ------------------------------------------------------------------ errors --
class Error(RuntimeError):
    """lps::Error (errors.hpp:9-11)."""


class PivotTooSmall(Error):
    """lps::PivotTooSmall (errors.hpp:58-60)."""


class DegenerateSpec(Error):
    """lps::DegenerateSpec / EmptyProblem (errors.hpp:66-68, 17-19)."""


class CudaError(Error):
    """Device failure (no CUDA device, launch error, out of memory)."""


class BudgetTooSmall(Error):
    """lps::BudgetTooSmall (tiled_engine.cpp:43-47)."""


_ERRORS = {1: PivotTooSmall, 2: CudaError, 3: CudaError, 4: Error, 5: CudaError, 6: DegenerateSpec,
           7: BudgetTooSmall}


def _check(rc: int) -> None:
    if rc != 0:
        msg = L.load().lpsg_last_error().decode()
        raise _ERRORS.get(rc, Error)(msg)


# ------------------------------------------------------------------- types --
# One pivot of the trace (include/lpsg.h lpsg_trace), as a numpy record.
TRACE_DTYPE = np.dtype([("iteration", np.int64), ("phase", np.int32), ("row", np.int32),
                        ("leaving", np.int32), ("entering", np.int32),
                        ("objective", np.float64)])

class SolveStatus(enum.IntEnum):
    """lps::SolveStatus (solver.hpp:14)."""
    optimal = 0
    unbounded = 1
    infeasible = 2
    iteration_limit = 3


class Anticycle(enum.IntEnum):
    tabu = 0
    none = 1


class ColKind(enum.IntEnum):
    structural = 0
    slack = 1
    artificial = 2


@dataclass
class SolverConfig:
    """lps::SolverConfig (solver.hpp:34-45) plus device placement."""
    opt_tol: float = 1e-7
    pivot_tol: float = 1e-9
    feas_tol: float = 1e-7
    ratio_tie_tol: float = 1e-9
    max_iter: int = 0
    anticycle: Anticycle = Anticycle.tabu
    kernel: int = 0          # KernelMode (tiled_engine.hpp): 0 cached (zero-skip), 1 naive
                             # (every element stored); the two differ only in zero signs
    workers: int = 1         # accepted, ignored (solver.hpp:43)
    device: int = 0
    batch: int = 0
    observer: Optional[Callable[["IterationView"], None]] = None
    observer_rows: bool = False  # view.row(i) readable in the observer (unfused, one pivot per round trip)
    # sharded solve over NCCL: one process per GPU, same problem
    # and config on every rank, nccl_id from nccl_unique_id() on rank 0
    world_size: int = 1
    rank: int = 0
    nccl_id: bytes = b""
    nccl_single: bool = False  # run the NCCL exchange path even for world_size 1 (testing)
    peer: Optional["PeerHeap"] = None  # P2P transport (NVLink stores + flags) instead of NCCL
    # verification modes, result-identical to the default (tests/test_gpu_parity.py):
    unfused_ratio: bool = False           # standalone ratio-test kernel, not the fused epilogue
    lookahead_exact_select: bool = False  # theta' keeps the y_i == 0 select
    # select_leaving's bounded selection: "auto" from 16
    # survivors up, "always" on every tie (verification), "off" (A/B)
    lookahead_bound: str = "auto"
    # opt-in periodic reinversion on the device (NOT bit-identical to the
    # reference; include/lpsg.h lpsg_config.reinvert_every): 0 = off
    reinvert_every: int = 0
    # lps::SolverConfig::memory_budget (solver.hpp:41): device bytes for the
    # tableau; over it the solve runs Case 2 (out-of-core, tiled). 0 = unlimited.
    memory_budget: int = 0

    def _c(self) -> L.Config:
        c = L.Config()
        L.load().lpsg_config_default(C.byref(c))
        c.opt_tol, c.pivot_tol, c.feas_tol = self.opt_tol, self.pivot_tol, self.feas_tol
        c.ratio_tie_tol, c.max_iter = self.ratio_tie_tol, int(self.max_iter)
        c.anticycle, c.kernel, c.workers = int(self.anticycle), int(self.kernel), int(self.workers)
        c.device, c.batch = int(self.device), int(self.batch)
        c.reserved[0] = 1 if self.unfused_ratio else 0
        c.world_size, c.rank = int(self.world_size), int(self.rank)
        c.reserved[1] = 1 if self.nccl_single else 0
        c.peer = self.peer.ptr if self.peer is not None else None
        c.reinvert_every = int(self.reinvert_every)
        c.memory_budget = int(self.memory_budget)
        # (tools/dbg set `_experiment` on an instance; it only has an effect in
        # the -DLPSG_EXPERIMENTS library, LPSG_EXPERIMENTS_LIB=1)
        if self.lookahead_bound not in ("auto", "always", "off"):
            raise Error(f"lookahead_bound must be auto, always or off, got {self.lookahead_bound!r}")
        c.reserved[2] = (16 if self.lookahead_exact_select else 0) | (
            {"auto": 0, "always": 32, "off": 64}[self.lookahead_bound]) | (
            int(getattr(self, "_experiment", 0)) & ~(16 | 32 | 64))
        if self.nccl_id:
            if len(self.nccl_id) != 128:
                raise Error("nccl_id must be 128 bytes")
            C.memmove(c.nccl_id, bytes(self.nccl_id), 128)
        return c


@dataclass
class IterationView:
    """Per-pivot snapshot (solver.hpp:21-32): phase, cumulative iteration,
    T[0][m], the whole basis, the pivot (row, leaving, entering), the memory
    counters, and -- with SolverConfig.observer_rows -- `row(i)`, the i-th
    tableau row of row_width doubles (row 0 = [W | obj | d])."""
    phase: int
    iteration: int
    objective: float
    row: int
    leaving: int
    entering: int
    basic: np.ndarray = None
    num_rows: int = 0
    row_width: int = 0
    counters: dict = None
    _read: Optional[Callable[[int], np.ndarray]] = None

    def tableau_row(self, i: int) -> np.ndarray:
        """IterationView::row(i) (solver.hpp:29); needs SolverConfig.observer_rows."""
        if self._read is None:
            raise Error("IterationView.tableau_row: enable SolverConfig.observer_rows")
        return self._read(i)


@dataclass
class SolveReport:
    """lps::SolveReport (solver.hpp:47-57)."""
    status: SolveStatus = SolveStatus.iteration_limit
    objective: float = 0.0
    x: np.ndarray = field(default_factory=lambda: np.zeros(0))
    iterations_phase1: int = 0
    iterations_phase2: int = 0
    total_seconds: float = 0.0
    tpi_seconds: float = 0.0
    case_used: str = "InCore"
    memory: dict = field(default_factory=dict)  # MemoryCounters counterpart (include/lpsg.h lpsg_memory)

    @property
    def iterations(self) -> int:
        return self.iterations_phase1 + self.iterations_phase2


@dataclass
class StandardFormLP:
    """lps::StandardFormLP (lp_model.hpp:49-60): Min c.x, A x = b, b >= 0, x >= 0."""
    m: int
    n_total: int
    A: np.ndarray
    b: np.ndarray
    c: np.ndarray
    col_kind: np.ndarray
    name: str = ""
    objective_sign: float = 1.0
    objective_constant: float = 0.0

    def __post_init__(self):
        self.A = np.ascontiguousarray(self.A, dtype=np.float64).reshape(self.m, self.n_total)
        self.b = np.ascontiguousarray(self.b, dtype=np.float64)
        self.c = np.ascontiguousarray(self.c, dtype=np.float64)
        self.col_kind = np.ascontiguousarray(self.col_kind, dtype=np.uint8)

    def _c(self) -> L.Problem:
        p = L.Problem()
        p.m, p.n_total = self.m, self.n_total
        p.A = self.A.ctypes.data_as(C.POINTER(C.c_double))
        p.b = self.b.ctypes.data_as(C.POINTER(C.c_double))
        p.c = self.c.ctypes.data_as(C.POINTER(C.c_double))
        p.col_kind = self.col_kind.ctypes.data_as(C.POINTER(C.c_uint8))
        return p


class SparsityClass(enum.IntEnum):
    dense = 0
    s20 = 1
    s60 = 2


class Form(enum.IntEnum):
    """Input forms of BASELINE.json's configs."""
    equality = 0      # generator verbatim: artificial start basis
    le_max = 1        # rows <=, maximize: slack start basis (config C1)
    degenerate = 2    # C4 recipe: half the rows a_i - a_{i+1} with b_i = 0


@dataclass
class GenSpec:
    """lps::GenSpec (generator.hpp:14-19) plus the input form."""
    rows: int
    cols: int
    sparsity: SparsityClass = SparsityClass.dense
    seed: int = 0
    form: Form = Form.equality


class PinnedBuffer:
    """Page-locked host memory from the library (lpsg_host_alloc), exposed as numpy."""

    def __init__(self, nbytes: int):
        self.lib = L.load()
        self.ptr = C.c_void_p()
        _check(self.lib.lpsg_host_alloc(max(int(nbytes), 16), C.byref(self.ptr)))
        self.nbytes = int(nbytes)

    def array(self, shape, dtype) -> np.ndarray:
        dtype = np.dtype(dtype)
        n = int(np.prod(shape))
        buf = (C.c_byte * (n * dtype.itemsize)).from_address(self.ptr.value)
        a = np.frombuffer(buf, dtype=dtype, count=n).reshape(shape)
        a.flags.writeable = True
        return a

    def __del__(self):
        try:
            if self.ptr:
                self.lib.lpsg_host_free(self.ptr)
                self.ptr = C.c_void_p()
        except Exception:
            pass


def generate(spec: GenSpec, pinned: bool = False) -> StandardFormLP:
    """lps::generate (generator.cpp:35-72) + canonicalize, straight to standard form.
    With pinned=True, A lives in page-locked memory (fast upload in lpsg_create)."""
    lib = L.load()
    n = lib.lpsg_generated_n_total(spec.rows, spec.cols, int(spec.form))
    if spec.rows <= 0 or spec.cols <= 0:
        raise DegenerateSpec("generate: rows and cols must be positive")
    keep = None
    if pinned:
        keep = PinnedBuffer(8 * spec.rows * n)
        A = keep.array((spec.rows, n), np.float64)
    else:
        A = np.empty((spec.rows, n))
    b = np.empty(spec.rows); c = np.empty(n)
    ck = np.empty(n, np.uint8)
    _check(lib.lpsg_generate(spec.rows, spec.cols, int(spec.sparsity), spec.seed, int(spec.form),
                             A.ctypes.data_as(C.POINTER(C.c_double)),
                             b.ctypes.data_as(C.POINTER(C.c_double)),
                             c.ctypes.data_as(C.POINTER(C.c_double)),
                             ck.ctypes.data_as(C.POINTER(C.c_uint8))))
    lp = StandardFormLP(spec.rows, n, A, b, c, ck,
                        name=f"{spec.rows}_{spec.cols}_{spec.form.name}_s{spec.seed}",
                        objective_sign=1.0 if spec.form == Form.equality else -1.0)
    lp._pinned = keep  # keeps the page-locked buffer alive with the LP
    return lp


class SimplexSolver:
    """lps::SimplexSolver (solver.hpp:79-168) on one B200."""

    def __init__(self, lp: StandardFormLP, cfg: Optional[SolverConfig] = None):
        self.lib = L.load()
        self.cfg = cfg or SolverConfig()
        self.lp = lp
        self._h = C.c_void_p()
        self._prob = lp._c()
        _check(self.lib.lpsg_create(C.byref(self._prob), C.byref(self.cfg._c()),
                                    C.byref(self._h)))
        self._cb = None
        if self.cfg.observer is not None:
            obs = self.cfg.observer
            rows = bool(self.cfg.observer_rows)
            width = lp.m + 2

            def _read(h, i):
                out = np.zeros(width)
                _check(self.lib.lpsg_read_row(h, i, out.ctypes.data_as(C.POINTER(C.c_double))))
                return out

            def _tramp(p, _user):
                v = p.contents
                basic = np.ctypeslib.as_array(v.basic, (v.num_rows,)).copy()
                mem = v.counters.contents
                obs(IterationView(v.phase, v.iteration, v.objective, v.row, v.leaving, v.entering,
                                  basic, v.num_rows, v.row_width, _mem_dict(mem),
                                  (lambda i, h=v.solver: _read(h, i)) if rows else None))

            self._cb = L.VIEW_OBSERVER(_tramp)
            _check(self.lib.lpsg_set_view_observer(self._h, self._cb, None, int(rows)))

    def close(self) -> None:
        if self._h:
            self.lib.lpsg_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # ---- driver
    def keep_trace(self, keep: bool = True) -> None:
        _check(self.lib.lpsg_keep_trace(self._h, int(keep)))

    def trace(self) -> np.ndarray:
        n = C.c_long()
        _check(self.lib.lpsg_get_trace(self._h, None, 0, C.byref(n)))
        out = np.zeros(n.value, TRACE_DTYPE)
        _check(self.lib.lpsg_get_trace(self._h, out.ctypes.data_as(C.POINTER(L.Trace)), n.value,
                                       C.byref(n)))
        return out

    def solve(self) -> SolveReport:
        rep = L.Report()
        _check(self.lib.lpsg_solve(self._h, C.byref(rep)))
        x = np.zeros(self.lp.n_total)
        _check(self.lib.lpsg_get_x(self._h, x.ctypes.data_as(C.POINTER(C.c_double)),
                                   self.lp.n_total))
        return SolveReport(SolveStatus(rep.status), rep.objective, x, rep.iterations_phase1,
                           rep.iterations_phase2, rep.total_seconds, rep.tpi_seconds,
                           "Tiled" if rep.case_used == 1 else "InCore", memory=self.memory())

    def reinvert_stats(self) -> dict:
        """Reinversion mode: rebuilds, Newton steps, max|I - B X| before / after
        the last rebuild, device seconds (include/lpsg.h lpsg_reinvert_stats)."""
        n, k = C.c_long(), C.c_long()
        r0, r1, t = C.c_double(), C.c_double(), C.c_double()
        _check(self.lib.lpsg_reinvert_stats(self._h, C.byref(n), C.byref(k), C.byref(r0),
                                            C.byref(r1), C.byref(t)))
        return dict(rebuilds=n.value, steps=k.value, residual_before=r0.value,
                    residual_after=r1.value, seconds=t.value)

    def lookahead_stats(self) -> dict:
        """select_leaving's lookaheads settled by the bounded selection vs scored
        in full; lookahead pricings settled by the DFMA screen vs the exact GEMM
        (include/lpsg.h lpsg_lookahead_stats)."""
        v = [C.c_longlong() for _ in range(5)]
        _check(self.lib.lpsg_lookahead_stats(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("bounded", "full", "price_bounded", "price_exact", "probe_rounds"),
                        (x.value for x in v)))

    def memory(self) -> dict:
        """SolveReport::memory counterpart (include/lpsg.h lpsg_memory)."""
        m = L.Memory()
        _check(self.lib.lpsg_get_memory(self._h, C.byref(m)))
        return _mem_dict(m)

    # ---- measurement (extensions; include/lpsg.h "measurement")
    def set_max_iter(self, max_iter: int) -> None:
        _check(self.lib.lpsg_set_max_iter(self._h, int(max_iter)))

    def profile(self, enable: bool = True) -> None:
        _check(self.lib.lpsg_profile(self._h, int(enable)))

    def profile_stats(self) -> dict:
        n = C.c_int()
        buf = (L.KernelStat * 16)()
        _check(self.lib.lpsg_profile_get(self._h, buf, 16, C.byref(n)))
        return {buf[k].name.decode(): dict(launches=buf[k].launches, ms=buf[k].milliseconds,
                                           bytes=buf[k].algorithmic_bytes)
                for k in range(min(n.value, 16))}

    def device_ms(self) -> float:
        v = C.c_double()
        _check(self.lib.lpsg_last_solve_device_ms(self._h, C.byref(v)))
        return v.value

    def comm_stats(self) -> dict:
        n, b = C.c_longlong(), C.c_double()
        _check(self.lib.lpsg_comm_stats(self._h, C.byref(n), C.byref(b)))
        return dict(calls=n.value, bytes=b.value)

    def shard_info(self) -> dict:
        v = [C.c_int() for _ in range(6)]
        _check(self.lib.lpsg_shard_info(self._h, *[C.byref(x) for x in v]))
        return dict(zip(("world", "rank", "row0", "rows", "col0", "col1"), (x.value for x in v)))

    def transport(self) -> str:
        return self.lib.lpsg_transport(self._h).decode()

    def counters(self) -> dict:
        a, b, c = C.c_long(), C.c_longlong(), C.c_longlong()
        _check(self.lib.lpsg_counters(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return dict(kernel_launches=a.value, h2d_bytes=b.value, d2h_bytes=c.value)

    # ---- step API
    @dataclass
    class Pricing:
        optimal: bool
        entering: int
        reduced_cost: float

    @dataclass
    class Ratio:
        unbounded: bool
        theta: float
        candidates: List[int]

    def price(self) -> "SimplexSolver.Pricing":
        o, e, z = C.c_int(), C.c_int(), C.c_double()
        _check(self.lib.lpsg_price(self._h, C.byref(o), C.byref(e), C.byref(z)))
        return SimplexSolver.Pricing(bool(o.value), e.value, z.value)

    def compute_direction(self, entering: int, reduced_cost: float) -> None:
        _check(self.lib.lpsg_compute_direction(self._h, entering, reduced_cost))

    def ratio_test(self) -> "SimplexSolver.Ratio":
        u, t, n = C.c_int(), C.c_double(), C.c_int()
        buf = (C.c_int * max(self.m(), 1))()
        _check(self.lib.lpsg_ratio_test(self._h, C.byref(u), C.byref(t), buf, self.m(),
                                        C.byref(n)))
        return SimplexSolver.Ratio(bool(u.value), t.value, list(buf[: n.value]))

    def select_leaving(self, candidates: List[int], entering: int) -> int:
        arr = (C.c_int * len(candidates))(*candidates)
        r = C.c_int()
        _check(self.lib.lpsg_select_leaving(self._h, arr, len(candidates), entering, C.byref(r)))
        return r.value

    def lookahead_scores(self, rows: List[int], entering: int) -> np.ndarray:
        arr = (C.c_int * max(len(rows), 1))(*rows)
        out = np.zeros(len(rows))
        _check(self.lib.lpsg_lookahead_scores(self._h, arr, len(rows), entering,
                                              out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def pivot_update(self, leaving_row: int, entering: int) -> None:
        _check(self.lib.lpsg_pivot_update(self._h, leaving_row, entering))

    # ---- Figure-1 tableau accessors (solver.hpp:139-151)
    def m(self) -> int:
        return self.lp.m

    def row(self, i: int) -> np.ndarray:
        out = np.zeros(self.lp.m + 2)
        _check(self.lib.lpsg_read_row(self._h, i, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def objective_value(self) -> float:
        return float(self.row(0)[self.lp.m])

    def basis(self) -> np.ndarray:
        out = np.zeros(self.lp.m, np.int32)
        _check(self.lib.lpsg_basis(self._h, out.ctypes.data_as(C.POINTER(C.c_int)), self.lp.m))
        return out

    def phase(self) -> int:
        return self.lib.lpsg_phase(self._h)


def _mem_dict(m) -> dict:
    return {k: int(getattr(m, k)) for k, _ in L.Memory._fields_}


def two_phase_solve(lp: StandardFormLP, cfg: Optional[SolverConfig] = None) -> SolveReport:
    """lps::two_phase_solve (solver.hpp:173)."""
    with SimplexSolver(lp, cfg) as s:
        return s.solve()


def device_count() -> int:
    return L.load().lpsg_device_count()


def fp64_peak(device: int = 0) -> float:
    """Measured fp64 SIMT throughput (TFLOP/s, DMUL/DADD without FMA), the
    roofline denominator of the batched lookahead (include/lpsg.h)."""
    v = C.c_double()
    _check(L.load().lpsg_fp64_peak(int(device), C.byref(v)))
    return v.value


def shard_range(n: int, world: int, rank: int):
    """[lo, hi) of n items owned by shard `rank` of `world` (rows of B^-1 or
    pricing columns; include/lpsg.h lpsg_shard_range)."""
    lo, hi = C.c_int(), C.c_int()
    _check(L.load().lpsg_shard_range(int(n), int(world), int(rank), C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId for SolverConfig.nccl_id (call on rank 0, share with the others)."""
    buf = (C.c_ubyte * 128)()
    _check(L.load().lpsg_nccl_unique_id(buf))
    return bytes(buf)


class PeerHeap:
    """Symmetric device heap of the P2P transport (include/lpsg.h lpsg_peer_*).

    Every rank: ``h = PeerHeap(rank, world, device)``; all-gather ``h.handle``
    (64 bytes) in rank order; ``h.connect(handles)``; pass ``SolverConfig(peer=h)``.
    Keep it alive until the solver is closed."""

    def __init__(self, rank: int, world: int, device: int = 0, heap_bytes: int = 0):
        self.lib = L.load()
        self.ptr = C.c_void_p()
        buf = (C.c_ubyte * 64)()
        _check(self.lib.lpsg_peer_create(int(rank), int(world), int(device), int(heap_bytes),
                                         C.byref(self.ptr), buf))
        self.handle = bytes(buf)

    def connect(self, handles) -> None:
        blob = b"".join(handles)
        arr = (C.c_ubyte * len(blob)).from_buffer_copy(blob)
        _check(self.lib.lpsg_peer_connect(self.ptr, arr))

    def close(self) -> None:
        if self.ptr:
            self.lib.lpsg_peer_destroy(self.ptr)
            self.ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def solve_sharded(lp: StandardFormLP, cfg: Optional[SolverConfig] = None, shards: int = 2,
                  spread_devices: bool = False, trace: bool = False, p2p: bool = False):
    """The sharded solver in one process: `shards` host threads with in-process
    device-to-device exchanges (all on cfg.device, or spread over the visible
    GPUs). Returns (SolveReport, trace or None) of shard 0."""
    cfg = cfg or SolverConfig()
    lib = L.load()
    rep = L.Report()
    x = np.zeros(lp.n_total)
    cap = 50 * (lp.m + 2 * lp.n_total) + 16 if trace else 0
    tr = np.zeros(cap, TRACE_DTYPE)
    n = C.c_long()
    prob = lp._c()
    flags = (1 if spread_devices else 0) | (2 if p2p else 0)
    _check(lib.lpsg_solve_sharded(C.byref(prob), C.byref(cfg._c()), int(shards), flags,
                                  C.byref(rep), x.ctypes.data_as(C.POINTER(C.c_double)),
                                  tr.ctypes.data_as(C.POINTER(L.Trace)) if trace else None, cap,
                                  C.byref(n)))
    out = SolveReport(SolveStatus(rep.status), rep.objective, x, rep.iterations_phase1,
                      rep.iterations_phase2, rep.total_seconds, rep.tpi_seconds)
    return out, (tr[: min(n.value, cap)].copy() if trace else None)
