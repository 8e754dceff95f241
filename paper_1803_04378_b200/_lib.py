"""ctypes binding of the lpsg C ABI (include/lpsg.h).

The library is built in-tree by paper_1803_04378_b200/build.py. There is no
fallback: if the shared library is missing or cannot be loaded, every entry
point raises.
"""
from __future__ import annotations

import ctypes as C
import os

from . import build as _build

LIB_PATH = _build.LIB


class Problem(C.Structure):
    _fields_ = [("m", C.c_int), ("n_total", C.c_int), ("A", C.POINTER(C.c_double)),
                ("b", C.POINTER(C.c_double)), ("c", C.POINTER(C.c_double)),
                ("col_kind", C.POINTER(C.c_uint8))]


class Config(C.Structure):
    _fields_ = [("opt_tol", C.c_double), ("pivot_tol", C.c_double), ("feas_tol", C.c_double),
                ("ratio_tie_tol", C.c_double), ("max_iter", C.c_long), ("anticycle", C.c_int),
                ("kernel", C.c_int), ("workers", C.c_int), ("device", C.c_int),
                ("batch", C.c_int), ("reserved", C.c_int * 6),
                ("world_size", C.c_int), ("rank", C.c_int), ("nccl_id", C.c_ubyte * 128),
                ("peer", C.c_void_p), ("reinvert_every", C.c_long),
                ("memory_budget", C.c_ulonglong)]


class Report(C.Structure):
    _fields_ = [("status", C.c_int), ("objective", C.c_double),
                ("iterations_phase1", C.c_long), ("iterations_phase2", C.c_long),
                ("total_seconds", C.c_double), ("tpi_seconds", C.c_double),
                ("case_used", C.c_int)]


class Trace(C.Structure):
    _fields_ = [("iteration", C.c_long), ("phase", C.c_int), ("row", C.c_int),
                ("leaving", C.c_int), ("entering", C.c_int), ("objective", C.c_double)]


class KernelStat(C.Structure):
    _fields_ = [("name", C.c_char_p), ("launches", C.c_long), ("milliseconds", C.c_double),
                ("algorithmic_bytes", C.c_double)]


OBSERVER = C.CFUNCTYPE(None, C.POINTER(Trace), C.c_void_p)


class Memory(C.Structure):
    _fields_ = [("device_read_bytes", C.c_uint64), ("device_write_bytes", C.c_uint64),
                ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("kernel_launches", C.c_uint64)]


class View(C.Structure):
    _fields_ = [("phase", C.c_int), ("iteration", C.c_long), ("objective", C.c_double),
                ("basic", C.POINTER(C.c_int)), ("num_rows", C.c_int), ("row_width", C.c_int),
                ("row", C.c_int), ("leaving", C.c_int), ("entering", C.c_int),
                ("counters", C.POINTER(Memory)), ("solver", C.c_void_p)]


VIEW_OBSERVER = C.CFUNCTYPE(None, C.POINTER(View), C.c_void_p)

# (name, restype, argtypes) for every symbol include/lpsg.h declares.
_P = C.c_void_p
_PD = C.POINTER(C.c_double)
_PI = C.POINTER(C.c_int)
SIGNATURES = [
    ("lpsg_last_error", C.c_char_p, []),
    ("lpsg_version", C.c_char_p, []),
    ("lpsg_device_count", C.c_int, []),
    ("lpsg_config_default", None, [C.POINTER(Config)]),
    ("lpsg_create", C.c_int, [C.POINTER(Problem), C.POINTER(Config), C.POINTER(_P)]),
    ("lpsg_solve", C.c_int, [_P, C.POINTER(Report)]),
    ("lpsg_get_x", C.c_int, [_P, _PD, C.c_int]),
    ("lpsg_destroy", None, [_P]),
    ("lpsg_two_phase_solve", C.c_int, [C.POINTER(Problem), C.POINTER(Config),
                                       C.POINTER(Report), _PD]),
    ("lpsg_set_observer", C.c_int, [_P, OBSERVER, _P]),
    ("lpsg_keep_trace", C.c_int, [_P, C.c_int]),
    ("lpsg_set_view_observer", C.c_int, [_P, VIEW_OBSERVER, _P, C.c_int]),
    ("lpsg_get_memory", C.c_int, [_P, C.POINTER(Memory)]),
    ("lpsg_reinvert_stats", C.c_int, [_P, C.POINTER(C.c_long), C.POINTER(C.c_long), _PD, _PD, _PD]),
    ("lpsg_lookahead_stats", C.c_int, [_P] + [C.POINTER(C.c_longlong)] * 5),
    ("lpsg_get_trace", C.c_int, [_P, C.POINTER(Trace), C.c_long, C.POINTER(C.c_long)]),
    ("lpsg_price", C.c_int, [_P, _PI, _PI, _PD]),
    ("lpsg_compute_direction", C.c_int, [_P, C.c_int, C.c_double]),
    ("lpsg_ratio_test", C.c_int, [_P, _PI, _PD, _PI, C.c_int, _PI]),
    ("lpsg_select_leaving", C.c_int, [_P, _PI, C.c_int, C.c_int, _PI]),
    ("lpsg_lookahead_scores", C.c_int, [_P, _PI, C.c_int, C.c_int, _PD]),
    ("lpsg_pivot_update", C.c_int, [_P, C.c_int, C.c_int]),
    ("lpsg_dims", C.c_int, [_P, _PI, _PI, _PI]),
    ("lpsg_read_row", C.c_int, [_P, C.c_int, _PD]),
    ("lpsg_basis", C.c_int, [_P, _PI, C.c_int]),
    ("lpsg_phase", C.c_int, [_P]),
    ("lpsg_set_max_iter", C.c_int, [_P, C.c_long]),
    ("lpsg_profile", C.c_int, [_P, C.c_int]),
    ("lpsg_profile_get", C.c_int, [_P, C.POINTER(KernelStat), C.c_int, _PI]),
    ("lpsg_last_solve_device_ms", C.c_int, [_P, _PD]),
    ("lpsg_counters", C.c_int, [_P, C.POINTER(C.c_long), C.POINTER(C.c_longlong),
                                C.POINTER(C.c_longlong)]),
    ("lpsg_host_alloc", C.c_int, [C.c_size_t, C.POINTER(C.c_void_p)]),
    ("lpsg_fp64_peak", C.c_int, [C.c_int, _PD]),
    ("lpsg_nccl_unique_id", C.c_int, [C.POINTER(C.c_ubyte)]),
    ("lpsg_solve_sharded", C.c_int, [C.POINTER(Problem), C.POINTER(Config), C.c_int, C.c_int,
                                     C.POINTER(Report), _PD, C.POINTER(Trace), C.c_long,
                                     C.POINTER(C.c_long)]),
    ("lpsg_shard_range", C.c_int, [C.c_int, C.c_int, C.c_int, _PI, _PI]),
    ("lpsg_peer_create", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_size_t, C.POINTER(_P),
                                   C.POINTER(C.c_ubyte)]),
    ("lpsg_peer_connect", C.c_int, [_P, C.POINTER(C.c_ubyte)]),
    ("lpsg_peer_destroy", None, [_P]),
    ("lpsg_transport", C.c_char_p, [_P]),
    ("lpsg_comm_stats", C.c_int, [_P, C.POINTER(C.c_longlong), _PD]),
    ("lpsg_shard_info", C.c_int, [_P, _PI, _PI, _PI, _PI, _PI, _PI]),
    ("lpsg_host_free", None, [C.c_void_p]),
    ("lpsg_generated_n_total", C.c_int, [C.c_int, C.c_int, C.c_int]),
    ("lpsg_generate", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_int, _PD, _PD, _PD,
                                C.POINTER(C.c_uint8)]),
]

_lib = None


def load(build_if_missing: bool = True) -> C.CDLL:
    """Loads the in-tree liblpsg.so (building it first when it is missing).
    LPSG_EXPERIMENTS_LIB=1 loads the performance-experiment build instead
    (tools/dbg only: its knobs produce invalid solves)."""
    global _lib
    if _lib is not None:
        return _lib
    xp = os.environ.get("LPSG_EXPERIMENTS_LIB") == "1"
    path = _build.LIB_XP if xp else LIB_PATH
    if not os.path.exists(path):
        if not build_if_missing:
            raise OSError(f"lpsg library not built: {path}")
        _build.build(experiments=xp)
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib
