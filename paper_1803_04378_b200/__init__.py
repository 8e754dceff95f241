"""paper_1803_04378_b200 — B200-native dense revised simplex (lpsg).

A drop-in for the iteration loop of the reference's C++ solver
(/root/reference/proj/src/solver.cpp): the host API mirrors lps::two_phase_solve /
lps::SimplexSolver, and all per-pivot work runs in hand-written sm_100a CUDA
kernels behind the C ABI in include/lpsg.h.
"""
from .solver import (  # noqa: F401
    Anticycle, BudgetTooSmall, ColKind, CudaError, DegenerateSpec, Error, Form, GenSpec, IterationView,
    PeerHeap, PivotTooSmall, SimplexSolver, SolveReport, SolverConfig, SolveStatus, SparsityClass,
    StandardFormLP, TRACE_DTYPE, device_count, fp64_peak, generate, nccl_unique_id, shard_range, solve_sharded,
    two_phase_solve)
from .lp_model import (  # noqa: F401
    CanonicalMap, EmptyProblem, GeneralLP, InconsistentBounds, LengthMismatch, RowKind, Sense,
    canonicalize, recover_solution)
from .mps import (  # noqa: F401
    DuplicateRow, MalformedNumber, MissingObjectiveRow, MpsDocument, UndeclaredRow,
    UnknownSection, UnsupportedBoundKind, load_mps, parse_mps, parse_mps_file, solve_mps,
    to_general_lp, to_mps_document, write_mps)

__all__ = [
    "Anticycle", "BudgetTooSmall", "ColKind", "CudaError", "DegenerateSpec", "Error", "Form", "GenSpec",
    "IterationView", "PeerHeap", "PivotTooSmall", "SimplexSolver", "SolveReport", "SolverConfig",
    "SolveStatus", "SparsityClass", "StandardFormLP", "TRACE_DTYPE", "device_count",
    "fp64_peak", "generate", "nccl_unique_id", "shard_range", "solve_sharded", "two_phase_solve",
    # LP ingestion (lp_model.py, mps.py)
    "CanonicalMap", "EmptyProblem", "GeneralLP", "InconsistentBounds", "LengthMismatch",
    "RowKind", "Sense", "canonicalize", "recover_solution", "DuplicateRow", "MalformedNumber",
    "MissingObjectiveRow", "MpsDocument", "UndeclaredRow", "UnknownSection",
    "UnsupportedBoundKind", "load_mps", "parse_mps", "parse_mps_file", "solve_mps",
    "to_general_lp", "to_mps_document", "write_mps",
]
