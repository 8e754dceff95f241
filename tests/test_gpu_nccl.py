"""The NCCL transport of the sharded solver, exercised on one B200.

NCCL refuses two ranks on one GPU, so this runs the full sharded code path
(pivot-row int64 allreduce, (z, j) and ratio-message all-gathers, ordered
rebuild chain, drive-out broadcast / min-reduce, sharded lookahead exchanges)
through a REAL one-rank NCCL communicator (SolverConfig.nccl_single), and
checks it against the golden traces bit for bit. Multi-rank NCCL runs come
from `torchrun ... bench.py --gpus N` on a multi-GPU box.
"""
import numpy as np
import pytest

from conftest import Golden

pytestmark = pytest.mark.gpu


def _P():
    import paper_1803_04378_b200 as P
    return P


def _bits(a):
    return np.asarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("name", ["gen_256x512_f0_s1", "gen_256x512_f2_s1", "gen_128x256_f2_s5",
                                  "netlib_afiro", "netlib_scsd1", "netlib_sctap1", "beale_3x7",
                                  "infeasible_2x2", "unbounded_1x3"])
def test_nccl_one_rank_golden_parity(name):
    P = _P()
    g = Golden(name)
    if g.spec is not None:
        rows, cols, form, seed, sp = g.spec
        lp = P.generate(P.GenSpec(rows, cols, P.SparsityClass(sp), seed, P.Form(form)))
    else:
        A, b, c, ck = g.arrays()
        lp = P.StandardFormLP(g.m, g.n_total, A, b, c, ck)
    cfg = P.SolverConfig(max_iter=g.max_iter, pivot_tol=g.pivot_tol, kernel=g.kernel,
                         anticycle=P.Anticycle(g.anticycle), nccl_single=True,
                         nccl_id=P.nccl_unique_id())
    with P.SimplexSolver(lp, cfg) as s:
        info = s.shard_info()
        assert info["world"] == 1
        s.keep_trace(True)
        rep = s.solve()
        tr = s.trace()
        stats = s.comm_stats()
    ref = g.trace[: g.trace_len]
    assert int(rep.status) == g.status
    assert len(tr) == len(ref)
    for f in ("row", "leaving", "entering"):
        assert np.array_equal(tr[f], ref[f]), f
    assert np.array_equal(_bits(tr["objective"]), _bits(ref["objective"]))
    assert np.array_equal(_bits(rep.x), _bits(g.x))
    assert stats["calls"] >= 3 * len(tr)  # three exchanges per pivot went through NCCL
