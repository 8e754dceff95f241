"""The P2P transport across PROCESSES: two ranks (torch.multiprocessing, gloo
bootstrap for the 64-byte CUDA IPC handles) map each other's symmetric heaps
with cudaIpcOpenMemHandle and solve through device-initiated peer stores and
flags, exactly as `torchrun bench.py --gpus N --transport p2p` does on N GPUs.
Here both ranks share one B200 (separate CUDA contexts, time-sliced), so only
small fixtures are used. Bar: the golden trace, bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import ROOT, Golden

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, out):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world))
    import torch.distributed as dist
    import paper_1803_04378_b200 as P
    from conftest import Golden as G
    dist.init_process_group("gloo")
    g = G(name)
    rows, cols, form, seed, sp = g.spec
    lp = P.generate(P.GenSpec(rows, cols, P.SparsityClass(sp), seed, P.Form(form)))
    heap = P.PeerHeap(rank, world, device=0)
    handles = [None] * world
    dist.all_gather_object(handles, heap.handle)
    heap.connect(handles)
    dist.barrier()
    with P.SimplexSolver(lp, P.SolverConfig(max_iter=g.max_iter, peer=heap)) as s:
        s.keep_trace(True)
        rep = s.solve()
        tr = s.trace()
        transport = s.transport()
    dist.barrier()
    heap.close()
    dist.destroy_process_group()
    out[rank] = (int(rep.status), rep.objective, tr.tobytes(), rep.x.tobytes(), transport)


@pytest.mark.parametrize("name", ["gen_64x128_f0_s2", "gen_20x40_f2_s1"])
def test_p2p_two_processes(name):
    g = Golden(name)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(2, _free_port(), name, out), nprocs=2, join=True)
    import paper_1803_04378_b200 as P
    ref = g.trace[: g.trace_len]
    for r in range(2):
        status, obj, trb, xb, transport = out[r]
        assert transport == "p2p"
        tr = np.frombuffer(trb, P.TRACE_DTYPE)
        assert status == g.status
        assert len(tr) == len(ref)
        for f in ("row", "leaving", "entering"):
            assert np.array_equal(tr[f], ref[f]), (r, f)
        assert np.array_equal(tr["objective"].view(np.uint64), ref["objective"].view(np.uint64))
        assert np.array_equal(np.frombuffer(xb, np.float64).view(np.uint64), g.x.view(np.uint64))


@pytest.mark.parametrize("name", ["gen_256x512_f2_s1", "gen_1000x2000_f0_s1_max_iter400"])
def test_p2p_two_processes_larger(name):
    """Tie-heavy (batched lookahead exchanged over P2P) and m = 1000 prefixes."""
    test_p2p_two_processes(name)


def test_bench_two_ranks_fills_the_exchange_report():
    """`torchrun --nproc-per-node 2 bench.py --gpus 2` end to end (both ranks on
    this one B200, LPSG_BENCH_SAME_DEVICE: time-sliced, so a smoke test of the
    multi-rank bench path, not a number): the line reports n_gpus 2 and the
    per-pivot exchange accounting (collectives, payload, device time)."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, LPSG_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", "c2", "--steps", "10",
           "--warmup", "3", "--e2e-max-iter", "30", "--no-reinversion"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    line = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["steps"] == 10
    ex = line["exchange"]
    assert ex["collectives_per_pivot"] > 0 and ex["payload_bytes_per_pivot_per_rank"] > 0
    assert ex["us_per_pivot_incl_merge_kernels"] is not None
