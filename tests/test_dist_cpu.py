"""Multi-process (world_size 2, gloo, CPU) tests of the N>1 host path.

The sharded data path itself runs on GPUs (tests/test_gpu_sharded.py runs it as
G shards on one B200; NCCL carries it across GPUs). What runs on the host and is
covered here: the shard partition every rank derives independently, the NCCL
unique-id hand-off and the max-over-ranks timing of bench.py's torchrun path.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

from conftest import ROOT


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    import paper_1803_04378_b200 as P
    w, r, local = bench.dist_ctx()
    nid = bench.share_nccl_id(w, r)
    mx = bench.max_over_ranks(10.0 + r, w)
    rows = P.shard_range(8000, w, r)
    cols = P.shard_range(16000, w, r)
    bench.barrier(w)
    import torch.distributed as dist
    dist.destroy_process_group()
    out[r] = (nid, mx, rows, cols, local)


def test_torchrun_control_plane_world2():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    ids = {out[r][0] for r in range(world)}
    assert len(ids) == 1 and len(next(iter(ids))) == 128  # one NCCL id, seen by both ranks
    assert all(out[r][1] == 11.0 for r in range(world))  # max over ranks
    assert [out[r][2] for r in range(world)] == [(0, 4000), (4000, 8000)]
    assert [out[r][3] for r in range(world)] == [(0, 8000), (8000, 16000)]


@pytest.mark.parametrize("n,world", [(8000, 8), (24000, 8), (7, 3), (1, 1), (257, 2), (5, 5)])
def test_shard_ranges_partition(n, world):
    import paper_1803_04378_b200 as P
    rs = [P.shard_range(n, world, r) for r in range(world)]
    assert rs[0][0] == 0 and rs[-1][1] == n
    assert all(rs[k][1] == rs[k + 1][0] for k in range(world - 1))
    sizes = [hi - lo for lo, hi in rs]
    assert max(sizes) - min(sizes) <= 1


def test_shard_range_rejects_bad_rank():
    import paper_1803_04378_b200 as P
    with pytest.raises(P.Error):
        P.shard_range(10, 2, 2)


class _FakeHeap:
    """PeerHeap stand-in: rank `bad` fails to create its heap (e.g. no CUDA IPC)."""
    bad = 1

    def __init__(self, rank, world, device=0):
        if rank == _FakeHeap.bad:
            raise RuntimeError("cudaMalloc(peer heap): out of memory")
        self.handle = bytes([rank]) * (64 * world)

    def connect(self, handles):
        pass


def _peer_worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import bench
    import paper_1803_04378_b200 as P
    P.PeerHeap = _FakeHeap
    w, r, local = bench.dist_ctx()
    try:
        bench.peer_heap(w, r, local)
        out[r] = "connected"
    except RuntimeError as e:
        out[r] = str(e)
    # both ranks must still be in step: a collective after the failure completes
    out[f"nid{r}"] = bench.share_nccl_id(w, r)
    import torch.distributed as dist
    dist.destroy_process_group()


def test_p2p_setup_failure_is_agreed_by_all_ranks():
    """bench.py's P2P heap setup: a failure on ONE rank raises on EVERY rank
    (so all fall back to NCCL together instead of deadlocking in mismatched
    collectives)."""
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_peer_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    for r in range(world):
        assert out[r].startswith("P2P heap unavailable: rank 1: cudaMalloc"), out[r]
    assert out["nid0"] == out["nid1"]
