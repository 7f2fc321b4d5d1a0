"""Multi-process (world size 2, gloo, CPU) coverage of the adapter-parallel
plumbing: LPT job partitioning, the one-off base-weight broadcast, and the
max-over-ranks timing reduction used by bench.py."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2312_02515_b200 import parallel as PL


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank 0 owns the freshly initialised base weights; the others start from garbage
        g = torch.Generator().manual_seed(1234)
        names = ["q", "k", "gate", "down"]
        shapes = {"q": (64, 64), "k": (64, 64), "gate": (172, 64), "down": (64, 172)}
        W = {}
        for n in names:
            ref = (torch.rand(*shapes[n], generator=g) * 2 - 1).to(torch.bfloat16)
            W[n] = ref.clone() if rank == 0 else torch.full(shapes[n], float(rank + 7), dtype=torch.bfloat16)
        PL.broadcast_base_weights(W, src=0)
        g = torch.Generator().manual_seed(1234)
        ok = all(torch.equal(W[n], (torch.rand(*shapes[n], generator=g) * 2 - 1).to(torch.bfloat16)) for n in names)
        # every rank computes the same partition independently
        parts = PL.partition_jobs([8192, 4096, 4096, 2048, 1024, 1024, 512, 512], world)
        gathered = [None] * world
        dist.all_gather_object(gathered, parts)
        mx = PL.max_over_ranks(10.0 * (rank + 1))
        tot = PL.sum_over_ranks(float(len(parts[rank])))
        # the native communicator's rendezvous: rank 0's NCCL id reaches every rank
        cid = PL.comm_rendezvous_id()
        ids = [None] * world
        dist.all_gather_object(ids, cid)
        out[rank] = (ok, gathered, mx, tot, parts, ids)
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_world2_broadcast_partition_and_timing():
    world = 2
    mgr = mp.get_context("spawn").Manager()  # no fork() of the multi-threaded test process
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert set(out.keys()) == {0, 1}
    for r in range(world):
        ok, gathered, mx, tot, parts, ids = out[r]
        assert len(ids[0]) == 128 and ids[0] == ids[1] and any(ids[0])  # one shared NCCL id
        assert ok, f"rank {r} did not receive rank 0's base weights"
        assert gathered[0] == gathered[1] == parts     # identical, independently computed partitions
        assert mx == 20.0                                # max over ranks
        assert tot == 8.0                                # every job owned by exactly one rank
    assert sorted(out[0][4][0] + out[0][4][1]) == list(range(8))


def test_partition_lpt_balance_and_determinism():
    tokens = [8192, 4096, 4096, 2048, 1024, 1024, 512, 512]
    p2 = PL.partition_jobs(tokens, 2)
    loads = [sum(tokens[j] for j in p) for p in p2]
    assert sorted(j for p in p2 for j in p) == list(range(8))
    assert max(loads) - min(loads) <= max(tokens)       # LPT bound
    assert PL.partition_jobs(tokens, 2) == p2
    # 32 equal jobs over 8 ranks (C5): 4 jobs each
    p8 = PL.partition_jobs([2048] * 32, 8)
    assert [len(p) for p in p8] == [4] * 8
    assert PL.partition_jobs([5], 3) == [[0], [], []]
