"""Host side of the multi-GPU paths on CPU: torch.distributed (gloo,
world_size 2) all-gather in rank order, row partitioning, and the per-rank
system shards of the batched path.  No kernels run here."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2104_12570_b200.sharded import DistComm, LocalComm, partition_rows, rank_order_sum


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.distributed.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = DistComm()
        local = torch.full((3,), float(rank + 1), dtype=torch.float64) * torch.tensor([1.0, 10.0, 100.0],
                                                                                        dtype=torch.float64)
        got = comm.all_gather([local])
        s = rank_order_sum(got)
        r0, r1 = partition_rows(1001, world, rank, align=4)
        q.put((rank, [g.tolist() for g in got], s.tolist(), (r0, r1)))
    finally:
        torch.distributed.destroy_process_group()


def test_distcomm_allgather_rank_order_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, gathered, s, rows in out:
        assert gathered == [[1.0, 10.0, 100.0], [2.0, 20.0, 200.0]]
        assert s == [3.0, 30.0, 300.0]  # identical on both ranks
    assert out[0][3] == (0, 504) and out[1][3] == (504, 1001)


def test_partition_rows_cover_and_align():
    for obs in (1, 7, 1000, 1 << 20, 12345):
        for world in (1, 2, 3, 4, 8):
            blocks = [partition_rows(obs, world, r, align=4) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == obs
            for (a0, a1), (b0, b1) in zip(blocks, blocks[1:]):
                assert a1 == b0
            assert all(b[0] % 4 == 0 or b[0] == obs for b in blocks)


def test_localcomm_and_rank_order_sum_fixed_order():
    comm = LocalComm(3)
    parts = [torch.tensor([1e16, 1.0]), torch.tensor([1.0, 1e16]), torch.tensor([-1e16, -1e16])]
    got = comm.all_gather(parts)
    s = rank_order_sum(got)
    # ((1e16 + 1) + -1e16) = 0 in fp64 rank order; a different order would give 1
    assert s.tolist() == [0.0, 0.0]
