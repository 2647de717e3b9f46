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


def test_launcher_spawns_ranks():
    """bench.py --gpus N's launcher: one process in, N gloo ranks out (127.0.0.1)."""
    import json
    import subprocess
    import sys
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "launch_worker.py")
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, worker, "--gpus", "2"], capture_output=True, text=True, timeout=300,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1  # rank 0 only
    d = json.loads(lines[0])
    assert d["world"] == 2 and d["ranks"] == [0, 1] and d["env_addr"] == "127.0.0.1"
    assert d["spans"] == [[0, 32768], [32768, 65536]]


def test_launcher_noop_under_launcher_or_one_rank(monkeypatch):
    from paper_2104_12570_b200 import launch
    assert launch.relaunch_if_needed(1, "x.py", []) is None
    monkeypatch.setenv("WORLD_SIZE", "2")
    assert launch.relaunch_if_needed(2, "x.py", []) is None
    argv = launch.torchrun_argv(4, "bench.py", ["--gpus", "4"], port=29555)
    assert argv[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node" in argv and argv[argv.index("--nproc-per-node") + 1] == "4"
    assert argv[argv.index("--master-addr") + 1] == "127.0.0.1"


def test_partition_systems_cover_balanced():
    from paper_2104_12570_b200.sharded import partition_systems
    for nsys in (1, 7, 8, 65536, 65537, 100003):
        for world in (1, 2, 3, 4, 8):
            spans = [partition_systems(nsys, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nsys
            assert all(spans[r][1] == spans[r + 1][0] for r in range(world - 1))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1


def test_mailbox_epochs_restart_before_wrap():
    """Epoch tags are 31-bit: the count restarts (mailboxes zeroed, collectively)
    before a reservation would cross the limit, never wrapping into old tags."""
    from paper_2104_12570_b200.sharded import Mailboxes
    mb = object.__new__(Mailboxes)
    resets = []
    mb.epoch = 0
    mb.reset = lambda: (resets.append(mb.epoch), setattr(mb, "epoch", 0))
    b0 = mb.next_epochs(1000)
    b1 = mb.next_epochs(1000)
    assert b0 == 0 and b1 == 1002 and not resets
    mb.epoch = Mailboxes.EPOCH_LIMIT - 500
    b2 = mb.next_epochs(1000)
    assert resets == [Mailboxes.EPOCH_LIMIT - 500] and b2 == 0 and mb.epoch == 1002
    with pytest.raises(ValueError):
        mb.next_epochs(Mailboxes.EPOCH_LIMIT)
