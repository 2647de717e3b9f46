"""Worker for tests/test_ipc_mailbox_gpu.py: two processes on ONE GPU (gloo
for the handle exchange) check that each rank's exported mailbox is mapped
at the right address by its peer — rank r writes a pattern through the peer
pointer, the owner reads it back.  No kernel waits on another process.
Not collected by pytest."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_12570_b200 import _lib  # noqa: E402
from paper_2104_12570_b200.sharded import Mailboxes  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
torch.cuda.set_device(dev)
dist.init_process_group("gloo")


class CpuGatherComm:
    """all_gather through gloo on host copies (two ranks share one GPU)."""

    def __init__(self):
        self.rank, self.world = rank, world

    def all_gather(self, per_rank):
        t = per_rank[0]
        outs = [torch.empty_like(t, device="cpu") for _ in range(self.world)]
        dist.all_gather(outs, t.cpu())
        return [o.to(t.device) for o in outs]


def wrap(ptr, nbytes):
    class _A:
        __cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_A(), device=dev)


mb = Mailboxes(world, CpuGatherComm(), dev)
nbytes = int(_lib.load().bak_mailbox_bytes(world))
peer = (rank + 1) % world
pattern = (torch.arange(nbytes, dtype=torch.int64, device=dev) * 7 + 13 * (rank + 1)).remainder(251).to(torch.uint8)
wrap(mb.ptrs[peer], nbytes).copy_(pattern)
torch.cuda.synchronize()
dist.barrier()
mine = wrap(mb.ptrs[rank], nbytes).clone()
writer = (rank - 1) % world
want = (torch.arange(nbytes, dtype=torch.int64, device=dev) * 7 + 13 * (writer + 1)).remainder(251).to(torch.uint8)
ok = bool(torch.equal(mine, want))
dist.barrier()
mb.close()
dist.destroy_process_group()
print(f"IPC rank={rank} ok={ok}", flush=True)
sys.exit(0 if ok else 1)
