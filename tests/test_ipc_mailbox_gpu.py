"""The row-sharded exact kernel's cross-rank mailboxes: each rank exports its
mailbox over CUDA IPC and maps its peers'.  Two processes on one GPU check the
mapping addresses (a pattern written through the peer pointer lands in the
owner's mailbox); the in-kernel exchange itself needs one GPU per rank."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_ipc_mailboxes_map_the_exported_allocation():
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", "29541", os.path.join(here, "ipc_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])
    assert out.stdout.count("ok=True") == 2, out.stdout
