"""The multi-process NCCL path (DistComm, one rank per GPU, launched by
torch.distributed.run with 127.0.0.1 rendezvous) end to end with as many
ranks as the box has GPUs (1 here): row-sharded GRAM and the exact
row-sharded kernel with its peer mailboxes match the oracle."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu


def test_nccl_rowsharded_solves_match_oracle():
    import torch
    n = max(1, min(torch.cuda.device_count(), 8))
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", "29533", os.path.join(here, "dist_worker.py")]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("RESULT ")][-1]
    res = json.loads(line[len("RESULT "):])
    assert res["gram"]["sweeps"] == 5 and res["gram"]["err"] <= 1e-10
    assert res["stream"]["sweeps"] == 5 and res["stream"]["err"] <= 1e-10
    assert res["stream"]["label"] == "stream-rowshard"
