"""One process per GPU: re-launch a script under ``torch.distributed.run``.

``bench.py --gpus N`` (and any script that wants the same behaviour) calls
:func:`relaunch_if_needed` first: when N > 1 and the process is not already a
rank (no ``WORLD_SIZE`` in the environment) it starts
``python -m torch.distributed.run --nnodes 1 --nproc-per-node N
--master-addr 127.0.0.1 --master-port <free port> <script> <args>``, waits,
and returns the launcher's exit code; the ranks' stdout goes to the given file
descriptor (rank 0 prints the one JSON line).  Under torchrun, or with N = 1,
it returns None and the caller runs in-process.

Rendezvous is always on 127.0.0.1 (the container hostname may not resolve).
"""

from __future__ import annotations

import os
import socket
import subprocess
import sys


def free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def torchrun_argv(nproc: int, script: str, args, port: int | None = None) -> list:
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(int(nproc)),
            "--master-addr", "127.0.0.1", "--master-port", str(port or free_port()), script, *list(args)]


def relaunch_if_needed(nproc: int, script: str, args, stdout=None, env=None, timeout=None):
    """Run ``script args`` as ``nproc`` ranks unless this process already is one.

    Returns the launcher's exit code, or None when the caller should run the
    work itself (nproc <= 1, or WORLD_SIZE already set by a launcher)."""
    if nproc <= 1 or "WORLD_SIZE" in os.environ:
        return None
    e = dict(os.environ if env is None else env)
    e.setdefault("OMP_NUM_THREADS", "1")
    if os.environ.get("BAK_NCCL_DEBUG", "1") == "1":
        e.setdefault("NCCL_DEBUG", "INFO")  # rank / transport lines on stderr
    proc = subprocess.run(torchrun_argv(nproc, script, args), stdout=stdout, env=e, timeout=timeout)
    return proc.returncode
