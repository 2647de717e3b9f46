"""(5) Multi-GPU row sharding of one very tall system (BASELINE config 3 at N > 1).

One process per GPU; rank r holds a contiguous block of rows of x, y and e
(``partition_rows``); the coefficients a and the column norms are replicated.
The per-sweep exchange is the GRAM variant's: every rank makes ONE pass over
its rows (e -= X d, sum e^2, partial g = X^T e), the ranks all-gather their
partials (a few hundred KB), and every rank runs the same forward substitution
on the same bytes summed in rank order - so d and a are bit-identical on all
ranks without a broadcast.  G = X^T X is all-gathered once.  The sweep is the
labelled GRAM reformulation (bak_gram.cu): same iterates as the reference in
exact arithmetic; parity is checked like every other variant.

``Comm`` abstracts the only collective used (all-gather, rank order):
``DistComm`` wraps torch.distributed (NCCL between GPUs, gloo on CPU) and
``LocalComm`` emulates N ranks inside one process (the shards live on one
device and the kernels of different ranks never wait on one another), which
is how the multi-rank path is tested on a single GPU.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .bak import (_host, DRIFT_TOL, DeviceMatrix, SolveConfig, SolveReport, _permutation_chunks, _ptr, _stream_ptr,
                  _to_device_vector, _torch, _Workspace, colnorms, to_device_matrix)


def partition_rows(obs, world, rank, align=2):
    """Contiguous row block [r0, r1) of `rank`; block starts are multiples of
    `align` rows (16-byte aligned columns for both precisions when align=4)."""
    per = -(-obs // world)
    per = -(-per // align) * align
    r0 = min(obs, rank * per)
    r1 = min(obs, r0 + per)
    return r0, r1


def partition_systems(nsys, world, rank):
    """Contiguous, balanced system range [s0, s1) of `rank` (sizes differ by at most one)."""
    base, extra = divmod(int(nsys), int(world))
    s0 = rank * base + min(rank, extra)
    return s0, s0 + base + (1 if rank < extra else 0)


def solve_bak_batched_sharded(xs, ys, config: SolveConfig | None = None, comm=None, *, local=False, gather=False,
                              device=None, return_device=False):
    """Many independent systems sharded over ranks with NO communication on the
    data path (north-star (5)): rank r solves the systems
    ``partition_systems(nsys, world, r)`` with ``solve_bak_batched`` (one CTA
    per system) on its own GPU — the reference's equivalent is a loop of
    ``solve_bak`` (bak.py:146) over the systems, which shards trivially.

    xs / ys: the whole batch (``local=False``: each rank takes its slice; host
    arrays are sliced without copying) or this rank's shard (``local=True``).
    Returns ``(s0, s1, BatchSolveReport)`` for the rank's systems (s0, s1 are
    None for a local shard without gather: no exchange tells the offset); with
    ``gather=True`` the per-system coefficients, sweeps and flags of ALL ranks
    are all-gathered once at the end (after the solves) and the report covers
    the whole batch (residuals stay per rank: ``residual`` is None).
    """
    from .bak import BatchSolveReport, solve_bak_batched
    world = getattr(comm, "world", 1) if comm is not None else 1
    rank = getattr(comm, "rank", 0) if comm is not None else 0
    def _n(b):
        return int(b.nsys) if hasattr(b, "nsys") else int(b.shape[0])

    if local:
        nloc = _n(xs)
        counts = [nloc]
        if comm is not None and world > 1 and gather:
            torch = _torch()
            dev = device or torch.device("cuda", torch.cuda.current_device())
            counts = [int(c.item()) for c in comm.all_gather([torch.tensor([nloc], dtype=torch.int64, device=dev)])]
        # global offsets are known only after the count exchange (gather=True)
        s0 = sum(counts[:rank]) if len(counts) == world else None
        s1 = s0 + nloc if s0 is not None else None
        xl, yl = xs, ys
    else:
        nsys = _n(xs)
        s0, s1 = partition_systems(nsys, world, rank)
        xl, yl = xs[s0:s1], ys[s0:s1]
    rep = solve_bak_batched(xl, yl, config, device=device, return_device=True)
    if not gather or comm is None or world == 1:
        if not return_device:
            rep = BatchSolveReport(_host(rep.a_hat), _host(rep.residual),
                                   None if rep.residual_norm_history is None else _host(rep.residual_norm_history),
                                   rep.sweeps_run, rep.converged, rep.wall_time, rep.drift_warning)
        return s0, s1, rep
    torch = _torch()
    dev = rep.a_hat.device
    # one collective after all the work: pad every rank's block to the largest
    sizes = ([partition_systems(_n(xs), world, r) for r in range(world)] if not local
             else [(sum(counts[:r]), sum(counts[: r + 1])) for r in range(world)])
    nmax = max(b - a for a, b in sizes)
    nv = rep.a_hat.shape[1]

    def pad(t, width):
        out = torch.zeros((nmax, width), dtype=t.dtype, device=dev)
        out[: t.shape[0]] = t.reshape(t.shape[0], width)
        return out

    flags = torch.stack([torch.as_tensor(rep.sweeps_run, dtype=torch.float64, device=dev),
                         torch.as_tensor(rep.converged, dtype=torch.float64, device=dev),
                         torch.as_tensor(rep.drift_warning, dtype=torch.float64, device=dev)], dim=1)
    ga = comm.all_gather([pad(rep.a_hat, nv)])
    gf = comm.all_gather([pad(flags, 3)])
    a_all = torch.cat([ga[r][: b - a] for r, (a, b) in enumerate(sizes)])
    f_all = torch.cat([gf[r][: b - a] for r, (a, b) in enumerate(sizes)]).cpu().numpy()
    out = BatchSolveReport(a_all if return_device else _host(a_all), None, None,
                           f_all[:, 0].astype(np.int64), f_all[:, 1].astype(bool), rep.wall_time,
                           f_all[:, 2].astype(bool))
    return 0, a_all.shape[0], out


def rank_order_sum(tensors):
    """Elementwise sum in rank order (fixed, identical on every rank)."""
    out = tensors[0].clone()
    for t in tensors[1:]:
        out += t
    return out


class LocalComm:
    """N emulated ranks in one process: all_gather of the per-rank list is the list itself."""

    def __init__(self, world):
        self.world = world

    def all_gather(self, per_rank):
        assert len(per_rank) == self.world
        return list(per_rank)

    def barrier(self):
        pass


class DistComm:
    """One rank per process over torch.distributed (NCCL for CUDA tensors, gloo for CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)

    def barrier(self):
        self.dist.barrier(group=self.group)

    def all_gather(self, per_rank):
        assert len(per_rank) == 1
        t = per_rank[0].contiguous()
        out = t.new_empty((self.world * t.numel(),))
        self.dist.all_gather_into_tensor(out, t.reshape(-1), group=self.group)
        return [out[r * t.numel():(r + 1) * t.numel()].view(t.shape) for r in range(self.world)]


class _Shard:
    def __init__(self, dm, y, ws):
        self.dm = dm
        self.y = y
        self.ws = ws


def solve_bak_rowsharded(x_shards, y_shards, config: SolveConfig | None = None, comm=None, a0=None, *,
                         variant="gram", return_device=False):
    """Solve one system whose rows are split over ranks.

    x_shards / y_shards: list of this process's shards (one for DistComm; all N
    for LocalComm), each a (rows_r, vars) matrix (numpy / torch / DeviceMatrix)
    and its (rows_r,) target.  Returns one SolveReport per local shard: a_hat is
    the (replicated) coefficient vector, residual the shard's rows of y - x a.

    variant="gram"  : one pass per sweep, partials all-gathered per sweep (labelled
                      reformulation, any ordering).
    variant="stream": the EXACT per-column sweep; every column's partial dot is
                      all-reduced inside the kernel through peer-mapped mailboxes
                      (one shard per process, cyclic ordering).
    """
    if variant not in ("gram", "stream"):
        raise ValueError(f"unknown variant {variant!r}")
    cfg = config if config is not None else SolveConfig()
    torch = _torch()
    lib = _lib.load()
    if comm is None:
        comm = LocalComm(len(x_shards))
    shards = []
    for xs, ys in zip(x_shards, y_shards):
        dm = to_device_matrix(xs)
        yd = _to_device_vector(ys, dm.np_dtype, dm.data.device)
        if yd.shape[0] != dm.obs:
            raise ValueError(f"y has length {yd.shape[0]}, expected {dm.obs}")
        shards.append(_Shard(dm, yd, None))
    nv = shards[0].dm.vars
    code = shards[0].dm.code
    if any(s.dm.vars != nv or s.dm.code != code for s in shards):
        raise ValueError("shards must share vars and dtype")
    dev = shards[0].dm.data.device
    st = _stream_ptr(torch, dev)
    t0 = time.perf_counter()
    for s in shards:
        wsb = max(lib.bak_gram_matrix_workspace(code, s.dm.obs, nv), lib.bak_colnorms_workspace(code, s.dm.obs, nv),
                  lib.bak_residual_workspace(code, s.dm.obs, nv), 1 << 16)
        s.ws = _Workspace(torch, dev, wsb)

    # ||y||^2, column norms and G: local pieces, gathered, summed in rank order
    def local_sumsq(s):
        out = torch.empty(1, dtype=s.y.dtype, device=dev)
        _lib.check(lib.bak_colnorms(code, _ptr(s.y), s.dm.obs, 1, s.dm.obs, _ptr(out), s.ws.ptr, s.ws.nbytes, st),
                   "bak_colnorms(y)")
        return out.double()

    ynorm2 = float(rank_order_sum(comm.all_gather([local_sumsq(s) for s in shards])).item())
    tdt = shards[0].y.dtype
    if ynorm2 == 0.0:
        reps = []
        for s in shards:
            a_z = torch.zeros(nv, dtype=tdt, device=dev)
            r_z = torch.zeros(s.dm.obs, dtype=tdt, device=dev)
            reps.append(SolveReport(a_z if return_device else a_z.cpu().numpy(),
                                    r_z if return_device else r_z.cpu().numpy(),
                                    [] if cfg.record_history else None, 0, True, time.perf_counter() - t0,
                                    variant="gram-rowshard"))
        return reps
    norms = rank_order_sum(comm.all_gather([colnorms(s.dm, s.ws).double() for s in shards])).to(tdt)
    norms_h = norms.cpu().numpy()
    if not norms_h.any():
        raise ValueError("every column of x has zero norm; nothing to solve")
    if a0 is not None:
        a = _to_device_vector(a0, shards[0].dm.np_dtype, dev, "a0").clone()
        if a.shape[0] != nv:
            raise ValueError(f"a0 has length {a.shape[0]}, expected {nv}")
    else:
        a = torch.zeros(nv, dtype=tdt, device=dev)
    for s in shards:
        s.e = torch.empty_like(s.y)
        if a0 is not None:
            _lib.check(lib.bak_residual(code, s.dm.ptr, s.dm.obs, nv, s.dm.ldx, _ptr(a), _ptr(s.y), _ptr(s.e),
                                        s.ws.ptr, s.ws.nbytes, st), "bak_residual")
        else:
            s.e.copy_(s.y)
    thresh2 = cfg.tol * cfg.tol * ynorm2 if cfg.tol > 0 else -1.0
    if variant == "stream":
        if len(shards) != 1 or isinstance(comm, LocalComm) and comm.world > 1:
            raise ValueError("variant='stream' runs one shard per process (DistComm); "
                             "use sweep_rowshard(nranks_local=N) to emulate ranks on one device")
        if cfg.ordering != "cyclic":
            raise ValueError("variant='stream' supports ordering='cyclic'")
        s0 = shards[0]
        world = getattr(comm, "world", 1)
        rank = getattr(comm, "rank", 0)
        mb = getattr(comm, "_bak_mailboxes", None)
        if mb is None or mb.nranks != world:
            if mb is not None:
                mb.close()  # release the replaced mailbox and its peer mappings
            mb = Mailboxes(world, comm if world > 1 else None, dev)
            try:
                comm._bak_mailboxes = mb
            except AttributeError:
                pass
        hist = torch.zeros(cfg.max_iter, dtype=torch.float64, device=dev) if cfg.record_history else None
        status = sweep_rowshard(s0.dm, s0.e, a, norms, cfg.max_iter, thresh2, mb, rank, world, 1, history=hist)
        stat = status.cpu().numpy()
        if int(stat[2]):
            raise _lib.BakError(f"bak_sweep_rowshard device error {int(stat[2])} (3 = exchange timeout)")
        sweeps, converged = int(stat[0]), bool(stat[1])
        # status[3]: the kernel that ran — the on-chip GRID sweep (rows fit on chip) or the STREAM pass
        label = "grid-rowshard" if int(stat[3]) == _lib.VARIANTS["grid"] else "stream-rowshard"
        return _finish_sharded(shards, comm, a, hist, sweeps, converged, ynorm2, t0, return_device, label)
    # G and the first sweep's dots g = X^T e in one read of each shard (the DMMA
    # kernel's diagonal-block CTAs produce the dots); rows of partials padded
    # to the largest shard's count so the all-gather has one shape everywhere
    g0rows = max(int(lib.bak_gram_dot_rows(code, s.dm.obs, nv)) for s in shards)
    g0rows = int(max(comm.all_gather([torch.tensor([g0rows], device=dev) for _ in shards])).item())
    G_parts, g0_parts = [], []
    for s in shards:
        G = torch.empty((nv, nv), dtype=torch.float64, device=dev)
        g0 = torch.zeros((g0rows, nv), dtype=torch.float64, device=dev)
        _lib.check(lib.bak_gram_matrix_dot(code, s.dm.ptr, s.dm.obs, nv, s.dm.ldx, _ptr(G), _ptr(s.e), _ptr(g0),
                                           s.ws.ptr, s.ws.nbytes, st), "bak_gram_matrix_dot")
        G_parts.append(G)
        g0_parts.append(g0)
    G = rank_order_sum(comm.all_gather(G_parts))

    nblk = lib.bak_gram_pass_blocks(code, nv)
    for s in shards:
        s.gpart = torch.zeros((nblk, nv), dtype=torch.float64, device=dev)
        s.sqpart = torch.zeros(nblk, dtype=torch.float64, device=dev)
    delta = torch.zeros(nv, dtype=torch.float64, device=dev)
    ctrl = torch.zeros(4, dtype=torch.int64, device=dev)
    status = torch.zeros(4, dtype=torch.int64, device=dev)
    hist = torch.zeros(cfg.max_iter, dtype=torch.float64, device=dev) if cfg.record_history else None
    nz_mask = norms_h != 0
    if cfg.ordering == "cyclic":
        if nz_mask.all():
            cols_all, ncols, stride = None, nv, 0
        else:
            cols_all = torch.from_numpy(np.flatnonzero(nz_mask).astype(np.int32)).to(dev)
            ncols, stride = int(cols_all.numel()), 0
    else:
        gen = _permutation_chunks(cfg.ordering_seed, nv, None if nz_mask.all() else nz_mask)
        perms = np.stack([next(gen) for _ in range(cfg.max_iter)]).astype(np.int32)
        cols_all = torch.from_numpy(perms).to(dev)
        ncols, stride = perms.shape[1], perms.shape[1]

    fused = thresh2 < 0 and nv <= 256  # no early break: the last (TMA) pass also writes resid = y - x a
    for s in shards:
        s.resid = torch.empty_like(s.y) if fused else None

    def passes(apply, dot, last=False):
        for s in shards:
            fin = last and fused
            _lib.check(lib.bak_gram_pass_resid(code, s.dm.ptr, s.dm.obs, nv, s.dm.ldx, _ptr(s.e), _ptr(delta), apply,
                                               dot, _ptr(s.gpart), _ptr(s.sqpart), _ptr(ctrl),
                                               _ptr(a if fin else None), _ptr(s.y if fin else None),
                                               _ptr(s.resid if fin else None), _ptr(status), st),
                       "bak_gram_pass")
        gp = comm.all_gather([s.gpart for s in shards])
        sp = comm.all_gather([s.sqpart for s in shards])
        return torch.cat([g.reshape(-1) for g in gp]), torch.cat(sp)

    def solve(gp, sp, sweep):
        _lib.check(lib.bak_gram_solve(code, nv, _ptr(gp), _ptr(sp), gp.numel() // nv, sweep, cfg.max_iter, thresh2,
                                      _ptr(cols_all), ncols, stride, _ptr(norms), _ptr(G), _ptr(a), _ptr(delta),
                                      _ptr(hist), _ptr(ctrl), _ptr(status), st), "bak_gram_solve")

    gp = torch.cat([g.reshape(-1) for g in comm.all_gather(g0_parts)])
    sp = torch.zeros(1, dtype=torch.float64, device=dev)  # not read by the first solve
    for sweep in range(1, cfg.max_iter + 1):
        solve(gp, sp, sweep)
        gp, sp = passes(1, 1 if sweep < cfg.max_iter else 0, last=sweep == cfg.max_iter)
        if thresh2 >= 0 and sweep % 16 == 0 and int(ctrl[0].item()):
            break
    solve(gp, sp, cfg.max_iter + 1)
    stat = status.cpu().numpy()
    if int(stat[2]):
        raise _lib.BakError(f"GRAM row-shard device error {int(stat[2])} (3 = pipeline timeout)")
    sweeps, converged = int(stat[0]), bool(stat[1])

    return _finish_sharded(shards, comm, a, hist, sweeps, converged, ynorm2, t0, return_device, "gram-rowshard",
                           fused_resid=fused)


def _finish_sharded(shards, comm, a, hist, sweeps, converged, ynorm2, t0, return_device, label, fused_resid=False):
    """Residual y - x a per shard (bak.py:130) and the drift flag (bak.py:133-142)."""
    torch = _torch()
    lib = _lib.load()
    dev = shards[0].dm.data.device
    st = _stream_ptr(torch, dev)
    code = shards[0].dm.code
    nv = shards[0].dm.vars
    resids = []
    d2_parts = []
    for s in shards:
        if fused_resid:
            r = s.resid                                  # written by the last GRAM pass
        else:
            r = torch.empty_like(s.y)
            _lib.check(lib.bak_residual(code, s.dm.ptr, s.dm.obs, nv, s.dm.ldx, _ptr(a), _ptr(s.y), _ptr(r),
                                        s.ws.ptr, s.ws.nbytes, st), "bak_residual")
        d2 = torch.empty(1, dtype=torch.float64, device=dev)
        _lib.check(lib.bak_diff_norm2(code, _ptr(s.e), _ptr(r), s.dm.obs, _ptr(d2), s.ws.ptr, s.ws.nbytes, st),
                   "bak_diff_norm2")
        resids.append(r)
        d2_parts.append(d2)
    drift = float(np.sqrt(rank_order_sum(comm.all_gather(d2_parts)).item()))
    wall = time.perf_counter() - t0
    drift_warn = bool(drift / max(np.sqrt(ynorm2), np.finfo(np.float64).tiny) > DRIFT_TOL)
    history = hist[:sweeps].cpu().tolist() if hist is not None else None
    a_out = a if return_device else a.cpu().numpy()
    return [SolveReport(a_hat=a_out, residual=r if return_device else _host(r), residual_norm_history=history,
                        sweeps_run=sweeps, converged=converged, wall_time=wall, drift_warning=drift_warn,
                        variant=label) for r in resids]


# --------------------------------------------------------------------------
# exact per-column row sharding: in-kernel cross-GPU exchange per column
# --------------------------------------------------------------------------

class Mailboxes:
    """Per-rank mailbox buffers for bak_sweep_rowshard plus the peer pointers.

    DistComm: each rank allocates its mailbox, exports a CUDA IPC handle, the
    handles are all-gathered and every rank maps its peers' mailboxes (NVLink
    peer memory).  local=N: N emulated ranks share one device buffer.
    Epochs increase from call to call (``next_epochs``), so a record left by an
    earlier call never matches a later one.  The kernel tags records with 31
    bits; before the counter would wrap, every rank zeroes its own mailbox
    between two collective barriers and the count restarts at 0 (every rank
    calls ``next_epochs`` with the same counts, so they all reset together).
    """

    EPOCH_LIMIT = 0x7FFFFFFF

    def __init__(self, nranks, comm=None, device=None):
        torch = _torch()
        lib = _lib.load()
        self.nranks = nranks
        self.epoch = 0
        self._own = None
        self._comm = None if (comm is None or isinstance(comm, LocalComm)) else comm
        per = int(lib.bak_mailbox_bytes(nranks))
        self._per = per
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self._opened = []
        if comm is None or isinstance(comm, LocalComm):
            self.buf = torch.zeros(nranks * per, dtype=torch.uint8, device=dev)
            self.ptrs = [self.buf.data_ptr() + r * per for r in range(nranks)]
        else:
            # the exported mailbox is an allocation of its own (not a caching-
            # allocator block): peers map the base of the allocation a handle names
            self.buf = None
            p_own = ctypes.c_void_p()
            _lib.check(lib.bak_dev_alloc(per, ctypes.byref(p_own)), "bak_dev_alloc")
            self._own = p_own.value
            h = (ctypes.c_uint8 * 64)()
            _lib.check(lib.bak_ipc_get_handle(ctypes.c_void_p(self._own), h), "bak_ipc_get_handle")
            mine = torch.tensor(list(bytes(h)), dtype=torch.uint8, device=dev)
            handles = comm.all_gather([mine])
            self.ptrs = []
            for r, hr in enumerate(handles):
                if r == comm.rank:
                    self.ptrs.append(self._own)
                    continue
                raw = (ctypes.c_uint8 * 64)(*hr.cpu().tolist())
                p = ctypes.c_void_p()
                _lib.check(lib.bak_ipc_open_handle(raw, ctypes.byref(p)), "bak_ipc_open_handle")
                self.ptrs.append(p.value)
                self._opened.append(p.value)
        self.array = (ctypes.c_void_p * nranks)(*self.ptrs)

    def next_epochs(self, count):
        """Reserve ``count`` epochs (tags base+1 .. base+count) for one call."""
        if count + 2 >= self.EPOCH_LIMIT:
            raise ValueError(f"one row-sharded call needs {count} exchange epochs (> 2^31)")
        if self.epoch + count + 2 >= self.EPOCH_LIMIT:
            self.reset()
        base = self.epoch
        self.epoch += count + 2
        return base

    def reset(self):
        """Zero the mailboxes and restart the epoch count (collective over the ranks)."""
        torch = _torch()
        lib = _lib.load()
        torch.cuda.synchronize()  # no kernel of this rank still reads or writes a mailbox
        if self._comm is not None:
            self._comm.barrier()  # ... nor one of a peer
        if self.buf is not None:
            self.buf.zero_()
        else:
            _lib.check(lib.bak_dev_zero(ctypes.c_void_p(self._own), self._per), "bak_dev_zero")
        torch.cuda.synchronize()
        if self._comm is not None:
            self._comm.barrier()  # every mailbox is zero before any rank posts again
        self.epoch = 0

    def close(self):
        """Unmap the peers' mailboxes and free this rank's (idempotent)."""
        try:
            lib = _lib.load()
        except Exception:  # interpreter shutdown
            return
        for p in getattr(self, "_opened", ()):
            lib.bak_ipc_close(ctypes.c_void_p(p))
        self._opened = []
        if getattr(self, "_own", None):
            lib.bak_dev_free(ctypes.c_void_p(self._own))
            self._own = None

    def __del__(self):
        self.close()


def sweep_rowshard(dm, e, a, norms, max_iter, thresh2, mailboxes, rank, nranks, nranks_local=1, history=None,
                   status=None, stream=None):
    """Launch the exact per-column row-sharded sweep (thin wrapper over the C ABI).

    nranks_local > 1 emulates that many ranks in one launch on this device:
    dm/e hold the rows of all of them (split evenly) and a/status/history hold
    one replica per emulated rank.
    """
    torch = _torch()
    lib = _lib.load()
    dev = dm.data.device
    st = stream if stream is not None else _stream_ptr(torch, dev)
    ctas = max(1, (lib.bak_device_sm_count() or 148) // nranks_local)
    # (>= the on-chip GRID kernel's exchange records, used when one rank's rows fit on chip)
    ws = _Workspace(torch, dev, max(nranks_local * max(2 * ctas * 32, 2048), 96 * 1024) + 4096)
    if status is None:
        status = torch.zeros(4 * nranks_local, dtype=torch.int64, device=dev)
    base = mailboxes.next_epochs(max_iter * dm.vars + 1)
    _lib.check(lib.bak_sweep_rowshard(dm.code, dm.ptr, dm.obs, dm.vars, dm.ldx, _ptr(norms), _ptr(e), _ptr(a),
                                      max_iter, thresh2, _ptr(history), _ptr(status), rank, nranks, mailboxes.array,
                                      base, nranks_local, ws.ptr, ws.nbytes, st), "bak_sweep_rowshard")
    return status
