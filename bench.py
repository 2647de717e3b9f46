#!/usr/bin/env python
"""SolveBak column sweep on B200 — sweeps/s and x-stream HBM GB/s vs roofline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

One JSON line on rank 0 (driver contract).  A "step" is one full solve through
the drop-in API (norms, the sweeps, the recomputed residual, drift) over one
synthetic system of the configuration's shape (BASELINE.json configs; seeded
device RNG with the reference's distributions — no dataset is involved).

  value      sweeps/s of whole solves with inputs resident in HBM (CUDA events)
  e2e        the same metric through solve_bak() with pinned HOST inputs:
             host->device copy of x, y and device->host of a, residual inside
             the timed region
  roofline   the dominant kernel (the sweep) timed alone with CUDA events:
             algorithmic bytes = obs*vars*sizeof(T) per sweep (one read of x)
  cpu_baseline  the CPU oracle (numpy restatement of the reference, bit-for-bit
             equal to it on the fixture host) on a bounded sample, 1 core as the
             reference pins BLAS to one thread (bak.py:184)

--impl reference runs that CPU port alone (the reference arm).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs
    "c1": dict(kind="system", obs=10_000, vars=100, dtype="f64", sweeps=100, tol=0.0, noise=0.01,
               desc="tall dense fp64 10,000x100, 100 sweeps"),
    "c2": dict(kind="c2", obs=4096, vars=4096, dtype="f64", sweeps=50, tol=0.0,
               desc="square fp64 n=4096 (4I + N(0,1)/sqrt(n)), 50 sweeps"),
    "c2b": dict(kind="c2", obs=4096, vars=4096, dtype="f64", sweeps=50, tol=1e-10,
                desc="square fp64 n=4096, early break at 1e-10"),
    "c3": dict(kind="system", obs=1 << 24, vars=256, dtype="f64", sweeps=20, tol=0.0, noise=0.01,
               desc="very tall fp64 2^24x256, 20 sweeps"),
    "c3f32": dict(kind="system", obs=1 << 24, vars=256, dtype="f32", sweeps=20, tol=0.0, noise=0.01,
                  desc="very tall fp32 2^24x256, 20 sweeps"),
    "c4": dict(kind="c4", obs=1000, vars=1_000_000, dtype="f64", sweeps=10, tol=0.0,
               desc="wide fp64 1,000x1,000,000, 10 sweeps"),
    "c5": dict(kind="batched", obs=512, vars=32, nsys=65536, dtype="f32", sweeps=200, tol=0.0, noise=0.01,
               desc="65,536 batched fp32 512x32 systems, 200 sweeps"),
}
DEFAULT_CONFIG = "c3"
METRIC = "sweeps/sec and x-stream HBM GB/s vs roofline at 1/2/4/8 B200; CPU baseline"
SPEC_HBM_GBS = 8000.0

REASON_FIELDS = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, index):
        self.index = index
        self.lines = []
        self.proc = None

    def __enter__(self):
        q = "clocks.sm,clocks.max.sm," + ",".join("clocks_event_reasons." + r for r in REASON_FIELDS)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 2 + len(REASON_FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(REASON_FIELDS, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------------------
# synthetic inputs on the device (seeded; reference distributions)
# --------------------------------------------------------------------------

def make_inputs(cfg, dev, seed=1234):
    import torch
    import paper_2104_12570_b200 as pb
    tdt = torch.float64 if cfg["dtype"] == "f64" else torch.float32
    npdt = np.float64 if cfg["dtype"] == "f64" else np.float32
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    obs, nv = cfg["obs"], cfg["vars"]
    vec = 16 // (8 if cfg["dtype"] == "f64" else 4)
    ld = (obs + vec - 1) // vec * vec
    if cfg["kind"] == "batched":
        nsys = cfg["nsys"]
        data = torch.zeros((nsys, nv, ld), dtype=tdt, device=dev)
        data[:, :, :obs].normal_(generator=g)
        a_true = torch.rand((nsys, nv), dtype=tdt, device=dev, generator=g) * 2 - 1
        y = torch.bmm(data[:, :, :obs].transpose(1, 2), a_true.unsqueeze(2)).squeeze(2)
        y += cfg["noise"] * torch.randn((nsys, obs), dtype=tdt, device=dev, generator=g)
        return pb.DeviceBatch(data, obs, npdt), y.contiguous()
    data = torch.zeros((nv, ld), dtype=tdt, device=dev)
    for j0 in range(0, nv, 4096):  # chunked to bound RNG temporaries
        j1 = min(nv, j0 + 4096)
        data[j0:j1, :obs].normal_(generator=g)
    if cfg["kind"] == "c2":
        data[:, :obs] /= float(np.sqrt(obs))
        idx = torch.arange(obs, device=dev)
        data[idx, idx] += 4.0
    if cfg["kind"] == "c4":
        y = torch.randn(obs, dtype=tdt, device=dev, generator=g)
    else:
        a_true = torch.rand(nv, dtype=tdt, device=dev, generator=g) * 2 - 1
        y = torch.zeros(obs, dtype=tdt, device=dev)
        for j0 in range(0, nv, 4096):
            j1 = min(nv, j0 + 4096)
            y += data[j0:j1, :obs].t() @ a_true[j0:j1]
        if cfg.get("noise"):
            y += cfg["noise"] * torch.randn(obs, dtype=tdt, device=dev, generator=g)
    return pb.DeviceMatrix(data, obs, nv, npdt), y


# --------------------------------------------------------------------------
# CPU baseline: the oracle on a bounded sample (1 core, like the reference)
# --------------------------------------------------------------------------

def cpu_baseline(cfg, dm, y, budget_s=12.0):
    import torch
    from threadpoolctl import threadpool_limits
    from oracle import bak_oracle as orc
    cores = 1
    if cfg["kind"] == "batched":
        data, obs = dm.data, dm.obs
        n = 0
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < budget_s and n < dm.nsys:
            x = np.asfortranarray(data[n, :, :obs].cpu().numpy().T)
            yy = y[n].cpu().numpy()
            ts = time.perf_counter()
            orc.solve(x, yy, max_iter=cfg["sweeps"], tol=cfg["tol"])
            if n == 0:
                t0 = ts  # exclude first-call warm-up
                n_done_t = 0.0
            n_done_t += time.perf_counter() - ts
            n += 1
        per_sys = n_done_t / n
        sps = cfg["sweeps"] / per_sys / dm.nsys  # batch-sweeps/s
        return {"value": sps, "unit": "sweeps/s", "cores": cores, "kind": "port",
                "sample": f"{n} of {dm.nsys} systems solved ({cfg['sweeps']} sweeps each) by the numpy oracle "
                          f"on 1 core; batch-sweeps/s = sweeps / (per-system time x {dm.nsys})"}
    obs, nv = dm.obs, dm.vars
    # a full-length column sample: per-column cost at the real obs
    ncs = min(nv, 32 if obs >= (1 << 22) else (256 if obs >= 100_000 else nv))
    if cfg["kind"] == "c4":
        ncs = 20_000
    x = np.asfortranarray(dm.data[:ncs, :obs].cpu().numpy().T)
    yy = y.cpu().numpy().copy()
    n2 = orc.column_norms_sq(x)
    a = np.zeros(ncs, dtype=x.dtype)
    tmp = np.empty_like(yy)
    order = np.arange(ncs)
    cols_done = 0
    with threadpool_limits(limits=1, user_api="blas"):
        orc.sweep_loop(x, yy, a, n2, tmp, order, None, 1, None, None)  # warm-up
        t0 = time.perf_counter()
        while True:
            orc.sweep_loop(x, yy, a, n2, tmp, order, None, 1, None, None)
            cols_done += ncs
            if time.perf_counter() - t0 > budget_s * 0.5:
                break
        t = time.perf_counter() - t0
    t_col = t / cols_done
    sps = 1.0 / (t_col * nv)
    return {"value": sps, "unit": "sweeps/s", "cores": cores, "kind": "port",
            "sample": f"{cols_done} column steps of the numpy oracle (bit-identical restatement of "
                      f"baksolve.bak._run_sweeps) on the first {ncs} full-length columns ({obs} rows), "
                      f"1 core; sweeps/s = 1/(t_col x {nv} columns)"}


# --------------------------------------------------------------------------
# our arm
# --------------------------------------------------------------------------

def run_ours(args, cfg, rank, world, dev):
    import torch
    import paper_2104_12570_b200 as pb
    from paper_2104_12570_b200 import _lib
    from paper_2104_12570_b200.bak import _Workspace, _ptr, _stream_ptr, _workspace_bytes

    lib = _lib.load()
    torch.cuda.set_device(dev)
    dm, y = make_inputs(cfg, dev, seed=1234 + rank)
    scfg = pb.SolveConfig(max_iter=cfg["sweeps"], tol=cfg["tol"])
    batched = cfg["kind"] == "batched"
    ts = 8 if cfg["dtype"] == "f64" else 4

    def step():
        if batched:
            return pb.solve_bak_batched(dm, y, scfg, return_device=True)
        return pb.solve_bak(dm, y, scfg, variant=args.variant, return_device=True)

    for _ in range(args.warmup):
        rep = step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    sweeps_done = int(np.sum(rep.sweeps_run)) if batched else rep.sweeps_run
    variant = "batched" if batched else rep.variant

    # ---- value: whole solves, inputs resident in HBM ----
    st = torch.cuda.current_stream()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = lib.bak_launch_count()
    total_sweeps = 0
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ev0.record(st)
        for _ in range(args.steps):
            rep = step()
            total_sweeps += (int(rep.sweeps_run.max()) if batched else rep.sweeps_run)
        ev1.record(st)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
    launches = lib.bak_launch_count() - l0
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    units = cfg["sweeps"] * world  # sweeps of one system / one batch per rank per step
    value = units * args.steps / (ms / 1e3)

    # ---- roofline: the sweep kernel alone ----
    code = dm.code
    if batched:
        xbytes_per_sweep = dm.nsys * cfg["obs"] * cfg["vars"] * ts
        kev0, kev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kev0.record(st)
        for _ in range(args.steps):
            r = pb.solve_bak_batched(dm, y, scfg, return_device=True)
        kev1.record(st)
        torch.cuda.synchronize()
        k_ms = kev0.elapsed_time(kev1) / args.steps
        k_sweeps = int(r.sweeps_run.max())
        kernel = "batched_kernel (whole per-system solve, one CTA per system)"
    else:
        ws = _Workspace(torch, dev, _workspace_bytes(lib, code, dm.obs, dm.vars, _lib.VARIANTS[args.variant]))
        norms = pb.colnorms(dm, ws)
        e = torch.empty_like(y)
        a = torch.zeros(dm.vars, dtype=y.dtype, device=dev)
        status = torch.zeros(4, dtype=torch.int64, device=dev)
        vcode = _lib.VARIANTS[args.variant]
        k_tot = 0.0
        for _ in range(args.steps):
            e.copy_(y)
            a.zero_()
            kev0, kev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            kev0.record(st)
            _lib.check(lib.bak_sweep(code, vcode, dm.ptr, dm.obs, dm.vars, dm.ldx, _ptr(norms), None, dm.vars, 0,
                                     _ptr(e), _ptr(a), cfg["sweeps"], -1.0 if cfg["tol"] == 0 else
                                     cfg["tol"] ** 2 * float((y.double() ** 2).sum()), None, _ptr(status),
                                     ws.ptr, ws.nbytes, _stream_ptr(torch, dev)), "bak_sweep")
            kev1.record(st)
            torch.cuda.synchronize()
            k_tot += kev0.elapsed_time(kev1)
        k_ms = k_tot / args.steps
        k_sweeps = int(status[0].item())
        xbytes_per_sweep = dm.obs * dm.vars * ts
        kernel = f"sweep_kernel[{variant}]"
    alg_bytes = xbytes_per_sweep * k_sweeps
    achieved = alg_bytes / (k_ms / 1e3) / 1e9
    peak, peak_kind = load_peaks()
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tr = json.load(f)
        key = f"{args.config}:{variant}"
        if key in tr:
            traffic = tr[key]
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "frac_of_spec_8000": round(achieved / SPEC_HBM_GBS, 4),
                "peak_source": peak_kind, "traffic": traffic, "kernel": kernel,
                "kernel_ms": round(k_ms, 4), "alg_bytes_per_launch": alg_bytes,
                "sweeps_per_launch": k_sweeps}

    # ---- e2e: through solve_bak with pinned host buffers ----
    e2e = None
    if not args.no_e2e:
        if batched:
            hx = torch.empty(dm.data.shape, dtype=dm.data.dtype, pin_memory=True)
            hx.copy_(dm.data)
            hxv = hx.transpose(1, 2)[:, :cfg["obs"], :]  # (nsys, obs, vars) view
            hy = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            hy.copy_(y)
            h2d = hx.numel() * ts + hy.numel() * ts

            def e2e_step():
                r = pb.solve_bak_batched(hxv, hy, scfg)
                return r, r.a_hat.nbytes + r.residual.nbytes + r.sweeps_run.nbytes * 4
        else:
            hx = torch.empty(dm.data.shape, dtype=dm.data.dtype, pin_memory=True)
            hx.copy_(dm.data)
            hxv = hx.t()[: dm.obs]  # (obs, vars) column-major view of the pinned buffer
            hy = torch.empty(y.shape, dtype=y.dtype, pin_memory=True)
            hy.copy_(y)
            h2d = hx.numel() * ts + hy.numel() * ts

            def e2e_step():
                r = pb.solve_bak(hxv, hy, scfg, variant=args.variant)
                return r, r.a_hat.nbytes + r.residual.nbytes + dm.vars * ts + 64
        r, d2h = e2e_step()
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ev0.record(st)
        for _ in range(args.steps):
            r, d2h = e2e_step()
        ev1.record(st)
        torch.cuda.synchronize()
        ems = ev0.elapsed_time(ev1)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": units * args.steps / (ems / 1e3), "unit": "sweeps/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": int(d2h), "ms_per_step": round(ems / args.steps, 3)}
        del hx, hy

    out = {
        "metric": METRIC, "value": round(value, 3), "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_per_step, 4), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": cfg["dtype"], "data": "synthetic",
        "config": {"workload": args.config, "desc": cfg["desc"], "obs": cfg["obs"], "vars": cfg["vars"],
                   "nsys": cfg.get("nsys", 1), "sweeps_per_step": cfg["sweeps"], "tol": cfg["tol"],
                   "variant": variant, "x_gb_per_sweep": round(xbytes_per_sweep / 1e9, 4),
                   "x_stream_gbs_whole_solve": round(xbytes_per_sweep * total_sweeps / (ms / 1e3) / 1e9, 1),
                   "l2": "inputs larger than L2 (126 MB)" if xbytes_per_sweep > 126e6 else
                         "x fits in L2: re-read each sweep from L2 by design",
                   "parallelism": f"dp{world}" if world > 1 else "single"},
        "roofline": roofline,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(cfg, dm, y)
    return out


def run_reference(args, cfg, rank, world):
    """The reference arm: the CPU port of the reference algorithm on this host."""
    if rank != 0:
        return None
    import torch
    dev = torch.device("cuda", 0) if torch.cuda.is_available() else None
    if dev is not None:
        dm, y = make_inputs(cfg, dev, seed=1234)
    else:  # CPU-only host: same shapes from the oracle generator (small configs only)
        raise SystemExit(json.dumps({"impl": "reference", "unavailable": "needs the synthetic inputs; no device"}))
    vals = []
    cb = None
    for _ in range(max(1, args.steps)):
        cb = cpu_baseline(cfg, dm, y, budget_s=max(4.0, 60.0 / max(1, args.steps)))
        vals.append(cb["value"])
    v = float(np.median(vals))
    cb["value"] = v
    return {"metric": METRIC, "value": v, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": cfg["dtype"], "data": "synthetic",
            "config": {"workload": args.config, "desc": cfg["desc"], "obs": cfg["obs"], "vars": cfg["vars"],
                       "nsys": cfg.get("nsys", 1), "sweeps_per_step": cfg["sweeps"]},
            "impl": "reference", "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default=DEFAULT_CONFIG, choices=sorted(CONFIGS))
    ap.add_argument("--variant", default="auto")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch
    if args.impl == "reference":
        out = run_reference(args, cfg, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if world > 1:
        torch.distributed.init_process_group("nccl", device_id=dev)
    out = run_ours(args, cfg, rank, world, dev)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
