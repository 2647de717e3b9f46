"""Raw pinned host -> device copy bandwidth (1 and 2 streams, chunked), to
compare with the e2e upload rate of the pipelined GRAM path."""
import torch

dev = torch.device("cuda", 0)
nbytes = 8 << 30
h = torch.empty(nbytes // 8, dtype=torch.float64, pin_memory=True)
h.fill_(1.0)
d = torch.empty_like(h, device=dev)
for nstreams in (1, 2, 4):
    for chunk in (256 << 20, 1 << 30):
        streams = [torch.cuda.Stream(dev) for _ in range(nstreams)]
        torch.cuda.synchronize()
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record()
        n = nbytes // 8
        c = chunk // 8
        main = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(main)
        for i, off in enumerate(range(0, n, c)):
            with torch.cuda.stream(streams[i % nstreams]):
                d[off:off + c].copy_(h[off:off + c], non_blocking=True)
        for s in streams:
            main.wait_stream(s)
        t1.record()
        torch.cuda.synchronize()
        ms = t0.elapsed_time(t1)
        print(f"streams={nstreams} chunk={chunk >> 20}MB: {nbytes / ms / 1e6:.1f} GB/s", flush=True)

# the pipelined GRAM upload pattern: row blocks of a column-major matrix via
# bak_copy_rows_h2d (cudaMemcpy2DAsync) on two copy streams
import ctypes  # noqa: E402
import os  # noqa: E402
import sys  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_12570_b200 import _lib  # noqa: E402

lib = _lib.load()
del d
obs, nv = 1 << 22, 256
hx = torch.empty((nv, obs), dtype=torch.float64, pin_memory=True)
hx.fill_(1.0)
dx = torch.empty((nv, obs), dtype=torch.float64, device=dev)
for rows_chunk in (1 << 17, 1 << 19, 1 << 20):
    streams = [torch.cuda.Stream(dev), torch.cuda.Stream(dev)]
    torch.cuda.synchronize()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0.record()
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for i, r0 in enumerate(range(0, obs, rows_chunk)):
        cs = streams[i % 2]
        _lib.check(lib.bak_copy_rows_h2d(ctypes.c_void_p(dx.data_ptr()), obs, ctypes.c_void_p(hx.data_ptr()), obs, r0,
                                         min(rows_chunk, obs - r0), nv, 8, ctypes.c_void_p(cs.cuda_stream)), "copy")
    for s in streams:
        main.wait_stream(s)
    t1.record()
    torch.cuda.synchronize()
    ms = t0.elapsed_time(t1)
    print(f"2D row blocks of {rows_chunk} rows ({rows_chunk * nv * 8 >> 20} MB): {obs * nv * 8 / ms / 1e6:.1f} GB/s",
          flush=True)
