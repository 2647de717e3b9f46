"""Achievable FP64 GEMM rate on this GPU (cuBLAS via torch) for G = X^T X shapes (tuning aid)."""
import torch

dev = torch.device("cuda", 0)


def t(f, n=3):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(n):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        f()
        e.record()
        torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


a = torch.randn(8192, 8192, dtype=torch.float64, device=dev)
ms = t(lambda: a @ a)
print("dgemm 8192^3", round(ms, 2), "ms", round(2 * 8192 ** 3 / ms / 1e9, 1), "TF")
del a
x = torch.randn(256, 1 << 24, dtype=torch.float64, device=dev)
fl = 2 * 256 * 256 * (1 << 24)
ms = t(lambda: x @ x.t())
print("G = X^T X (256 x 2^24) via matmul", round(ms, 2), "ms", round(fl / ms / 1e9, 1), "TF")
xb = x.view(256, 64, 1 << 18).permute(1, 0, 2)
ms = t(lambda: torch.bmm(xb, xb.transpose(1, 2)).sum(0))
print("G via bmm 64 chunks", round(ms, 2), "ms", round(fl / ms / 1e9, 1), "TF")
del x, xb
xf = torch.randn(256, 1 << 24, dtype=torch.float32, device=dev)
torch.backends.cuda.matmul.allow_tf32 = False
ms = t(lambda: xf @ xf.t())
print("sgemm G f32", round(ms, 2), "ms", round(fl / ms / 1e9, 1), "TF")
