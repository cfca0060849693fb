"""HBM bandwidth calibration for the memory-bound kernels' traffic mix:
write-only (fill), 1:1 copy and a 1:2 read:write pattern (two copies of one
source), 1 GiB buffers, CUDA events, best of 10."""
import torch
n = 1 << 28  # 2^28 float32 = 1 GiB
x = torch.randn(n, device="cuda")
y = torch.empty(n, device="cuda")
z = torch.empty(n, device="cuda")


def t(fn):
    best = 1e9
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    return best / 1e3


gb = 4 * n / 1e9
tf = t(lambda: y.fill_(1.0)); print(f"write-only fill : {gb / tf:.0f} GB/s")
tc = t(lambda: y.copy_(x)); print(f"copy 1:1        : {2 * gb / tc:.0f} GB/s (read+write)")
td = t(lambda: (y.copy_(x), z.copy_(x))); print(f"two copies 1:1  : {4 * gb / td:.0f} GB/s")
tm = t(lambda: torch.mul(x, 2.0, out=y)); print(f"mul 1:1         : {2 * gb / tm:.0f} GB/s")
