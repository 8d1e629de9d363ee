"""Write-only and copy HBM bandwidth on this GPU (CUDA events, best of 5).

    python tools/hbm_probe.py
"""
import torch

n = 1 << 31  # 16 GiB of fp64
a = torch.empty(n, dtype=torch.float64, device="cuda")
b = torch.empty(n // 4, dtype=torch.float64, device="cuda")
c = torch.empty(n // 4, dtype=torch.float64, device="cuda")


def t(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


ms = t(lambda: a.fill_(1.5))
print("fill_ (write-only) 16 GiB: %.3f ms  %.1f GB/s" % (ms, 8 * n / ms / 1e6))
ms = t(lambda: a.zero_())
print("zero_ (memset)     16 GiB: %.3f ms  %.1f GB/s" % (ms, 8 * n / ms / 1e6))
ms = t(lambda: c.copy_(b))
print("copy_ 4 GiB -> 4 GiB:      %.3f ms  %.1f GB/s (read+write)" % (ms, 2 * 8 * (n // 4) / ms / 1e6))
