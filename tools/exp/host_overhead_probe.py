"""Host-side cost per short call (C4 regime): the Python Generator path vs the bare C-ABI call."""
import sys
import time
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P

g = P.Generator(3, 1 << 16)
out = torch.empty(1 << 10, dtype=torch.float64, device='cuda')
ptr = out.data_ptr()
lib = P.lib()
for _ in range(100):
    g.normal("B1", out=out)
torch.cuda.synchronize()


def t(fn, n=2000):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return (t1 - t0) / n * 1e6, (t2 - t0) / n * 1e6


print("Generator.normal   enqueue %.2f us  total %.2f us" % t(lambda: g.normal("B1", out=out)))
print("ctypes ABI call    enqueue %.2f us  total %.2f us" % t(lambda: lib.nrng_normal_boxmuller(g.h, ptr, 1024, 0.0, 1.0, 1)))
print("current_stream     %.2f us" % t(lambda: torch.cuda.current_stream().cuda_stream)[0])
print("set_stream (ctypes) %.2f us" % t(lambda: lib.nrng_set_stream(g.h, torch.cuda.current_stream().cuda_stream))[0])
print("empty kernel (torch add) enqueue %.2f total %.2f" % t(lambda: out.add_(0.0)))
