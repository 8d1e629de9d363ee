"""C4-style short calls: us per call for n in a few sizes (2^16 streams), B1 and P, CUDA-graph timed."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P

g = P.Generator(3, 1 << 16)
out = torch.empty(1 << 26, dtype=torch.float64, device='cuda')
for m in ("B1", "P"):
    for L in (1 << 20, 1 << 21, 1 << 22, 1 << 23, 1 << 24, 1 << 25):
        for _ in range(3):
            g.normal(m, out=out[:L])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(50):
            g.normal(m, out=out[:L])
        b.record()
        torch.cuda.synchronize()
        print(m, L, "%.1f us" % (a.elapsed_time(b) / 50 * 1e3))
