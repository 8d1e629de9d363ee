"""Mid-size calls for B3, P2, R (2^16 streams): us per call."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P

g = P.Generator(3, 1 << 16)
out = torch.empty(1 << 24, dtype=torch.float64, device='cuda')
for m in ("B3", "P2", "R"):
    for L in (1 << 21, 1 << 22, 1 << 23):
        for _ in range(3):
            g.normal(m, out=out[:L])
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(30):
            g.normal(m, out=out[:L])
        b.record()
        torch.cuda.synchronize()
        print(m, L, "%.1f us" % (a.elapsed_time(b) / 30 * 1e3))
