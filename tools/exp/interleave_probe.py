"""Per-call kernel time of each method when repeated vs interleaved with the other methods
(the bench's step order), on the bench shape.  Diagnoses the gap between ab_rounds and bench."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W

c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device='cuda')
M = ["B1", "B2", "B3", "P"]


def timed(seq):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in seq]
    for (a, b), m in zip(ev, seq):
        a.record()
        g.normal(m, out=out)
        b.record()
    torch.cuda.synchronize()
    return [a.elapsed_time(b) for a, b in ev]


for m in M:
    g.normal(m, out=out)
torch.cuda.synchronize()
for m in M:
    t = timed([m] * 6)
    print("repeated %-3s" % m, " ".join("%.3f" % x for x in t))
t = timed(M * 6)
for i, m in enumerate(M):
    print("interleaved %-3s" % m, " ".join("%.3f" % x for x in t[i::4]))
# gaps: a kernel right after a sync (idle GPU) vs back-to-back
for m in M:
    r = []
    for _ in range(4):
        torch.cuda.synchronize()
        r += timed([m])
    print("after-idle %-3s" % m, " ".join("%.3f" % x for x in r))
