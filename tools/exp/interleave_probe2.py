"""B1's per-call time after different predecessors: what makes B1 slower inside the bench's
step than when repeated?"""
import sys
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W

c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device='cuda')
other = torch.empty(c.n // 8, dtype=torch.float64, device='cuda')
for m in ["B1", "B2", "B3", "P"]:
    g.normal(m, out=out)
torch.cuda.synchronize()


def b1_after(pre, reps=5):
    ts = []
    for _ in range(reps):
        pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        g.normal("B1", out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return " ".join("%.3f" % t for t in ts)


cyc = int(1.9e9 * 0.005)
print("after B1     ", b1_after(lambda: g.normal("B1", out=out)))
print("after sleep5 ", b1_after(lambda: torch.cuda._sleep(cyc)))
print("after sleep1 ", b1_after(lambda: torch.cuda._sleep(cyc // 5)))
print("after fill2G ", b1_after(lambda: other.fill_(1.0)))
print("after B2     ", b1_after(lambda: g.normal("B2", out=out)))
print("after B3     ", b1_after(lambda: g.normal("B3", out=out)))
print("after P      ", b1_after(lambda: g.normal("P", out=out)))
print("after B1+sl1 ", b1_after(lambda: (g.normal("B1", out=out), torch.cuda._sleep(cyc // 5))))
print("after P+sl5  ", b1_after(lambda: (g.normal("P", out=out), torch.cuda._sleep(cyc))))
# a different output buffer for B1 after B1
out2 = torch.empty(c.n, dtype=torch.float64, device='cuda')
print("after B1(out2)", b1_after(lambda: g.normal("B1", out=out2)))
