"""Step time of the bench step for each cyclic order of the four methods (steady state)."""
import itertools
import sys
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W

c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device='cuda')
orders = [("B1",) + p for p in itertools.permutations(("B2", "B3", "P"))]
for rnd in range(2):
    for order in orders:
        for _ in range(3):
            for m in order:
                g.normal(m, out=out)
        ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in order] for _ in range(10)]
        for s in range(10):
            for i, m in enumerate(order):
                ev[s][i][0].record()
                g.normal(m, out=out)
                ev[s][i][1].record()
        torch.cuda.synchronize()
        per = {m: sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(10)) / 10 for i, m in enumerate(order)}
        print(rnd, ",".join(order), "step %.2f" % sum(per.values()), " ".join("%s %.3f" % (m, per[m]) for m in ("B1", "B2", "B3", "P")))
