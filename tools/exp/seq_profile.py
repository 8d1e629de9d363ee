"""One warm-up + one profiled sequential-mode call (2^31 normals over 2^16 streams) per method, for ncu."""
import sys, torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W
c = W.C5_SHARD
out = torch.empty(c.n, dtype=torch.float64, device='cuda')
for m in sys.argv[1].split(','):
    g = P.Generator(c.seed, c.streams)
    for _ in range(2):
        g.normal_seq(m, out=out)
    torch.cuda.synchronize()
    g.close()
print("ok")
