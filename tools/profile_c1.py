"""Warm C1 calls (B1, 2^20 normals over 1024 streams) for an ncu capture of the last one:
    ncu --cache-control none -k regex:kernel -s 5 -c 1 python tools/profile_c1.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

c = W.C1
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
for _ in range(6):
    g.normal("B1", out=out)
torch.cuda.synchronize()
print("ok")
