"""One warm-up call + one profiled call per method at the bench shape (for ncu captures).

    python tools/profile_step.py [--methods B1,B2,B3,P] [--n LOG2N]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--methods", default="B1,B2,B3,P,P2,R,R1")
ap.add_argument("--log2n", type=int, default=31)
args = ap.parse_args()
c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(1 << args.log2n, dtype=torch.float64, device="cuda")
ms = args.methods.split(",")
for m in ms:
    g.normal(m, out=out)
torch.cuda.synchronize()
for m in ms:
    g.normal(m, out=out)
torch.cuda.synchronize()
print("ok", g.kernel_launches)
