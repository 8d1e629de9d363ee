"""One warm-up call + one profiled call of each BASELINE config's hot launch at its own shape
(C1 B1, C2 P, C3 B3, C4 n=2^22 B1 and P), for ncu captures of the small-S / mid-size paths.

    python tools/profile_configs.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

out = torch.empty(1 << 28, dtype=torch.float64, device="cuda")
cases = [(W.C1, "B1", W.C1.n), (W.C2, "P", W.C2.n), (W.C3, "B3", W.C3.n), (W.C4, "B1", 1 << 22), (W.C4, "P", 1 << 22)]
for c, m, n in cases:
    g = P.Generator(c.seed, c.streams)
    for _ in range(2):
        g.normal(m, out=out[:n], mu=c.mu, sigma=c.sigma)
    torch.cuda.synchronize()
    g.close()
print("ok")
