"""One warm-up + one profiled C3-shape call (2^28 normals over 2^16 streams) per method, for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

c = W.C3
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
for m in (sys.argv[1] if len(sys.argv) > 1 else "B2,B3").split(","):
    g = P.Generator(c.seed, c.streams)
    for _ in range(2):
        g.normal(m, out=out, mu=c.mu, sigma=c.sigma)
    torch.cuda.synchronize()
    g.close()
print("ok")
