"""C2-shape call time (2^24 normals over 2^14 streams, seed 7) for the given methods and the
library in use (NRNG_LIB_OVERRIDE selects an A/B build): best of 5 runs of 20 calls.

    python tools/exp/c2_ab.py [METHODS]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

c = W.C2
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
res = []
for m in (sys.argv[1] if len(sys.argv) > 1 else "P,P2").split(","):
    g = P.Generator(c.seed, c.streams)
    for _ in range(20):
        g.normal(m, out=out)
    best = 1e9
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(20):
            g.normal(m, out=out)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) * 1000 / 20)
    res.append("%s %.1f us" % (m, best))
    g.close()
print(os.path.basename(os.environ.get("NRNG_LIB_OVERRIDE", "default")), " ".join(res))
