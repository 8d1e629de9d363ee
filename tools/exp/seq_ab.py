"""Sequential-mode call time at the bench shape (2^31 normals over 2^16 streams, device output)
for the library in use (NRNG_LIB_OVERRIDE selects an A/B build): best of 3 after warm-up.

    python tools/exp/seq_ab.py [METHODS]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

c = W.C5_SHARD
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
res = []
for m in (sys.argv[1] if len(sys.argv) > 1 else "B1,B2,B3,P").split(","):
    g = P.Generator(c.seed, c.streams)
    for _ in range(10):
        g.normal_seq(m, out=out)
    best = 1e9
    for _ in range(3):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(3):
            g.normal_seq(m, out=out)
        b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b) / 3)
    res.append("%s %.3f" % (m, best))
    g.close()
print(os.path.basename(os.environ.get("NRNG_LIB_OVERRIDE", "default")), " ".join(res))
