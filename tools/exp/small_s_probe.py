"""Calls over few streams (C1-like): us per call, CUDA-graph replay to remove host overhead."""
import sys
import torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P

for S, n in ((1024, 1 << 20), (1024, 1 << 22), (2048, 1 << 24)):
    g = P.Generator(1, S)
    out = torch.empty(n, dtype=torch.float64, device='cuda')
    for m in ("B1", "B2", "B3", "P"):
        for _ in range(3):
            g.normal(m, out=out)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            with torch.cuda.graph(gr, stream=s):
                for _ in range(20):
                    g.normal(m, out=out)
        torch.cuda.current_stream().wait_stream(s)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        gr.replay()
        b.record()
        torch.cuda.synchronize()
        print(m, S, n, "%.1f us" % (a.elapsed_time(b) / 20 * 1e3))
    g.close()
