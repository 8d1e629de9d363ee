"""Sustained per-method clocks/power: each method back to back for ~1.5 s with nvidia-smi
sampling (clocks.sm, power.draw, throttle reasons): python tools/power_trace.py"""
import subprocess
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
for m in (sys.argv[1].split(",") if len(sys.argv) > 1 else ("B1", "B2", "B3", "P", "P2")):
    g.normal(m, out=out)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    k = 0
    t0 = time.time()
    while time.time() - t0 < 1.5:
        for _ in range(20):
            g.normal(m, out=out)
        k += 20
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    rows = [r.split(",") for r in smi.communicate()[0].strip().splitlines() if r.strip()]
    load = [r for r in rows if float(r[1]) > 200]
    clk = sorted(float(r[0]) for r in load) or [0]
    pw = sorted(float(r[1]) for r in load) or [0]
    reasons = sorted(set(r[2].strip() for r in load))
    print("%-3s %.3f ms/call over %d calls | sm MHz median %d min %d | W median %d max %d | reasons %s" % (
        m, e0.elapsed_time(e1) / k, k, clk[len(clk) // 2], clk[0], pw[len(pw) // 2], pw[-1], reasons))
