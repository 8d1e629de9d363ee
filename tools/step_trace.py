"""Per-call device times of the bench step (B1,B2,B3,P back to back) over many steps, with
nvidia-smi clocks/power sampled alongside: python tools/step_trace.py [steps]"""
import subprocess
import sys

import torch

sys.path.insert(0, ".")
import paper_1004_3105_b200 as P  # noqa: E402
from paper_1004_3105_b200 import workloads as W  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device="cuda")
M = ("B1", "B2", "B3", "P")
for _ in range(3):
    for m in M:
        g.normal(m, out=out)
torch.cuda.synchronize()
smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active",
                        "--format=csv,noheader", "-lms", "50"], stdout=subprocess.PIPE, text=True)
ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in M] for _ in range(steps)]
for s in range(steps):
    for i, m in enumerate(M):
        ev[s][i][0].record()
        g.normal(m, out=out)
        ev[s][i][1].record()
torch.cuda.synchronize()
smi.terminate()
lines = smi.communicate()[0].strip().splitlines()
for s in range(steps):
    print("step %2d " % s + " ".join("%s %.3f" % (m, ev[s][i][0].elapsed_time(ev[s][i][1])) for i, m in enumerate(M)))
print("smi:", lines[: 3], "...", lines[-3:], len(lines))
