"""Per-call time of one method over many consecutive calls (does it drift, and with what?)."""
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, '.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W

m = sys.argv[1] if len(sys.argv) > 1 else "B1"
calls = int(sys.argv[2]) if len(sys.argv) > 2 else 60
c = W.C5_SHARD
g = P.Generator(c.seed, c.streams)
out = torch.empty(c.n, dtype=torch.float64, device='cuda')
samples = []
stop = False


def smi():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,temperature.memory,clocks_throttle_reasons.active",
                            "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append((time.time(), r))
        time.sleep(0.05)


th = threading.Thread(target=smi)
th.start()
ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(calls)]
t0 = time.time()
for a, b in ev:
    a.record()
    g.normal(m, out=out)
    b.record()
torch.cuda.synchronize()
stop = True
th.join()
ts = [a.elapsed_time(b) for a, b in ev]
print(m, " ".join("%.2f" % t for t in ts))
for t, r in samples[:: max(1, len(samples) // 12)]:
    print("%.2fs %s" % (t - t0, r))
