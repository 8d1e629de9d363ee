#!/bin/bash
# Interleaved A/B under sustained load, the way bench.py runs: ROUNDS x (each lib in its own
# process): 3 warm-up steps, then 10 steps of B1,B2,B3,P back to back, per-method mean.
# usage: bash tools/ab_sustained.sh ROUNDS LIB1 LIB2 ...
ROUNDS=$1; shift
for r in $(seq $ROUNDS); do
  for lib in "$@"; do
    export NRNG_LIB_OVERRIDE=$lib
    python - <<PY
import sys, torch
sys.path.insert(0, '.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W
c = W.C5_SHARD; g = P.Generator(c.seed, c.streams); out = torch.empty(c.n, dtype=torch.float64, device='cuda')
M = ["B1", "B2", "B3", "P"]
for _ in range(3):
    for m in M: g.normal(m, out=out)
ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in M] for _ in range(10)]
for s in range(10):
    for i, m in enumerate(M):
        ev[s][i][0].record(); g.normal(m, out=out); ev[s][i][1].record()
torch.cuda.synchronize()
per = [sum(ev[s][i][0].elapsed_time(ev[s][i][1]) for s in range(10)) / 10 for i in range(len(M))]
print("r$r %-14s step %.2f" % ("$lib".split('/')[-1], sum(per)), " ".join("%s %.3f" % (m, t) for m, t in zip(M, per)))
PY
  done
done
