#!/bin/bash
# Interleaved A/B: ROUNDS x (each lib in its own process), best-of-3 per method after AB_WARM
# (default 25) warm-up calls of that method (the board's power controller carries state from one
# kernel to the next), with the SM clock sampled during each run.  usage: bash tools/ab_rounds.sh ROUNDS METHODS LIB1 LIB2 ...
ROUNDS=$1; METHODS=$2; shift 2
for r in $(seq $ROUNDS); do
  for lib in "$@"; do
    if [ $lib = default ]; then unset NRNG_LIB_OVERRIDE; else export NRNG_LIB_OVERRIDE=$lib; fi
    nvidia-smi --query-gpu=clocks.sm,power.draw --format=csv,noheader,nounits -lms 100 > /tmp/clk.$$ 2>/dev/null &
    SMI=$!
    python - <<PY
import torch, sys
sys.path.insert(0,'.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W
c=W.C5_SHARD; g=P.Generator(c.seed,c.streams); out=torch.empty(c.n,dtype=torch.float64,device='cuda')
res=[]
for m in "$METHODS".split(','):
    for _ in range(int('${AB_WARM:-25}')): g.normal(m,out=out)  # settle the power controller on this method
    torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    best=1e9
    for rep in range(3):
        a.record()
        for _ in range(4): g.normal(m,out=out)
        b.record(); torch.cuda.synchronize(); best=min(best,a.elapsed_time(b)/4)
    res.append("%s %.3f" % (m, best))
print("r$r %-16s" % "$lib".split('/')[-1], *res, end=" ")
PY
    kill $SMI 2>/dev/null; wait $SMI 2>/dev/null
    python -c "
import statistics
v=[l.split(',') for l in open('/tmp/clk.$$') if l.strip()]
c=[float(x[0]) for x in v]; p=[float(x[1]) for x in v]
print('| clk med %d min %d  pwr max %d' % (statistics.median(c), min(c), max(p)))"
  done
done
