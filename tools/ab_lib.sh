#!/bin/bash
# A/B two builds of libnrng.so in one GPU session: bash tools/ab_lib.sh ALT.so METHODS
ALT=$1; METHODS=${2:-P,P2}
for lib in default $ALT; do
  if [ $lib = default ]; then unset NRNG_LIB_OVERRIDE; else export NRNG_LIB_OVERRIDE=$lib; fi
  for rep in 1 2; do
  python - <<PY
import torch, sys
sys.path.insert(0,'.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W
c=W.C5_SHARD; g=P.Generator(c.seed,c.streams); out=torch.empty(c.n,dtype=torch.float64,device='cuda')
res=[]
for m in "$METHODS".split(','):
    for _ in range(2): g.normal(m,out=out)
    torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): g.normal(m,out=out)
    b.record(); torch.cuda.synchronize(); res.append("%s %.3f ms" % (m, a.elapsed_time(b)/5))
print("$lib".split('/')[-1], *res)
PY
  done
done
