#!/bin/bash
# Time METHODS for several builds of libnrng.so in one GPU session (bench shape, 2^31 normals).
# usage: bash tools/ab_multi.sh METHODS LIB1.so LIB2.so ...   ("default" = the in-tree build)
METHODS=$1; shift
for lib in "$@"; do
  if [ $lib = default ]; then unset NRNG_LIB_OVERRIDE; else export NRNG_LIB_OVERRIDE=$lib; fi
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
    best=1e9
    for rep in range(3):
        a.record()
        for _ in range(4): g.normal(m,out=out)
        b.record(); torch.cuda.synchronize(); best=min(best,a.elapsed_time(b)/4)
    res.append("%s %.3f" % (m, best))
print("%-28s" % "$lib".split('/')[-1], *res)
PY
done
