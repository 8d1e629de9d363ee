python tools/profile_step.py --methods P,P2 > /dev/null 2>&1
for v in direct queue; do
  if [ $v = queue ]; then export NRNG_POLAR_QUEUE=1; fi
  python - <<PY
import torch, sys
sys.path.insert(0,'.')
import paper_1004_3105_b200 as P
from paper_1004_3105_b200 import workloads as W
c=W.C5_SHARD; g=P.Generator(c.seed,c.streams); out=torch.empty(c.n,dtype=torch.float64,device='cuda')
for m in ('P','P2'):
    for _ in range(2): g.normal(m,out=out)
    torch.cuda.synchronize(); a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): g.normal(m,out=out)
    b.record(); torch.cuda.synchronize(); print("$v", m, a.elapsed_time(b)/5, 'ms')
PY
done
