#!/bin/bash
# configs A/B: per lib, bench_configs (100-call sweep) summarised to the non-trivial configs.
# usage: bash tools/exp/cfg_ab.sh ROUNDS LIB1 LIB2 ...
ROUNDS=$1; shift
for r in $(seq $ROUNDS); do for lib in "$@"; do
NRNG_LIB_OVERRIDE=$lib timeout 300 python tools/bench_configs.py --sweep-calls 100 2>/dev/null | python -c "
import json,sys; d=json.load(sys.stdin); print('r$r %-10s' % '$lib'.split('/')[-1], ' '.join('%s %.1f' % (k.replace('_n67108864','_2^26').replace('_n4194304','_2^22'), v['us_per_call']) for k, v in d.items() if not k.startswith('C4') or k in ('C4_B1_n4194304','C4_P_n4194304','C4_B1_n67108864')))"
done; done
