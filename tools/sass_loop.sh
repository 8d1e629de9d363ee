#!/bin/bash
# Print the instruction count of each backward-branch loop body of one kernel (static SASS).
# usage: bash tools/sass_loop.sh MANGLED_NAME [LIB]
LIB=${2:-/root/repo/paper_1004_3105_b200/libnrng.so}
T=$(mktemp -d); cd $T; cuobjdump -xelf all $LIB > /dev/null
cuobjdump -sass -fun "$1" *.cubin | grep -E '^\s+/\*[0-9a-f]+\*/' | sed -E 's@^\s+/\*([0-9a-f]+)\*/\s+@\1 @; s@\s*/\*.*\*/\s*$@@' > k.sass
python3 - <<PY
import re
lines=[l.split(' ',1) for l in open('k.sass').read().splitlines()]
addr=[int(a,16) for a,_ in lines]
for a,ins in lines:
    m=re.search(r'BRA (0x[0-9a-f]+)',ins)
    if m and int(m.group(1),16) < int(a,16):
        t=int(m.group(1),16); n=(int(a,16)-t)//16+1
        print("loop %05x..%05x: %d instr  (%s)" % (t,int(a,16),n,ins))
PY
cp k.sass /tmp/last_kernel.sass
