"""Opcode histogram of a SASS address range: python tools/sass_hist.py FILE LO HI [--list]"""
import collections, sys
f, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
c = collections.Counter()
for l in open(f):
    a, ins = l.split(' ', 1)
    if lo <= int(a, 16) <= hi:
        op = ins.split()[1] if ins.startswith('@') else ins.split()[0]
        c[op.split('.')[0]] += 1
        if '--list' in sys.argv: print(a, ins.rstrip())
print(sum(c.values()), ' '.join('%s:%d' % kv for kv in c.most_common()))
