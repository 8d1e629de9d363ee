"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: one line per kernel
instantiation with its launch count and total device time (ncu: cold-cache, serialised).

    python tools/launch_list.py gpurun_out/X_launches.csv "title" > profiles/X_launches.txt
"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
title = sys.argv[2] if len(sys.argv) > 2 else sys.argv[1]
hdr, cnt, tot = None, collections.Counter(), collections.defaultdict(float)
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
        k = r[hdr.index("Kernel Name")]
        cnt[k] += 1
        tot[k] += float(r[hdr.index("Metric Value")].replace(",", "")) * scale[r[hdr.index("Metric Unit")]]
print("# %s" % title)
print("# ncu --metrics gpu__time_duration.sum launch list: launches, total device time (us), kernel")
for k in sorted(cnt, key=lambda k: (not k.startswith(("void nrng", "nrng")), k)):
    name = k if len(k) < 110 else k[:107] + "..."
    print("%5d %12.1f  %s" % (cnt[k], tot[k], name))
