"""Share of device time per kernel in an `ncu --metrics gpu__time_duration.sum` launch list.

    python tools/launch_share.py gpurun_out/launches_TAG.csv "COMMAND" > profiles/TAG_launches_share.txt
"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
hdr = rows[0]
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
tot, cnt = collections.Counter(), collections.Counter()
for r in rows[1:]:
    if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0]
    v = float(r[vi].replace(",", ""))
    unit = r[hdr.index("Metric Unit")]
    v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}[unit]
    tot[name] += v
    cnt[name] += 1
S = sum(tot.values())
print("# share of device time per kernel in `%s` (cold-cache, serialised launches)" % (sys.argv[2] if len(sys.argv) > 2 else ""))
for k, v in tot.most_common():
    print("%-44s launches %3d  mean %10.3f us  share %5.1f%%" % (k, cnt[k], v / cnt[k], 100 * v / S))
