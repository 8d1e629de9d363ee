"""Issue-slot model of each kernel in an ncu capture: executed warp instructions split into
FP64-pipe and other, predicted issue-bound time with an FP64 warp instruction holding the
dispatch for 2 cycles (measured on B200: the transform-only B1 variant ran at 99% of it),
and the shared-memory/LSU wavefront count.

    python tools/issue_model.py PROF.ncu-rep
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
meta = {}
for r in rows[2:]:
    g = lambda k: float(r[hdr.index(k)])
    meta.setdefault(r[4], []).append(dict(ms=g("gpu__time_duration.sum"), clk=g("sm__cycles_elapsed.avg.per_second"),
                                          sms=148))
FP64 = ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX")
cur, k, hdr2 = None, -1, None
counts = collections.OrderedDict()
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = r[1]
        k += 1
        counts[(k, cur)] = collections.Counter()
        continue
    if r and r[0] == "Address":
        hdr2 = r
        continue
    if not r or not r[0].startswith("0x"):
        continue
    n = int(r[hdr2.index("Instructions Executed")] or 0)
    ins = r[1].strip()
    op = (ins.split()[1] if ins.startswith("@") else ins.split()[0]).split(".")[0]
    counts[(k, cur)]["fp64" if op in FP64 else "other"] += n
    counts[(k, cur)]["shared_wf"] += int(r[hdr2.index("L1 Wavefronts Shared")] or 0)
metas = [dict(name=r[4], ms=float(r[hdr.index("gpu__time_duration.sum")]),
              clk=float(r[hdr.index("sm__cycles_elapsed.avg.per_second")]), sms=148) for r in rows[2:]]
# the source page lists each profiled launch's kernel once per (function, launch); keep one per launch
uniq = []
for (k, name), c in counts.items():
    if uniq and uniq[-1][0] == name and uniq[-1][1] == c:
        continue
    uniq.append((name, c))
for (name, c), info in zip(uniq, metas):
    short = info["name"]
    cyc = 2 * c["fp64"] + c["other"]
    per_smsp = cyc / (info["sms"] * 4)
    t_model = per_smsp / (info["clk"] * 1e6)  # clk in GHz -> ms
    print("%-32s fp64 %.3g other %.3g -> %.3f ms at 100%% issue (measured %.3f ms: %.0f%%); shared wf/SM-cycle %.2f" % (
        short, c["fp64"], c["other"], t_model, info["ms"], 100 * t_model / info["ms"],
        c["shared_wf"] / info["sms"] / (info["ms"] * 1e6 * info["clk"])))
