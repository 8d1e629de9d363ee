"""Warp-stall samples per CUDA source line (and stall reason) for one kernel of an ncu capture.

    python tools/stall_by_line.py PROF.ncu-rep KERNEL_REGEX MANGLED_NAME [LIB]

LIB: the libnrng.so build that was profiled (default: the in-tree one) -- its line table maps
the capture's SASS addresses to source lines.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, mangled = sys.argv[1:4]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
lib = os.path.abspath(sys.argv[4]) if len(sys.argv) > 4 else os.path.join(root, "paper_1004_3105_b200", "libnrng.so")
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
func, line, addr2line = None, None, {}
for ln in dis.splitlines():
    m = re.match(r"\s*\.text\.(\S+):", ln)
    if m:
        func = m.group(1)
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        line = "%s:%s" % (os.path.basename(m.group(1)), m.group(2))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*)", ln)
    if m and func == mangled:
        addr2line[int(m.group(1), 16)] = line
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows, cur, seen, hdr = [], None, 0, None
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = r[1]
        if re.search(kre, cur):
            seen += 1
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if cur and re.search(kre, cur) and seen == 1 and r and r[0].startswith("0x"):
        rows.append(r)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(rows[0][0], 16)
per_line = collections.Counter()
per_reason = collections.defaultdict(collections.Counter)
tot_reason = collections.Counter()
for r in rows:
    ln = addr2line.get(int(r[0], 16) - base, "?")
    for h in reasons:
        v = int(r[hdr.index(h)] or 0)
        if h == "stall_selected":
            continue
        per_line[ln] += v
        per_reason[ln][h] += v
        tot_reason[h] += v
tot = sum(tot_reason.values())
print("stall samples (excluding 'selected'):", tot)
print("  " + ", ".join("%s %.1f%%" % (k[6:], 100 * v / tot) for k, v in tot_reason.most_common(8)))
for ln, c in per_line.most_common(25):
    f, n = ln.rsplit(":", 1) if ":" in ln else (ln, "0")
    path = os.path.join(root, "paper_1004_3105_b200", "csrc", f)
    text = ""
    if os.path.exists(path):
        lines = open(path).read().splitlines()
        text = lines[int(n) - 1].strip()[:60] if 0 < int(n) <= len(lines) else ""
    top = ", ".join("%s %d" % (k[6:], v) for k, v in per_reason[ln].most_common(3))
    print("%5.1f%%  %-26s %-60s | %s" % (100 * c / tot, ln, text, top))
