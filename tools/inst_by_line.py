"""Executed warp instructions per CUDA source line (inlined call sites resolved to the innermost
line) for one kernel of an ncu capture, weighted by issue cost (FP64 = 2 cycles, other = 1).

    python tools/inst_by_line.py PROF.ncu-rep KERNEL_REGEX MANGLED_NAME [TOP]
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
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(root, "paper_1004_3105_b200", "libnrng.so")], cwd=tmp,
               capture_output=True)
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
ie, si = hdr.index("Instructions Executed"), hdr.index("Source")
base = int(rows[0][0], 16)
cost = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for r in rows:
    n = int(r[ie] or 0)
    s = r[si].strip()
    op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
    w = 2 if op in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX") else 1
    ln = addr2line.get(int(r[0], 16) - base, "?")
    cost[ln] += w * n
    ops[ln][op] += n
tot = sum(cost.values())
print("issue cycles (FP64 x2) per source line, total %.3e" % tot)
for ln, c in cost.most_common(top):
    f, n = ln.rsplit(":", 1) if ":" in ln else (ln, "0")
    path = os.path.join(root, "paper_1004_3105_b200", "csrc", f)
    text = ""
    if os.path.exists(path):
        lines = open(path).read().splitlines()
        text = lines[int(n) - 1].strip()[:58] if 0 < int(n) <= len(lines) else ""
    print("%5.1f%%  %-24s %-58s | %s" % (100 * c / tot, ln, text,
                                        " ".join("%s:%d" % kv for kv in ops[ln].most_common(4))))
