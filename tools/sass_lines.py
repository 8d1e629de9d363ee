"""Attribute ncu per-instruction execution counts to CUDA source lines.

    python tools/sass_lines.py PROF.ncu-rep KERNEL_REGEX MANGLED_NAME [pairs]
Needs libnrng.so built with -lineinfo (it is).  Prints warp-instructions per output pair
for the hottest source lines.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, kre, mangled = sys.argv[1], sys.argv[2], sys.argv[3]
npairs = float(sys.argv[4]) if len(sys.argv) > 4 else 2.0**30
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(root, "paper_1004_3105_b200", "libnrng.so")], cwd=tmp,
               capture_output=True)
cubin = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
# walk the listing: track current function and current line info
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
        addr2line[int(m.group(1), 16)] = (line, m.group(2).split(";")[0].strip())
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows, cur, seen = [], None, 0
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "Kernel Name":
        cur = r[1]
        if re.search(kre, cur):
            seen += 1
        continue
    if cur and re.search(kre, cur) and seen == 1 and r and r[0].startswith("0x"):
        rows.append(r)
base = int(rows[0][0], 16)
per_line = collections.Counter()
ops = collections.defaultdict(collections.Counter)
for r in rows:
    off = int(r[0], 16) - base
    ln, ins = addr2line.get(off, ("?", r[1]))
    c = int(r[5])
    per_line[ln] += c
    ops[ln][ins.split()[0] if not ins.startswith("@") else ins.split()[1]] += c
tot = sum(per_line.values())
print("total %.1f warp-instr per pair" % (tot * 32 / npairs))
srcs = {}
for ln, c in per_line.most_common(40):
    f, n = ln.rsplit(":", 1) if ":" in ln else (ln, "0")
    path = os.path.join(root, "paper_1004_3105_b200", "csrc", f)
    text = ""
    if os.path.exists(path):
        lines = srcs.setdefault(path, open(path).read().splitlines())
        text = lines[int(n) - 1].strip()[:70] if int(n) - 1 < len(lines) else ""
    top = ", ".join("%s %.1f" % (o, v * 32 / npairs) for o, v in ops[ln].most_common(4))
    print("%6.1f  %-28s %-70s | %s" % (c * 32 / npairs, ln, text, top))
