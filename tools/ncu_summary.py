"""Summarise an ncu report: key metrics per kernel + dynamic SASS opcode mix per output pair.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [pairs_per_launch]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
npairs = float(sys.argv[2]) if len(sys.argv) > 2 else 2.0**30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_misc_per_issue_active.ratio"]
for d in data:
    print("----")
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print("  %-80s %s %s" % (w, d[i], units[i]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
kern, per = None, {}
for r in csv.reader(io.StringIO(src)):
    if len(r) >= 2 and r[0] == "Kernel Name":
        kern = r[1]
        per[kern] = []
        continue
    if kern and r and r[0].startswith("0x"):
        per[kern].append(r)
for k, rs in per.items():
    tot = sum(int(r[5]) for r in rs)
    ops = collections.Counter()
    for r in rs:
        parts = r[1].split()
        if not parts:
            continue
        op = parts[1] if parts[0].startswith("@") else parts[0]
        ops[op.split(".")[0]] += int(r[5])
    print(k, "warp-inst", tot, "per pair (lane)", round(tot * 32 / npairs, 1))
    print("   ", [(o, round(c * 32 / npairs, 1)) for o, c in ops.most_common(32)])
