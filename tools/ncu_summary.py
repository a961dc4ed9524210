"""Summarise an ncu report: headline metrics + per-opcode instruction mix and stalls."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
units = float(sys.argv[2]) if len(sys.argv) > 2 else 0  # cells (for per-cell counts)


def ncu(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


rows = list(csv.reader(ncu("--page", "raw", "--csv").splitlines()))
hdr, un, val = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"]
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h:70s} {val[i]:>14s} {un[i]}")
stalls = [(h, val[i]) for i, h in enumerate(hdr) if h.startswith("smsp__average_warp_latency_issue_stalled") or
          (h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"))]
st = sorted(((float(v), h) for h, v in stalls if v not in ("", "n/a")), reverse=True)[:10]
for v, h in st:
    print(f"  stall {h.replace('smsp__average_warps_issue_stalled_', ''):60s} {v:.3f}")
src = list(csv.reader(ncu("--page", "source", "--csv", "--print-source", "sass").splitlines()))
h2 = src[1]
ia = h2.index("Instructions Executed")
iss = h2.index("Warp Stall Sampling (All Samples)")
cnt, stl = collections.Counter(), collections.Counter()
for r in src[2:]:
    if len(r) <= ia or not r[ia].isdigit():
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split()[0].split(".")[0]
    cnt[op] += int(r[ia])
    stl[op] += int(r[iss]) if r[iss].isdigit() else 0
tot = sum(cnt.values())
print("total warp instructions", tot, (f"= {tot / units:.1f} per unit" if units else ""))
for op, c in cnt.most_common(24):
    print(f"  {op:10s} {c:10d} {c / units if units else 0:8.1f}  stall-samples {stl[op]}")
