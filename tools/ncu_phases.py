"""Instructions executed per unit, grouped by source-line ranges of a kernel file.

    python tools/ncu_phases.py REPORT UNITS FILE "{'core': (286, 333), ...}"
SASS rows are attributed to the CUDA line they follow; helpers inlined from
other files are listed under their own file name.
"""
import collections
import csv
import subprocess
import sys

rep, units, target, ranges = sys.argv[1], float(sys.argv[2]), sys.argv[3], eval(sys.argv[4])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
fname, hdr, line = "", None, 0
agg = collections.Counter()
for r in csv.reader(out):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0].isdigit():
        line = int(r[0])
        continue
    if not r[2].startswith("0x"):
        continue
    n = int(float(r[hdr.index("Instructions Executed")] or 0))
    key = fname
    if fname == target:
        key = f"{target}:other"
        for name, (a, b) in ranges.items():
            if a <= line <= b:
                key = name
    agg[key] += n
tot = sum(agg.values())
print(f"total {tot / units:.1f} per unit")
for k, v in agg.most_common():
    print(f"{v / units:8.1f}  {k}")
