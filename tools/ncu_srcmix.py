"""Instructions per unit by CUDA source line (and top opcodes) from an ncu
report's mixed cuda+sass source page.
    python tools/ncu_srcmix.py REPORT UNITS [TOP]"""
import collections
import csv
import re
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
top = int(sys.argv[3]) if len(sys.argv) > 3 else 45
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
isamp = hdr.index("Warp Stall Sampling (All Samples)")
cur, fname = None, ""
agg = collections.defaultdict(collections.Counter)
samp = collections.Counter()
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) < len(hdr) or r[0] == "Line No":
        continue
    if r[0]:
        cur = f"{fname}:{r[0]} {r[1].strip()[:50]}"
    if r[2] not in ("-", "", "..."):
        op = re.sub(r"^@!?U?P\w+\s+", "", r[3].strip()).split()[0].split(".")[0]
        try:
            agg[cur][op] += int(r[ie])
            samp[cur] += int(r[isamp] or 0)
        except ValueError:
            pass
tot = sum(sum(c.values()) for c in agg.values())
print(f"total per unit {tot / units:.1f}, stall samples {sum(samp.values())}")
lst = sorted(((sum(c.values()), l, c) for l, c in agg.items()), reverse=True)[:top]
for s, l, c in lst:
    print(f"{s / units:6.1f} {samp[l]:5d} {l[:70]:70s} " + " ".join(f"{k}:{v / units:.0f}" for k, v in c.most_common(4)))
