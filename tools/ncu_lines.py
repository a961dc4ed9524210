"""Per-CUDA-source-line instruction counts / stall samples from an ncu report."""
import collections
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
agg = collections.defaultdict(lambda: [0, 0, ""])
fname = ""
hdr = None
cur = None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:
        cur = (fname, r[0], r[1])
    try:
        ie = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        n = int(float(r[ie] or 0))
        s = int(float(r[isamp] or 0))
    except (ValueError, IndexError):
        continue
    if cur:
        a = agg[cur[:2]]
        a[0] += n
        a[1] += s
        a[2] = cur[2]
tot = sum(v[0] for v in agg.values())
print(f"total {tot / units:.1f} per unit")
for (f, ln), (n, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:int(sys.argv[3]) if len(sys.argv) > 3 else 40]:
    print(f"{n / units:7.1f} stall {s:5d} {f}:{ln:>4s} {src.strip()[:100]}")
