"""Stall samples by (opcode, reason) and the hottest SASS instructions of an ncu report."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[1]
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
by_op = collections.defaultdict(collections.Counter)
inst = []
for r in rows[2:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[1].strip()).split()[0]
    d = {h: int(float(r[hdr.index(h)] or 0)) for h in reasons}
    for h, v in d.items():
        by_op[op.split(".")[0]][h] += v
    inst.append((sum(d.values()), r[0][-5:], r[1].strip()[:70], {k[6:]: v for k, v in d.items() if v}))
tot = collections.Counter()
for c in by_op.values():
    tot.update(c)
print("total samples by reason:", dict(tot.most_common()))
for op, c in sorted(by_op.items(), key=lambda kv: -sum(kv[1].values()))[:15]:
    print(f"{op:10s} {sum(c.values()):6d}  " + " ".join(f"{k[6:]}={v}" for k, v in c.most_common(4)))
print("--- hottest instructions")
for s, a, src, d in sorted(inst, reverse=True)[:top]:
    print(f"{s:5d} {a} {src:70s} {d}")
