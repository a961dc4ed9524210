"""ncu --csv (dram bytes per gemv_tiled launch, tools/profile_block.py) ->
profiles/gemv_traffic.json, the `traffic` figure bench.py reports."""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

csv_path, log_path, out = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(l for l in open(csv_path) if l.startswith('"'))]
hdr = rows[0]
ik, im, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
iid = hdr.index("ID")
per = {}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
for r in rows[1:]:
    if "gemv_cta" not in r[ik]:
        continue
    v = float(r[iv].replace(",", "")) * scale.get(r[iu], 1)
    per.setdefault(int(r[iid]), {})[r[im]] = v
alg = [int(m.group(1)) for m in re.finditer(r"alg_bytes (\d+)", open(log_path).read())]
launches = [per[k] for k in sorted(per)]
assert len(launches) == len(alg) == len(bench.GROUPS), (len(launches), len(alg))
items = []
shapes = re.findall(r"^(\S+) (\d+x\d+) alg_bytes", open(log_path).read(), re.M)
for (name, shape), a, d in zip(shapes, alg, launches):
    dram = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    items.append({"layer": name, "shape": shape, "alg_bytes": a, "dram_bytes": int(dram),
                  "dram_over_alg": round(dram / a, 4), "ncu_us": round(d["gpu__time_duration.sum"] / 1e3, 3)})
res = {"source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum "
                 "--clock-control none -k regex:gemv_cta (tools/profile_block.py), cold cache per launch",
       "dram_bytes_per_launch_avg": int(sum(i["dram_bytes"] for i in items) / len(items)),
       "alg_bytes_per_launch_avg": int(sum(i["alg_bytes"] for i in items) / len(items)),
       "launches": items}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
