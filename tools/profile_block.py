"""ncu driver: the bench's block (bench.make_streams, bench.GROUPS: fused QKV,
o, fused gate/up, down), one launch per group, twice.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:gemv_cta -s 4 -c 4 --csv python tools/profile_block.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2306_03078_b200 as P  # noqa: E402

streams = bench.make_streams()
layers = []
for gname, members in bench.GROUPS:
    parts = [streams[i] for i in members]
    layers.append(P.Layer(parts[0]) if len(parts) == 1 else P.Layer.stacked(parts))
xs = [torch.randn(L.cols, device="cuda", dtype=torch.float16) for L in layers]
ys = [torch.empty(L.rows, device="cuda") for L in layers]
for _ in range(2):
    for L, x, y in zip(layers, xs, ys):
        L.matvec(x, y)
torch.cuda.synchronize()
for (gname, members), L in zip(bench.GROUPS, layers):
    print(f"{gname} {L.rows}x{L.cols} alg_bytes {bench.alg_bytes(L.info['payload_bytes'], L.rows, L.cols)}")
