"""ncu driver: the bench's seven LLaMA-65B layers (bench.make_streams), x
prepared once (stage 1), then the fused kernel (stage 2) once per layer, twice.

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        -k regex:gemv_cta -s 7 -c 7 --csv python tools/profile_block.py
"""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2306_03078_b200 as P  # noqa: E402

layers = [P.Layer(s) for s in bench.make_streams()]
xs = [torch.randn(L.cols, device="cuda", dtype=torch.float16) for L in layers]
ys = [torch.empty(L.rows, device="cuda") for L in layers]
for L, x, y in zip(layers, xs, ys):
    L.matvec_stage(x, y, stage=1)
for _ in range(2):
    for L, x, y in zip(layers, xs, ys):
        L.matvec_stage(x, y, stage=2)
torch.cuda.synchronize()
for (name, m, n), L in zip(bench.LAYERS, layers):
    print(f"{name} {m}x{n} alg_bytes {bench.alg_bytes(L.info['payload_bytes'], m, n)}")
