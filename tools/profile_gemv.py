"""Small driver for ncu: one LLaMA-65B layer, a few eager matvecs.

    ncu --set full -k regex:gemv_tiled -s 3 -c 1 -o prof python tools/profile_gemv.py [m n [rate [f16|f32]]]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 22016
n = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
rate = float(sys.argv[3]) if len(sys.argv) > 3 else 0.01
xdt = torch.float32 if len(sys.argv) > 4 and sys.argv[4] == "f32" else torch.float16
L = P.Layer(synth.random_stream(m, n, 3, 3, 3, rate, seed=1))
x = torch.randn(n, device="cuda", dtype=xdt)
y = torch.empty(m, device="cuda")
for _ in range(6):
    L.matvec(x, y)
torch.cuda.synchronize()
print("payload", L.info["payload_bytes"], "fast", L.info["fast_path"])
