"""Small driver for ncu: the batch-pair gemv_cta (x mode 2) on one LLaMA-65B layer.
    ncu --set full -k regex:gemv_cta -s 3 -c 1 -o prof python tools/profile_pair.py [m n]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
n = int(sys.argv[2]) if len(sys.argv) > 2 else 22016
L = P.Layer(synth.random_stream(m, n, 3, 3, 3, 0.01, seed=1))
x = torch.randn(2, n, device="cuda", dtype=torch.float16)
y = torch.empty(2, m, device="cuda")
for _ in range(6):
    L.matvec(x, y, batch=2)
torch.cuda.synchronize()
print("pair ok")
