"""Small end-to-end exercise of every kernel path, for compute-sanitizer:
    compute-sanitizer --tool memcheck python tools/sanitize_small.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

for (m, n, perm) in ((96, 544, True), (256, 2048, False)):
    s = P.encode_arrays(synth.make_layer(m, n, outlier_rate=0.03, seed=m, permute=perm))
    L = P.Layer(s)
    for dt in (torch.float16, torch.float32):
        x = torch.randn(n, device="cuda").to(dt)
        y = torch.empty(m, device="cuda")
        L.matvec(x, y)
    X = torch.randn(6, n, device="cuda", dtype=torch.float16)
    Y = torch.empty(6, m, device="cuda")
    L.matvec(X, Y, batch=6)
    w = torch.empty(m, n, device="cuda")
    L.dequantize(w)
    L.matvec_host(np.random.default_rng(0).standard_normal(n).astype(np.float32))
    torch.cuda.synchronize()
print("sanitize run ok")
