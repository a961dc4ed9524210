"""ncu driver for the batched path: one 8192x22016 layer, batch B (default 16).
    ncu --set full -k regex:gemm_tc -s 2 -c 1 python tools/profile_tc.py [B] [--exact]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
EXACT = "--exact" in sys.argv  # exact batched mode (gemm_ex)
m, n = 8192, 22016
L = P.Layer(synth.random_stream(m, n, 3, 3, 3, 0.01, seed=1))
L.exact = EXACT
X = torch.randn(B, n, device="cuda", dtype=torch.float16)
Y = torch.empty(B, m, device="cuda")
for _ in range(4):
    L.matvec(X, Y, batch=B)
torch.cuda.synchronize()
