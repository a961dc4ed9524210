"""One batched call per batch size (for ncu launch lists of the batched kernels).
    python tools/ex_prof.py [batches] [--exact]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

m, n = 8192, 22016
s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=5)
L = P.Layer(s, device=0)
L.exact = "--exact" in sys.argv
args = [a for a in sys.argv[1:] if not a.startswith("--")]
for B in map(int, (args[0] if args else "2,16,64").split(",")):
    X = torch.randn(B, n, device="cuda", dtype=torch.float16)
    Y = torch.empty(B, m, device="cuda")
    for _ in range(2):
        L.matvec(X, Y, batch=B)
    torch.cuda.synchronize()
print("done")
