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
    for b in (2, 3, 6):  # batch pair (x mode 2), pair + single, gemm_tc
        X = torch.randn(b, n, device="cuda", dtype=torch.float16)
        Y = torch.empty(b, m, device="cuda")
        L.matvec(X, Y, batch=b)
    L.exact = True  # exact batched mode: gemm_bm (batch 20, fp16 x) / gemm_ex (fp32 x), f16 and fp32 x
    for dt in (torch.float16, torch.float32):
        X = torch.randn(20, n, device="cuda").to(dt)
        Y = torch.empty(20, m, device="cuda")
        L.matvec(X, Y, batch=20)
    L.exact = False
    w = torch.empty(m, n, device="cuda")
    L.dequantize(w)
    L.matvec_host(np.random.default_rng(0).standard_normal(n).astype(np.float32))
    torch.cuda.synchronize()
# wide statistic groups (repeated per tile), the NCCL sharded path (world 1)
s = P.encode_arrays(synth.make_layer(128, 512, beta1=32, beta2=64, outlier_rate=0.03, seed=5))
L = P.Layer(s)
y = torch.empty(2, 128, device="cuda")
L.matvec(torch.randn(2, 512, device="cuda").half(), y, batch=2)
L.dequantize(torch.empty(128, 512, device="cuda"))
comm = P.NcclComm(P.nccl_unique_id(), 1, 0, 0)
S = P.ShardedNccl([s, s], comm, device=0)
S.matvec(torch.randn(2, 512, device="cuda").half(), torch.empty(2, 256, device="cuda"), batch=2)
torch.cuda.synchronize()
S.close()
comm.close()
print("sanitize run ok")
