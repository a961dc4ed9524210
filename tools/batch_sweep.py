"""Batch sweep (BASELINE configs[3]): 8192x22016 (down_proj of LLaMA-65B),
3-bit, 1% outliers, batch 1..64.  batch 1 runs gemv_cta; batch 2-4 the
batch-pair gemv_cta (two columns per launch); batch >= 5 the tcgen05
dequant-then-MMA path (xprep_tc + gemm_tc).  Per batch: us per call
(CUDA graph over L2-defeating copies), effective GB/s on the compressed
bytes, TFLOP/s (2 m n B), and cuBLAS fp16 (torch.matmul) on the same shape.

    python tools/batch_sweep.py [--shape MxN] [--out file.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--shape", default="8192x22016")
ap.add_argument("--batches", default="1,2,4,8,16,32,64")
ap.add_argument("--out")
ap.add_argument("--exact", action="store_true", help="exact mode (spqr_layer_set_exact): gemv_cta pairs / gemm_ex")
a = ap.parse_args()
m, n = map(int, a.shape.split("x"))
s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=5)
copies = max(2, int(400e6 // len(s)) + 1)
Ls = [P.Layer(s, device=0) for _ in range(copies)]
for L_ in Ls:
    L_.exact = a.exact
st = torch.cuda.Stream()
res = {"shape": a.shape, "payload_bytes": len(s) - 48, "copies_cycled": copies,
       "path": ("exact mode: batch 1-6 gemv_cta (pairs + a single column), 7-32 xprep_bm + gemm_bm, > 32 xprep_ex + gemm_ex" if a.exact else
                "batch 1: gemv_cta; 2-4: batch-pair gemv_cta (+ one single column); >= 5: xprep_tc + gemm_tc"),
       "rows": []}


def timed(fn, reps=20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        fn()
    with torch.cuda.stream(st):
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    with torch.cuda.stream(st):
        for _ in range(reps):
            g.replay()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


W16 = torch.randn(m, n, device="cuda", dtype=torch.float16) * 0.02
for B in map(int, a.batches.split(",")):
    X = torch.randn(B, n, device="cuda", dtype=torch.float16)
    Ys = [torch.empty(B, m, device="cuda") for _ in Ls]

    def step():
        for L, Y in zip(Ls, Ys):
            L.matvec(X, Y, batch=B, stream=st)

    ms = timed(step) / len(Ls)
    Xt = X.t().contiguous()
    ms_d = timed(lambda: torch.matmul(W16, Xt))
    row = {"batch": B, "us": round(ms * 1e3, 3), "GB/s": round((len(s) - 48) / (ms * 1e-3) / 1e9, 1),
           "TFLOP/s": round(2 * m * n * B / (ms * 1e-3) / 1e12, 2), "tokens_per_s_layer": round(B / (ms * 1e-3)),
           "cublas_fp16_us": round(ms_d * 1e3, 3), "speedup_vs_cublas": round(ms_d / ms, 3)}
    res["rows"].append(row)
    print(row, flush=True)
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
