"""BASELINE configs[1] and configs[4] on one GPU:
  * LLaMA-7B linear shapes (4096x4096, 11008x4096, 4096x11008), 3-bit, 1 % outliers;
  * 8192x8192 with outlier density 0..5 % (3-bit) and 3/4-bit weights at 0/1/5 %.
Per case: us per matvec (CUDA graph over L2-defeating copies, fp16 x), effective
GB/s on stream_payload_bytes + x + y, fraction of the measured HBM peak, and
cuBLAS fp16 GEMV (torch.mv) on the same shape.

    python tools/config_sweep.py [--out file.json]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out")
a = ap.parse_args()
peak, peak_kind = bench.load_peaks()
st = torch.cuda.Stream()


def timed(fn, reps=30):
    with torch.cuda.stream(st):
        fn()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
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


cases = [("llama7b", 4096, 4096, 3, 0.01), ("llama7b", 11008, 4096, 3, 0.01), ("llama7b", 4096, 11008, 3, 0.01)]
cases += [("density", 8192, 8192, 3, r) for r in (0.0, 0.005, 0.01, 0.02, 0.03, 0.04, 0.05)]
cases += [("bits", 8192, 8192, 4, r) for r in (0.0, 0.01, 0.05)]
cases = [c + ((16, 16),) for c in cases]
# wider statistic groups (PAPER Appendix D: beta2 = 32; Table 10's grid) on the
# fast kernel: GB/s on the stream's (smaller) payload
cases += [("groups", 8192, 8192, 3, 0.01, bb) for bb in ((16, 32), (32, 32), (16, 64), (64, 128), (128, 128))]
rows = []
for group, m, n, bits, rate, (b1, b2) in cases:
    s = synth.random_stream(m, n, bits, bits, bits, rate, seed=11, beta1=b1, beta2=b2)
    copies = max(2, int(400e6 // len(s)) + 1)
    Ls = [P.Layer(s, device=0) for _ in range(copies)]
    x = torch.randn(n, device="cuda").half()
    ys = [torch.empty(m, device="cuda") for _ in Ls]

    def step():
        for L, y in zip(Ls, ys):
            L.matvec(x, y, stream=st)

    us = 1e3 * timed(step) / copies
    ab = bench.alg_bytes(len(s) - 48, m, n)
    W = torch.randn(m, n, device="cuda", dtype=torch.float16)
    us_d = 1e3 * timed(lambda: torch.mv(W, x))
    row = {"group": group, "shape": f"{m}x{n}", "weight_bits": bits, "stat_bits": bits, "outlier_rate": rate,
           "beta1": b1, "beta2": b2, "fast_path": Ls[0].info["fast_path"],
           "payload_bytes": len(s) - 48, "us": round(us, 3), "GB/s": round(ab / (us * 1e-6) / 1e9, 1),
           "frac_of_peak": round(ab / (us * 1e-6) / 1e9 / peak, 4), "cublas_fp16_us": round(us_d, 3),
           "speedup_vs_cublas": round(us_d / us, 3)}
    rows.append(row)
    print(row, flush=True)
    del Ls, W
res = {"peak_GBs": peak, "peak_kind": peak_kind, "x": "fp16, batch 1", "timing": "CUDA graph, L2-defeating copies",
       "rows": rows}
print(json.dumps(res))
if a.out:
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
