"""dequantize_full on the device (spqr_dequantize): us per call and the
write-bound roofline (algorithmic bytes = cell records read + 4*m*n written)
at LLaMA-65B shapes, fast path (dequant_cells) vs the raw-stream kernels
(dequant_raw + outliers_raw, force_generic).  Timed with CUDA events over a
CUDA graph of repeated calls; the 721 MB output defeats L2.

    python tools/dequant_bench.py [--out file.json]
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
peak, kind = bench.load_peaks()
rows = []
for m, n in ((8192, 8192), (22016, 8192), (8192, 22016)):
    s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=3)
    w = torch.empty(m, n, device="cuda")
    for generic in (False, True):
        L = P.Layer(s, force_generic=generic)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            L.dequantize(w, stream=st)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(5):
                L.dequantize(w, stream=st)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 10
        e0.record(st)
        with torch.cuda.stream(st):
            for _ in range(reps):
                g.replay()
        e1.record(st)
        torch.cuda.synchronize()
        us = 1e3 * e0.elapsed_time(e1) / (5 * reps)
        alg = (len(s) - 48) + 4 * m * n
        gbs = alg / (us * 1e-6) / 1e9
        r = {"shape": f"{m}x{n}", "path": "raw stream (dequant_raw + outliers_raw)" if generic else
             "cells (dequant_cells)", "us": round(us, 2), "alg_bytes": alg, "GB/s": round(gbs, 1),
             "frac_of_peak": round(gbs / peak, 4), "device_bytes": L.info["device_bytes"],
             "payload_bytes": L.info["payload_bytes"]}
        print(r, flush=True)
        rows.append(r)
        L.close()
    del w
out = {"peak_GBs": peak, "peak_kind": kind, "rows": rows}
print(json.dumps(out))
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
