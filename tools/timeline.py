"""Per-shape timing decomposition: full matvec vs x preparation alone vs the
fused GEMV alone, each as a CUDA graph cycling enough distinct layer copies to
defeat L2.  Used to split a layer's time into a fixed part and a per-cell part.

    python tools/timeline.py [shape ...]      (shape = MxN)
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

shapes = [tuple(map(int, s.split("x"))) for s in sys.argv[1:]] or [
    (1024, 1024), (4096, 4096), (8192, 8192), (22016, 8192), (8192, 22016)]
dev = torch.device("cuda", 0)
st = torch.cuda.Stream()
out = {}
for m, n in shapes:
    s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=5)
    copies = max(2, min(24, int(400e6 // len(s)) + 1))
    Ls = [P.Layer(s, device=0) for _ in range(copies)]
    x = torch.randn(n, device=dev).half()
    ys = [torch.empty(m, device=dev) for _ in range(copies)]
    res = {"copies": copies, "payload": len(s) - 48, "cells": ((m + 31) // 32) * ((n + 255) // 256)}
    for L, y in zip(Ls, ys):
        L.matvec_stage(x, y, stage=1, stream=st)
    torch.cuda.synchronize()
    for label, stage in (("full", 0), ("xprep", 1), ("gemv", 2)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for L, y in zip(Ls, ys):
                L.matvec_stage(x, y, stage=stage, stream=st)
        with torch.cuda.stream(st):
            for _ in range(3):
                g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 30
        a.record(st)
        with torch.cuda.stream(st):
            for _ in range(reps):
                g.replay()
        b.record(st)
        torch.cuda.synchronize()
        res[label + "_us"] = round(1e3 * a.elapsed_time(b) / (reps * copies), 3)
    res["gemv_GBs"] = round((len(s) - 48) / (res["gemv_us"] * 1e-6) / 1e9, 1)
    out[f"{m}x{n}"] = res
    print(f"{m}x{n}", res, flush=True)
    for L in Ls:
        L.close()
    del Ls
print(json.dumps(out))
