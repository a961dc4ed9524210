"""Layer creation time: host transcode vs device transcode (spqr_layer_create),
for the bench's LLaMA-65B layer shapes.
    python tools/load_time.py"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

torch.cuda.init()
for m, n in ((8192, 8192), (22016, 8192), (8192, 22016)):
    s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=3)
    P.Layer(s).close()  # warm the driver
    for host in (True, False):
        t0 = time.perf_counter()
        L = P.Layer(s, host_transcode=host)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(f"{m}x{n} ({len(s) / 1e6:.1f} MB): {'host' if host else 'device'} transcode create {dt * 1e3:.1f} ms")
        L.close()
