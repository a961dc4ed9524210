"""One layer shape timed two ways in a CUDA graph: the same handle replayed
(weights may stay L2-resident) vs cycling 5 handles (L2-defeating).
    python tools/same_vs_cycled.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402


def graph_us(fns, reps=20):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for f in fns:
            f(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for f in fns:
            f(s)
    with torch.cuda.stream(s):
        g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            g.replay()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / reps / len(fns)


for m, n in ((8192, 8192), (8192, 22016)):
    Ls = [P.Layer(synth.random_stream(m, n, 3, 3, 3, 0.01, seed=100 + i)) for i in range(5)]
    x = torch.randn(n, device="cuda", dtype=torch.float16)
    ys = [torch.empty(m, device="cuda") for _ in range(5)]
    same = graph_us([lambda s, L=Ls[0], y=ys[0]: L.matvec(x, y, stream=s)] * 50)
    cyc = graph_us([lambda s, L=Ls[i % 5], y=ys[i % 5]: L.matvec(x, y, stream=s) for i in range(50)])
    print(f"{m}x{n}: same handle {same:.2f} us/launch, 5 handles cycled {cyc:.2f} us/launch", flush=True)
