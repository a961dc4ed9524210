"""fp32-x (hi/lo split, XLO) vs fp16-x gemv_cta: us per launch in a CUDA graph
of 20 launches cycling 5 layers (L2-defeating).   python tools/xlo_cost.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

s = torch.cuda.Stream()


def graph_us(fns, reps=20):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        for f in fns:
            f()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        for f in fns:
            f()
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


SHAPES = [tuple(map(int, a.split("x"))) for a in sys.argv[1:]] or [(8192, 8192), (22016, 8192), (8192, 22016)]
for m, n in SHAPES:
    Ls = [P.Layer(synth.random_stream(m, n, 3, 3, 3, 0.01, seed=300 + i)) for i in range(5)]
    x32 = torch.randn(n, device="cuda")
    x16 = x32.half()
    y = torch.empty(m, device="cuda")
    r = {}
    for name, x in (("f16", x16), ("f32", x32)):
        r[name] = graph_us([lambda L=Ls[i % 5], x=x: L.matvec(x, y, stream=s) for i in range(20)])
    print(f"{m}x{n}: f16 x {r['f16']:.2f} us, f32 x {r['f32']:.2f} us ({r['f32'] / r['f16']:.2f}x)", flush=True)
