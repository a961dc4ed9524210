"""Fixed cost of one spqr_matvec_host call (tiny layer: the kernel is ~3 us):
pageable vs page-locked buffers, and a bare CUDA-graph launch + sync for
comparison.    python tools/host_call_overhead.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

L = P.Layer(synth.random_stream(256, 512, 3, 3, 3, 0.01, seed=1))
x = np.random.default_rng(0).standard_normal(512).astype(np.float32)
xp, yp = torch.from_numpy(x).pin_memory(), torch.empty(256).pin_memory()


def t(fn, reps=2000):
    for _ in range(50):
        fn()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    return (time.perf_counter() - t0) / reps * 1e6


print(f"matvec_host pageable: {t(lambda: L.matvec_host(x)):.1f} us")
print(f"matvec_host pinned  : {t(lambda: L.matvec_host(xp.numpy(), out=yp.numpy())):.1f} us")
s = torch.cuda.Stream()
xd, yd = torch.from_numpy(x).cuda(), torch.empty(256, device="cuda")
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    L.matvec(xd, yd, stream=s)
torch.cuda.synchronize()
with torch.cuda.graph(g, stream=s):
    L.matvec(xd, yd, stream=s)


def replay_sync(gr):
    with torch.cuda.stream(s):  # replay on s: the graph runs where s.synchronize() waits
        gr.replay()
    s.synchronize()


print(f"graph(matvec) replay + sync: {t(lambda: replay_sync(g)):.1f} us")
e = torch.cuda.CUDAGraph()
with torch.cuda.graph(e, stream=s):
    yd.add_(0)
print(f"graph(one tiny torch kernel) replay + sync: {t(lambda: replay_sync(e)):.1f} us")

# where the host-buffer call's GPU time goes (tiny layer)
def gtime(fn):
    gg = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(gg, stream=s):
        fn()
    return t(lambda: replay_sync(gg))


print(f"graph(matvec -> device y): {gtime(lambda: L.matvec(xd, yd, stream=s)):.1f} us")
print(f"graph(matvec -> pinned host y): {gtime(lambda: L.matvec(xd, yp, stream=s)):.1f} us")
print(f"graph(matvec, x from pinned host): {gtime(lambda: L.matvec(xp, yd, stream=s)):.1f} us")
print(f"graph(H2D copy_ of x, matvec): {gtime(lambda: (xd.copy_(xp, non_blocking=True), L.matvec(xd, yd, stream=s))):.1f} us")

# big layer: the host-buffer call vs the same kernel on device buffers
Lb = P.Layer(synth.random_stream(8192, 8192, 3, 3, 3, 0.01, seed=2))
xb = torch.randn(8192)
xbp, xbd = xb.pin_memory(), xb.cuda()
ybd, ybp = torch.empty(8192, device="cuda"), torch.empty(8192).pin_memory()
print(f"8192x8192 graph(matvec, device x, device y) + sync: {gtime(lambda: Lb.matvec(xbd, ybd, stream=s)):.1f} us")
print(f"8192x8192 graph(H2D copy_, matvec, host y) + sync: "
      f"{gtime(lambda: (xbd.copy_(xbp, non_blocking=True), Lb.matvec(xbd, ybp, stream=s))):.1f} us")
print(f"8192x8192 matvec_host pinned: {t(lambda: Lb.matvec_host(xbp.numpy(), out=ybp.numpy()), 500):.1f} us")
