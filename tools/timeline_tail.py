"""Tail anatomy of one gemv_cta launch (tools-only -DSPQR_TIMELINE build):
per warp the cell count, the start of its last cell and its loop end; per CTA
the spread of loop ends.  Four identical layers replayed in a CUDA graph (the
last launch is recorded), as in the bench.

    python tools/timeline_tail.py [MxN ...]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_03078_b200 import build as B  # noqa: E402

lib_path = os.path.join(ROOT, "build", "libspqr_tl.so")
B.build(out=lib_path, defines=("SPQR_TIMELINE",), force=not os.path.exists(lib_path))
os.environ["SPQR_LIB"] = lib_path
import torch  # noqa: E402

import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

P.LIB_PATH = lib_path
lib = P.lib()
lib.spqr_debug_timeline.restype = C.c_int
lib.spqr_debug_timeline.argtypes = [C.c_void_p, C.c_size_t]
NC = 16
shapes = [tuple(map(int, s.split("x"))) for s in sys.argv[1:]] or [(8192, 8192), (44032, 8192)]
for m, n in shapes:
    s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=5)
    Ls = [P.Layer(s, device=0) for _ in range(4)]
    x = torch.randn(n, device="cuda").half()
    y = torch.empty(m, device="cuda")
    st = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(st):
        for L in Ls:
            L.matvec(x, y, stream=st)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        for L in Ls:
            L.matvec(x, y, stream=st)
    with torch.cuda.stream(st):
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    buf = np.zeros(148 * 32 * 8, dtype=np.uint64)
    assert lib.spqr_debug_timeline(buf.ctypes.data, buf.size) == 0
    T = buf.reshape(-1, 8).astype(np.int64)[: 148 * NC]
    ok = T[:, 3] > 0
    t0 = T[ok, 1].min()  # earliest PDL release
    us = lambda v: (v - t0) / 1e3
    cells, last, end = T[ok, 5], us(T[ok, 6]), us(T[ok, 3])
    first = us(T[ok, 2])
    dur_last = end - last
    print(f"== {m}x{n}: warps {ok.sum()}, cells/warp min {cells.min()} median {np.median(cells):.0f} max {cells.max()}")
    print("   first cell start  p0/50/100 (us):", np.round(np.percentile(first, [0, 50, 100]), 2))
    print("   last cell start   p0/50/100 (us):", np.round(np.percentile(last, [0, 50, 100]), 2))
    print("   last cell length  p0/50/100 (us):", np.round(np.percentile(dur_last, [0, 50, 100]), 2))
    print("   loop end          p0/50/100 (us):", np.round(np.percentile(end, [0, 10, 50, 90, 100]), 2))
    mean_cell = (end - first) / np.maximum(cells, 1)
    print("   mean cell time per warp p50 (us):", round(float(np.median(mean_cell)), 3))
    ctas = np.arange(148 * NC)[ok] // NC
    spread = [end[ctas == c].max() - end[ctas == c].min() for c in np.unique(ctas)]
    cend = [end[ctas == c].max() for c in np.unique(ctas)]
    print("   per-CTA loop-end spread p50/max (us):", round(float(np.median(spread)), 2), round(float(max(spread)), 2))
    print("   per-CTA last end p0/50/100 (us):", np.round(np.percentile(cend, [0, 50, 100]), 2))
    # busy warps over time (SM utilisation proxy) in the tail
    grid = np.linspace(np.percentile(end, 1), end.max(), 8)
    print("   active warps after t:", [(round(float(t), 1), int((end > t).sum())) for t in grid])
    for L in Ls:
        L.close()
