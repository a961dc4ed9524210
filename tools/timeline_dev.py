"""Device-side timeline of one gemv_tiled launch (tools-only build with
-DSPQR_TIMELINE): per warp %globaltimer at entry, after the PDL wait, first
cell staged, loop end and exit, relative to the earliest warp entry.

    python tools/timeline_dev.py [MxN ...]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_03078_b200 import build as B  # noqa: E402

lib_path = os.path.join(ROOT, "build", "libspqr_tl.so")
if not os.path.exists(lib_path):
    B.build(out=lib_path, defines=("SPQR_TIMELINE",))
os.environ["SPQR_LIB"] = lib_path
import torch  # noqa: E402

import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

P.LIB_PATH = lib_path
lib = P.lib()
lib.spqr_debug_timeline.restype = C.c_int
lib.spqr_debug_timeline.argtypes = [C.c_void_p, C.c_size_t]
shapes = [tuple(map(int, s.split("x"))) for s in sys.argv[1:]] or [(8192, 8192), (22016, 8192)]
for m, n in shapes:
    s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=5)
    Ls = [P.Layer(s, device=0) for _ in range(4)]
    x = torch.randn(n, device="cuda").half()
    y = torch.empty(m, device="cuda")
    st = torch.cuda.Stream()
    for L in Ls:
        L.matvec(x, y, stream=st)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for L in Ls:
            L.matvec(x, y, stream=st)
    with torch.cuda.stream(st):
        for _ in range(3):
            g.replay()
    torch.cuda.synchronize()
    buf = np.zeros(148 * 32 * 8, dtype=np.uint64)
    assert lib.spqr_debug_timeline(buf.ctypes.data, buf.size) == 0
    T = buf.reshape(-1, 8).astype(np.int64)
    if True:  # gemv_cta per-warp stamps
        prod = T[(T[:, 7] == 1) & (T[:, 3] > 0)]
        t0p = T[T[:, 0] > 0][:, 0].min()
        if len(prod): print(f"== {m}x{n} producers: n={len(prod)} done at (us) " +
              " ".join(f"{v:7.2f}" for v in np.percentile((prod[:, 3] - t0p) / 1e3, [0, 50, 100])) +
              f"; empty waits/cell {prod[:, 5].mean():.1f}, wait us/producer " +
              " ".join(f"{v:6.2f}" for v in np.percentile(prod[:, 6] / 1e3, [0, 50, 100])))
        cons = T[(T[:, 7] >= 1000) & (T[:, 4] > 0)]
        # per CTA: slowest warp's loop end vs SM id and CTA index
        t0c = T[T[:, 0] > 0][:, 0].min()
        per = {}
        for i, row in enumerate(T):
            if row[7] >= 1000 and row[4] > 0:
                b = i // 16
                per.setdefault(b, [row[7] - 1000, 0])
                per[b][1] = max(per[b][1], (row[3] - t0c) / 1e3)
        items = sorted(per.items(), key=lambda kv: kv[1][1])
        print("   per-CTA last loop end (us): fastest", [(b, sm, round(t, 2)) for b, (sm, t) in items[:5]])
        print("                               slowest", [(b, sm, round(t, 2)) for b, (sm, t) in items[-8:]])
        ends = np.array([t for _, (sm, t) in items])
        ent = {}
        for i, row in enumerate(T):
            if row[7] >= 1000 and row[0] > 0:
                ent.setdefault(i // 16, []).append((row[0] - t0c) / 1e3)
        q4 = [np.mean([np.mean(ent[b]) for b in ent if lo <= b < lo + 37]) for lo in (0, 37, 74, 111)]
        e4 = [np.mean([per[b][1] for b in per if lo <= b < lo + 37]) for lo in (0, 37, 74, 111)]
        for b, (sm, tend) in items[-4:] + items[len(items) // 2:len(items) // 2 + 1]:
            rows_b = T[16 * b:16 * b + 16]
            rel = lambda k: (rows_b[:, k][rows_b[:, k] > 0] - t0c) / 1e3
            print(f"   CTA {b:3d} sm {sm:3d}: entry {rel(0).min():6.2f} pdl {rel(1).min():6.2f} first {rel(2).min():6.2f}"
                  f"..{rel(2).max():6.2f} loop_end {rel(3).min():6.2f}..{rel(3).max():6.2f} cells/warp "
                  f"{rows_b[:, 5].tolist()}")
        print("   mean CTA entry by blockIdx quarter", [round(x, 2) for x in q4], "mean loop end", [round(x, 2) for x in e4])
        print("   per-CTA end percentiles", " ".join(f"{v:6.2f}" for v in np.percentile(ends, [0, 10, 50, 90, 100])))
        print(f"   consumers: cells/warp {cons[:, 5].mean():.2f} (slot 6 = start of the last cell: tools/timeline_tail.py)")
        T[:, 5:] = 0
    t = T[:, :5]
    meta = T[:, 5:][t[:, 4] > 0]
    t = t[t[:, 4] > 0]
    t0 = t[:, 0].min()
    r = (t - t0) / 1e3  # us
    print(f"== {m}x{n}: {len(t)} warps, span {r[:, 4].max():.2f} us")
    for k, name in enumerate(["entry", "pdl_wait", "first_cell", "loop_end", "exit"]):
        q = np.percentile(r[:, k], [0, 10, 50, 90, 100])
        print(f"  {name:11s} " + " ".join(f"{v:7.2f}" for v in q))
    work = r[:, 3] - r[:, 2]
    print(f"  loop time   " + " ".join(f"{v:7.2f}" for v in np.percentile(work, [0, 10, 50, 90, 100])))
    ends = np.sort(r[:, 4])
    for f in (0.5, 0.9, 0.99):
        print(f"  {int(f * 100)}% of warps done by {ends[int(f * len(ends)) - 1]:.2f} us")
    order = np.argsort(-work)
    print("  slowest warps: loop_us cells smid outliers")
    for i in order[:8]:
        print(f"    {work[i]:6.2f} {meta[i, 0]:3d} {meta[i, 1]:4d} {meta[i, 2]:5d}")
    print("  fastest:", [(round(work[i], 2), int(meta[i, 0]), int(meta[i, 2])) for i in order[-4:]])
    for c in sorted(set(meta[:, 0].tolist())):
        sel = meta[:, 0] == c
        print(f"  cells={c}: n={sel.sum()} loop median {np.median(work[sel]):.2f} max {work[sel].max():.2f}")
    for L in Ls:
        L.close()
