"""Single-GPU cost of the fused all-gather machinery (world = 1: the GATHER
kernel variant with its end-of-grid round signal, plus the gather_wait
launch) against the plain band kernel, per launch in a CUDA graph of the
bench's block.  Peer stores over NVLink need a multi-GPU box.
    python tools/gather_overhead.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2306_03078_b200 as P  # noqa: E402

streams = bench.make_streams()
groups = []
for gname, members in bench.GROUPS:
    L = P.Layer(streams[members[0]]) if len(members) == 1 else P.Layer.stacked([streams[i] for i in members])
    x = torch.randn(L.cols, device="cuda").half()
    y = torch.empty(L.rows, device="cuda")
    g = P.Gather(0, L.rows, 1, 0)
    g.open([g.handle()], [0])
    groups.append((gname, L, x, y, g))
s = torch.cuda.Stream()


def graph_ms(fn, reps=30, inner=10):
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        fn()
    torch.cuda.synchronize()
    with torch.cuda.graph(gr, stream=s):
        for _ in range(inner):
            fn()
    with torch.cuda.stream(s):
        gr.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    with torch.cuda.stream(s):
        for _ in range(reps):
            gr.replay()
    b.record(s)
    torch.cuda.synchronize()
    return a.elapsed_time(b) / (reps * inner)


plain = graph_ms(lambda: [L.matvec(x, y, stream=s) for _, L, x, y, _ in groups])
fused = graph_ms(lambda: [(g.matvec(L, x, stream=s), g.wait(stream=s)) for _, L, x, y, g in groups])
print(f"block step: plain band kernels {1e3 * plain:.1f} us, GATHER variant + gather_wait (world 1) "
      f"{1e3 * fused:.1f} us (+{1e3 * (fused - plain) / len(groups):.2f} us per launch)", flush=True)
signal_only = graph_ms(lambda: [g.matvec(L, x, stream=s) for _, L, x, y, g in groups])
print(f"  of which the GATHER variant's end-of-grid signal alone: "
      f"+{1e3 * (signal_only - plain) / len(groups):.2f} us per launch", flush=True)
