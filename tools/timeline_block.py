"""Device timeline of one launch inside the bench's block sequence (-DSPQR_TIMELINE
build): the four groups run back to back in a CUDA graph, then the sequence
up to the chosen group is replayed once more so the timeline buffer holds that
group's launch with its real predecessor.

    python tools/timeline_block.py [qkv|o|gate_up|down]
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

import bench  # noqa: E402
import paper_2306_03078_b200 as P  # noqa: E402

P.LIB_PATH = lib_path
lib = P.lib()
lib.spqr_debug_timeline.restype = C.c_int
lib.spqr_debug_timeline.argtypes = [C.c_void_p, C.c_size_t]
target = sys.argv[1] if len(sys.argv) > 1 else "o"
streams = bench.make_streams()
groups = []
for gname, members in bench.GROUPS:
    parts = [streams[i] for i in members]
    L = P.Layer(parts[0]) if len(parts) == 1 else P.Layer.stacked(parts)
    groups.append((gname, L, torch.randn(L.cols, device="cuda").half(), torch.empty(L.rows, device="cuda")))
st = torch.cuda.Stream()
upto = [g[0] for g in groups].index(target)


def run(seq):
    for gname, L, x, y in seq:
        L.matvec(x, y, stream=st)


with torch.cuda.stream(st):
    run(groups)
torch.cuda.synchronize()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g, stream=st):
    run(groups)
    run(groups[: upto + 1])
with torch.cuda.stream(st):
    for _ in range(3):
        g.replay()
torch.cuda.synchronize()
buf = np.zeros(148 * 32 * 8, dtype=np.uint64)
assert lib.spqr_debug_timeline(buf.ctypes.data, buf.size) == 0
T = buf.reshape(-1, 8).astype(np.int64)
T = T[(T[:, 4] > 0) & (T[:, 7] >= 1000)]
t0 = T[:, 0].min()
r = (T[:, :5] - t0) / 1e3
print(f"== {target} (after {groups[upto - 1][0] if upto else groups[-1][0]}): span {r[:, 4].max():.2f} us")
for k, name in enumerate(["entry", "pdl_wait", "first_cell", "loop_end", "exit"]):
    q = np.percentile(r[:, k], [0, 10, 50, 90, 100])
    print(f"  {name:11s} " + " ".join(f"{v:7.2f}" for v in q))
Tall = buf.reshape(-1, 8).astype(np.int64)
per = []
for b in range(148):
    rows_b = Tall[16 * b:16 * b + 16]
    rows_b = rows_b[(rows_b[:, 4] > 0) & (rows_b[:, 7] >= 1000)]
    if len(rows_b) == 0:
        continue
    per.append((((rows_b[:, 3].max() - t0) / 1e3), b, int(rows_b[0, 7] - 1000), (rows_b[:, 0].min() - t0) / 1e3,
                (rows_b[:, 1].min() - t0) / 1e3, (rows_b[:, 2].min() - t0) / 1e3, (rows_b[:, 3].min() - t0) / 1e3))
per.sort()
print("  CTA loop-end percentiles", " ".join(f"{v:6.2f}" for v in np.percentile([x[0] for x in per], [0, 10, 50, 90, 100])))
for x in per[-6:]:
    print(f"  slow CTA {x[1]:3d} sm {x[2]:3d}: entry {x[3]:5.2f} pdl {x[4]:5.2f} first {x[5]:5.2f} loop_end {x[6]:5.2f}..{x[0]:5.2f}")
if T[:, 5].max() > 1e12:  # panels-built stamp (SHX layers)
    q = np.percentile((T[:, 5] - t0) / 1e3, [0, 10, 50, 90, 100])
    print(f"  {'panels':11s} " + " ".join(f"{v:7.2f}" for v in q))
print(f"  full-wait us per warp (median) {np.median(T[:, 6]) / 1e3:.2f}")
