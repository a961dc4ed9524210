"""Wait-time breakdown of gemm_tc (-DSPQR_TIMELINE build): per warp role, the
time spent in each mbarrier wait vs the kernel span.
    python tools/timeline_tc.py [B]"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_03078_b200 import build as Bd  # noqa: E402

lib_path = os.path.join(ROOT, "build", "libspqr_tl.so")
if not os.path.exists(lib_path):
    Bd.build(out=lib_path, defines=("SPQR_TIMELINE",))
os.environ["SPQR_LIB"] = lib_path
import torch  # noqa: E402

import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

P.LIB_PATH = lib_path
lib = P.lib()
lib.spqr_debug_timeline.restype = C.c_int
lib.spqr_debug_timeline.argtypes = [C.c_void_p, C.c_size_t]
B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
m, n = 8192, 22016
L = P.Layer(synth.random_stream(m, n, 3, 3, 3, 0.01, seed=1))
X = torch.randn(B, n, device="cuda", dtype=torch.float16)
Y = torch.empty(B, m, device="cuda")
for _ in range(3):
    L.matvec(X, Y, batch=B)
torch.cuda.synchronize()
buf = np.zeros(148 * 32 * 8, dtype=np.uint64)
assert lib.spqr_debug_timeline(buf.ctypes.data, buf.size) == 0
T = buf.reshape(-1, 8).astype(np.int64)
T = T[T[:, 7] == 7]
span = (T[:, 1] - T[:, 0]) / 1e3
print(f"B={B}: warps {len(T)}, span median {np.median(span):.1f} us, units/CTA {np.median(T[:, 5])}")
ctrl = T[:, 6] == T[:, 6].max()  # the control warp is the last warp (16 or 8 by HPW)
for name, sel, labels in (("control", ctrl, ("a_full", "b_full", "d_free")),
                          ("dequant", ~ctrl, ("rec_full", "a_free", "d_full"))):
    w = T[sel]
    print(f"  {name}: " + ", ".join(f"{lab} {np.median(w[:, 2 + i]) / 1e3:.1f} us" for i, lab in enumerate(labels)))
