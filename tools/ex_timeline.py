"""Where gemm_ex's time goes (tools-only -DSPQR_TIMELINE build): per role the
mean ns per launch each warp spends in its waits, 8192x22016 3-bit 1 %, exact
mode with fp32 x (the gemm_ex path; fp16 x up to 32 columns runs gemm_bm).

    python tools/ex_timeline.py [batch ...]
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_03078_b200 import build as B  # noqa: E402

extra = tuple(d for d in os.environ.get("EX_DEFINES", "").split(",") if d)
lib_path = os.path.join(ROOT, "build", "libspqr_tl%s.so" % ("_" + "_".join(extra) if extra else ""))
B.build(out=lib_path, defines=("SPQR_TIMELINE",) + extra, force=True)
os.environ["SPQR_LIB"] = lib_path
import torch  # noqa: E402

import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

P.LIB_PATH = lib_path
lib = P.lib()
lib.spqr_debug_ex_timeline.restype = C.c_int
lib.spqr_debug_ex_timeline.argtypes = [C.c_void_p, C.c_size_t]
m, n = 8192, 22016
s = synth.random_stream(m, n, 3, 3, 3, 0.01, seed=5)
L = P.Layer(s, device=0)
L.exact = True
names = {"ctrl": ["a_full", "x_full", "d_free", "-", "o_free", "-"],
         "prod": ["rec_full", "d_full", "o_full", "a_free", "-", "-"],
         "epi": ["a_full", "d_full+b_full", "outliers", "rec_full", "tmem ld", "-"]}
for Bt in map(int, sys.argv[1:] or ["16"]):
    X = torch.randn(Bt, n, device="cuda", dtype=torch.float32)
    Y = torch.empty(Bt, m, device="cuda")
    for _ in range(3):
        L.matvec(X, Y, batch=Bt)
    torch.cuda.synchronize()
    buf = np.zeros(148 * 32 * 8, np.uint64)
    assert lib.spqr_debug_ex_timeline(buf.ctypes.data, buf.size) == 0
    t = buf[: 148 * 17 * 8].reshape(148, 17, 8)[:, :9].astype(np.float64)
    print(f"batch {Bt}: stages/CTA {t[:, 0, 7].mean():.0f}, total us {t[:, :, 6].mean() / 1e3:.1f}")
    for role, ws in (("prod", range(0, 8)), ("ctrl", [8])):
        sub = t[:, list(ws), :]
        print(f"  {role}: " + ", ".join(f"{names[role][i]} {sub[:, :, i].mean() / 1e3:.1f} us"
                                         for i in range(6) if names[role][i] != "-"))
