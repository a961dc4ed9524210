"""The GPU encoder (Hessian + inverse Cholesky + block-GPTQ with the outlier
screen + bilevel fit + encode) timed against the reference encoder on the host
(oracle/_ref/libspqr_ref_enc.so, 1 thread, our minimal Eigen).  Streams are
compared byte for byte where the reference runs.

    python tools/encoder_bench.py [--out file.json]
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle as O  # noqa: E402
import paper_2306_03078_b200 as P  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--out")
a = ap.parse_args()
E = O.ReferenceEncoder() if os.path.exists(O.REF_ENC_SO) else None
rows = []
for m, n, samples, with_ref in ((512, 512, 1024, True), (1024, 1024, 2048, True), (4096, 4096, 4096, False),
                                (8192, 8192, 4096, False), (22016, 8192, 4096, False)):
    rng = np.random.default_rng(m + n)
    W = (rng.standard_normal((m, n)) * 0.02).astype(np.float32)
    X = rng.standard_normal((n, samples)).astype(np.float32)
    Wd, Xd = torch.from_numpy(W).cuda(), torch.from_numpy(X).cuda()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    H = P.Hessian(n, device=0)
    H.accumulate(Xd)
    t1 = time.perf_counter()
    tau = 0.2 * samples / 1024  # the screen's error sums scale with the Hessian (~2 x samples): ~1 % outliers
    s, rep = H.quantize(Wd, tau=tau)
    t2 = time.perf_counter()
    row = {"shape": f"{m}x{n}", "samples": samples, "tau": tau, "gpu_hessian_s": round(t1 - t0, 4),
           "gpu_quantize_s": round(t2 - t1, 4), "relative_error": rep["relative_error"],
           "outlier_rate": rep["outlier_rate"], "bits_per_param": rep["bits_per_param"]}
    if with_ref and E is not None:
        t3 = time.perf_counter()
        s_ref, _ = E.quantize(W, X, tau=tau)
        row["reference_cpu_s"] = round(time.perf_counter() - t3, 3)
        row["identical_stream"] = s_ref == s
    print(row, flush=True)
    rows.append(row)
    H.close()
out = {"config": "3/3/3 bits, beta 16x16, tau 0.2 x samples/1024, lambda_rel 0.01, natural order; synthetic W ~ N(0, 0.02^2), X ~ N(0, 1)",
       "rows": rows}
print(json.dumps(out))
if a.out:
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
