"""Quick parity + timing probe of the exact-code batched kernel (gemm_ex)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402
from oracle import oracle as O  # noqa: E402

orc = O.Oracle()
worst = 0.0
for (m, n, bw, rate, perm) in [(128, 256, 3, 0.0, False), (128, 256, 3, 0.02, False), (96, 544, 2, 0.02, True),
                               (300, 2048, 4, 0.05, True), (256, 8192, 3, 0.01, False), (160, 1000, 3, 0.02, True)]:
    a = synth.make_layer(m, n, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=m + n, permute=perm, outlier_rate=rate)
    s = P.encode_arrays(a)
    t = orc.decode(s)
    L = P.Layer(s)
    L.exact = True
    for batch in (2, 3, 8, 16, 17, 33, 64, 70):
        for dt in (np.float16, np.float32):
            X = np.random.default_rng(batch).standard_normal((batch, n)).astype(dt)
            Y = torch.empty(batch, m, device="cuda")
            L.matvec(torch.from_numpy(X).cuda(), Y, batch=batch)
            torch.cuda.synchronize()
            got = Y.cpu().numpy()
            errs = [O.relative_l2(got[b], t.matvec(X[b].astype(np.float32))) for b in range(batch)]
            worst = max(worst, max(errs))
            flag = "" if max(errs) <= 1e-5 else "  <-- "
            print(f"m={m} n={n} bw={bw} rate={rate} perm={perm} B={batch} {dt.__name__}: max rel {max(errs):.2e}{flag}",
                  flush=True)
print("worst", worst)
