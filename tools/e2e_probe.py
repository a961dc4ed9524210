"""Per-call latency of the host-buffer C-ABI matvec (spqr_matvec_host) vs the
kernel alone, one 8192x8192 layer: where the e2e time goes.
    python tools/e2e_probe.py"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2306_03078_b200 as P  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

for m, n in ((8192, 8192), (8192, 22016)):
    L = P.Layer(synth.random_stream(m, n, 3, 3, 3, 0.01, seed=1))
    x = np.random.default_rng(0).standard_normal(n).astype(np.float32)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.empty(m).pin_memory()
    for _ in range(20):
        L.matvec_host(x)
    reps = 200
    t0 = time.perf_counter()
    for _ in range(reps):
        L.matvec_host(x)
    t_py = (time.perf_counter() - t0) / reps * 1e6
    t0 = time.perf_counter()
    for _ in range(reps):
        L.matvec_host(xp.numpy(), out=yp.numpy())
    t_pin = (time.perf_counter() - t0) / reps * 1e6
    y_ref = torch.empty(m)
    L.matvec_host(x, out=y_ref.numpy())
    assert np.array_equal(y_ref.numpy(), L.matvec_host(xp.numpy())), "pinned / pageable paths differ"
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty(m, device="cuda")
    s = torch.cuda.Stream()
    for _ in range(10):
        L.matvec(xd, yd, stream=s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        L.matvec(xd, yd, stream=s)
        s.synchronize()
    t_dev_sync = (time.perf_counter() - t0) / reps * 1e6
    t0 = time.perf_counter()
    for _ in range(reps):
        L.matvec(xd, yd, stream=s)
    s.synchronize()
    t_dev = (time.perf_counter() - t0) / reps * 1e6
    print(f"{m}x{n}: matvec_host pageable {t_py:.1f} us, pinned x and y {t_pin:.1f} us, "
          f"device matvec+sync {t_dev_sync:.1f} us, device matvec back-to-back {t_dev:.1f} us", flush=True)
