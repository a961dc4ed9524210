import numpy as np, torch, sys
sys.path.insert(0, '.')
import paper_2306_03078_b200 as P
from paper_2306_03078_b200 import synth
from oracle import oracle as O
np.set_printoptions(precision=4, suppress=True, linewidth=150)
for (m, n, perm, rate) in [(32, 256, False, 0.02), (32, 256, True, 0.0), (64, 512, False, 0.0), (512, 2048, False, 0.01)]:
    a = synth.make_layer(m, n, seed=1, permute=perm, outlier_rate=rate)
    s = P.encode_arrays(a)
    t = O.Oracle().decode(s)
    L = P.Layer(s)
    B = 3
    X = np.random.default_rng(0).standard_normal((B, n)).astype(np.float16)
    Y = torch.empty((B, m), device="cuda")
    L.matvec(torch.from_numpy(X).cuda(), Y, batch=B)
    got = Y.cpu().numpy()
    ref = np.stack([t.matvec(X[b].astype(np.float32)) for b in range(B)])
    bad = np.where(~np.isfinite(got[0]))[0]
    err = np.abs(got - ref).max(axis=0)
    worst = np.argsort(-np.nan_to_num(err, nan=1e9))[:6]
    print(m, n, perm, rate, "nan rows", bad[:20], "worst rows", worst, err[worst])
