"""Exact batched mode (spqr_layer_set_exact): every batch on exact-code
kernels -- gemv_cta (pairs) below batch 12, xprep_ex + gemm_ex (codes as
exact binary16 on the tcgen05 tensor cores, per-block fp32 scales, tf32 hi/lo
zero-point terms) from 7 -- against the reference's matvec (kernel.hpp:89-124)
per batch column.  The bar is the batch-1 kernel's: 1e-5 relative L2 per
column (fp32 rounding only), not the 1e-3 of fp16 weights."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2306_03078_b200 as P
from oracle import relative_l2
from paper_2306_03078_b200 import synth

pytestmark = pytest.mark.gpu

TOL = 1e-5


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _check(cuda, oracle_c, L, t, m, n, batch, dt, seed=0):
    X = np.random.default_rng(seed).standard_normal((batch, n)).astype(dt)
    Y = cuda.empty((batch, m), device="cuda")
    L.matvec(_dev(cuda, X), Y, batch=batch)
    got = Y.cpu().numpy()
    errs = [relative_l2(got[b], t.matvec(X[b].astype(np.float32))) for b in range(batch)]
    assert max(errs) <= TOL, (m, n, batch, dt.__name__, max(errs))
    return got


@pytest.mark.parametrize("bw", [2, 3, 4])
@pytest.mark.parametrize("shape,rate,perm", [((128, 256), 0.0, False), ((96, 544), 0.02, True),
                                             ((300, 2048), 0.05, True), ((256, 8192), 0.01, False)])
def test_exact_batched_vs_oracle(cuda, oracle_c, bw, shape, rate, perm):
    m, n = shape
    a = synth.make_layer(m, n, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=bw + m, permute=perm,
                         outlier_rate=rate)
    s = P.encode_arrays(a)
    L = P.Layer(s)
    L.exact = True
    t = oracle_c.decode(s)
    for batch, dt in ((2, np.float16), (5, np.float32), (7, np.float16), (12, np.float16), (17, np.float32),
                      (32, np.float16), (33, np.float16), (64, np.float32), (70, np.float16)):
        _check(cuda, oracle_c, L, t, m, n, batch, dt, seed=batch)


def test_exact_mode_paths_and_switch(cuda, oracle_c):
    """Launch plans of the two modes on one handle, switching back and forth;
    exact results equal the batch-1 kernel's column by column (batch < 7)."""
    m, n = 256, 2048
    s = synth.random_stream(m, n, seed=7)
    L = P.Layer(s)
    t = oracle_c.decode(s)
    X = cuda.randn(16, n, device="cuda", dtype=cuda.float16)
    Y = cuda.empty(16, m, device="cuda")
    L.matvec(X, Y, batch=16)
    assert P.last_launch_count() == 2  # xprep_tc + gemm_tc
    L.exact = True
    L.matvec(X, Y, batch=16)
    assert P.last_launch_count() == 2  # xprep_ex + gemm_ex
    ref = np.stack([t.matvec(X[b].float().cpu().numpy()) for b in range(16)])
    assert max(relative_l2(Y[b].cpu().numpy(), ref[b]) for b in range(16)) <= TOL
    Y4 = cuda.empty(4, m, device="cuda")
    L.matvec(X[:4].contiguous(), Y4, batch=4)
    assert P.last_launch_count() == 2  # two batch-pair gemv_cta launches
    y1 = cuda.empty(1, m, device="cuda")
    for b in range(4):
        L.matvec(X[b:b + 1].contiguous(), y1, batch=1)
        assert cuda.equal(y1[0], Y4[b])
    L.exact = False
    L.matvec(X, Y, batch=16)
    assert P.last_launch_count() == 2
    assert not L.exact


def test_exact_deterministic_and_split_tiles(cuda, oracle_c):
    """Many ranges per 128-row tile (partial slots) and dense outliers; two runs
    bitwise equal."""
    for rate in (0.0, 0.05):
        a = synth.make_layer(256, 8192, seed=9, outlier_rate=rate)
        s = P.encode_arrays(a)
        L = P.Layer(s)
        L.exact = True
        t = oracle_c.decode(s)
        y1 = _check(cuda, oracle_c, L, t, 256, 8192, 24, np.float16, seed=3)
        y2 = _check(cuda, oracle_c, L, t, 256, 8192, 24, np.float16, seed=3)
        assert np.array_equal(y1, y2)


def test_exact_host_api(cuda, oracle_c):
    """spqr_matvec_host follows the mode (its cached graph is dropped on a switch)."""
    m, n = 128, 1024
    s = synth.random_stream(m, n, seed=2)
    L = P.Layer(s)
    t = oracle_c.decode(s)
    X = np.random.default_rng(0).standard_normal((20, n)).astype(np.float32)
    ref = np.stack([t.matvec(X[b]) for b in range(20)])
    fast = L.matvec_host(X)
    L.exact = True
    ex = L.matvec_host(X)
    assert max(relative_l2(ex[b], ref[b]) for b in range(20)) <= TOL
    assert max(relative_l2(fast[b], ref[b]) for b in range(20)) <= 1e-3


@pytest.mark.slow
def test_exact_full_size_down_proj(cuda, oracle_c):
    """BASELINE configs[3] shape (8192x22016) at batch 16 in exact mode: every
    4th column against the oracle."""
    m, n = 8192, 22016
    s = synth.random_stream(m, n, seed=5)
    L = P.Layer(s)
    L.exact = True
    t = oracle_c.decode(s)
    X = np.random.default_rng(1).standard_normal((16, n)).astype(np.float16)
    Y = cuda.empty((16, m), device="cuda")
    L.matvec(_dev(cuda, X), Y, batch=16)
    got = Y.cpu().numpy()
    for b in range(0, 16, 4):
        assert relative_l2(got[b], t.matvec(X[b].astype(np.float32))) <= TOL


def test_exact_caller_workspace_and_stacked(cuda, oracle_c):
    """spqr_matvec_ws with a caller workspace sized after the switch (the exact
    plan needs more), and a stacked handle (q/k/v style) in exact mode."""
    m, n = 192, 1536
    streams = [synth.random_stream(m, n, seed=20 + i) for i in range(3)]
    L = P.Layer.stacked(streams)
    fast_bytes = L.workspace_bytes(24)
    L.exact = True
    assert L.workspace_bytes(24) >= fast_bytes
    ws = cuda.zeros(L.workspace_bytes(24), dtype=cuda.uint8, device="cuda")
    X = cuda.randn(24, n, device="cuda", dtype=cuda.float16)
    Y = cuda.empty(24, 3 * m, device="cuda")
    L.matvec(X, Y, batch=24, workspace=ws)
    got = Y.cpu().numpy()
    xs = X.float().cpu().numpy()
    for i, s in enumerate(streams):
        t = oracle_c.decode(s)
        for b in range(0, 24, 5):
            assert relative_l2(got[b, i * m:(i + 1) * m], t.matvec(xs[b])) <= TOL
