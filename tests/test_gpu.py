"""Parity of the CUDA path (through the C ABI) against the oracle.

* dequantize_full: bit-exact (uint32 patterns) against the reference's golden
  output and the oracle, every geometry.
* matvec: relative L2 (kernel.hpp:154-163) <= 1e-3 against the reference
  (north star); the measured error is ~1e-7, so the test also pins 1e-5 for
  fp32 x on the tiled path (hi/lo split) and fp16-exact x.
"""
from __future__ import annotations

import numpy as np
import pytest

import paper_2306_03078_b200 as P
from oracle import relative_l2
from paper_2306_03078_b200 import synth

pytestmark = pytest.mark.gpu

TOL = 1e-3  # north star: matvec within 1e-3 relative (fp32 accumulation)


def _dev(torch, a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def test_library_reports_fast_kernel_launches(cuda):
    s = synth.random_stream(64, 512, seed=0)
    L = P.Layer(s)
    assert L.info["fast_path"] == 1
    x = cuda.randn(512, device="cuda", dtype=cuda.float16)
    y = cuda.empty(64, device="cuda")
    L.matvec(x, y)
    cuda.cuda.synchronize()
    assert P.last_launch_count() == 1  # one fused launch (x preparation inside)


def test_dequantize_bit_exact_golden(cuda, golden, golden_cases):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        for generic in (False, True):
            L = P.Layer(s, force_generic=generic)
            w = cuda.empty((L.rows, L.cols), device="cuda", dtype=cuda.float32)
            L.dequantize(w)
            got = w.cpu().numpy().view(np.uint32)
            assert np.array_equal(got, golden[f"{name}/w_bits"]), (name, generic)


def test_matvec_golden_all_paths(cuda, golden, golden_cases):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        for generic in (False, True):
            L = P.Layer(s, force_generic=generic)
            for x, yref in zip(golden[f"{name}/x"], golden[f"{name}/y"]):
                for dt in (cuda.float32, cuda.float16):  # golden x values are fp16-exact
                    xd = _dev(cuda, x).to(dt)
                    y = cuda.empty(L.rows, device="cuda")
                    L.matvec(xd, y)
                    err = relative_l2(y.cpu().numpy(), yref)
                    assert err <= 1e-5, (name, generic, dt, err)


def test_x_zero_and_unit_vectors(cuda, oracle_c):
    a = synth.make_layer(96, 512, seed=11, permute=True, outlier_rate=0.02)
    s = P.encode_arrays(a)
    L = P.Layer(s)
    w = oracle_c.decode(s).dequantize_full()
    y = cuda.empty(96, device="cuda")
    L.matvec(cuda.zeros(512, device="cuda"), y)
    assert float(y.abs().max()) == 0.0
    for j in (0, 7, 255, 256, 511):
        x = cuda.zeros(512, device="cuda")
        x[j] = 1.0
        L.matvec(x, y)
        assert relative_l2(y.cpu().numpy(), w[:, j]) < 1e-6, j


@pytest.mark.parametrize("bw", [2, 3, 4])
@pytest.mark.parametrize("shape", [(32, 256), (50, 300), (160, 1000), (256, 4096)])
def test_matvec_fast_vs_oracle(cuda, oracle_c, bw, shape):
    a = synth.make_layer(*shape, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=bw, permute=True,
                         outlier_rate=0.03)
    s = P.encode_arrays(a)
    L = P.Layer(s)
    assert L.info["fast_path"] == 1
    t = oracle_c.decode(s)
    rng = np.random.default_rng(7)
    for dt in (np.float32, np.float16):
        x = rng.standard_normal(shape[1]).astype(dt)
        y = cuda.empty(shape[0], device="cuda")
        L.matvec(_dev(cuda, x), y)
        ref = t.matvec(x.astype(np.float32))
        assert relative_l2(y.cpu().numpy(), ref) < 1e-5


def test_f32_x_exponent_extremes(cuda, oracle_c):
    """fp32 x far from 1 (block exponents where 2^k is not a normal float, and
    fp32 subnormals): the panel scaling falls back to ldexpf/frexpf."""
    a = synth.make_layer(96, 1024, seed=11, outlier_rate=0.02)
    s = P.encode_arrays(a)
    L = P.Layer(s)
    t = oracle_c.decode(s)
    rng = np.random.default_rng(9)
    for scale in (1e-38, 1e-30, 1e25):
        x = (rng.standard_normal(1024) * scale).astype(np.float32)
        y = cuda.empty(96, device="cuda")
        L.matvec(_dev(cuda, x), y)
        ref = t.matvec(x)
        assert relative_l2(y.cpu().numpy(), ref) < 1e-5, scale


def test_outlier_density_sweep(cuda, oracle_c):
    for rate in (0.0, 0.005, 0.01, 0.02, 0.05):
        a = synth.make_layer(256, 2048, seed=3, outlier_rate=rate)
        s = P.encode_arrays(a)
        L = P.Layer(s)
        x = np.random.default_rng(1).standard_normal(2048).astype(np.float16)
        y = cuda.empty(256, device="cuda")
        L.matvec(_dev(cuda, x), y)
        assert relative_l2(y.cpu().numpy(), oracle_c.decode(s).matvec(x.astype(np.float32))) < 1e-5, rate


def test_clustered_outliers_overflow_smem_cap(cuda, oracle_c):
    """A cell with more outliers than the TMA slot holds (2048 B) takes the
    global-memory tail path."""
    m, n = 64, 512
    a = synth.make_layer(m, n, seed=2, outlier_rate=0.0)
    rows = np.repeat(np.arange(32, dtype=np.uint32), 50)  # 1600 entries in rows 0..31
    cols = np.tile(np.arange(0, 250, 5, dtype=np.uint32), 32)
    a["outlier_rows"], a["outlier_cols"] = rows, cols
    a["outlier_vals"] = (np.random.default_rng(0).standard_normal(rows.size) * 0.1).astype(np.float16).view(np.uint16)
    s = P.encode_arrays(a)
    L = P.Layer(s)
    x = np.random.default_rng(3).standard_normal(n).astype(np.float32)
    y = cuda.empty(m, device="cuda")
    L.matvec(_dev(cuda, x), y)
    assert relative_l2(y.cpu().numpy(), oracle_c.decode(s).matvec(x)) < 1e-5


def test_batch_and_host_api(cuda, oracle_c):
    a = synth.make_layer(128, 768, seed=5, permute=True)
    s = P.encode_arrays(a)
    t = oracle_c.decode(s)
    for generic in (False, True):
        L = P.Layer(s, force_generic=generic)
        X = np.random.default_rng(2).standard_normal((3, 768)).astype(np.float32)
        Y = cuda.empty((3, 128), device="cuda")
        L.matvec(_dev(cuda, X), Y, batch=3)
        Yh = L.matvec_host(X)
        # batch >= 2 on the fast path is the tcgen05 dequant-then-MMA kernel
        # (fp16 weights: the north star's 1e-3); the generic path stays fp32
        tol = 1e-5 if generic else TOL
        for b in range(3):
            ref = t.matvec(X[b])
            assert relative_l2(Y[b].cpu().numpy(), ref) < tol
            assert relative_l2(Yh[b], ref) < tol


def test_host_api_graph_reuse(cuda, oracle_c):
    """spqr_matvec_host replays one captured [H2D, kernels, D2H] graph: new x
    every call, pageable and page-locked buffers, batch changes re-capture."""
    s = synth.random_stream(512, 1024, seed=7)
    t = oracle_c.decode(s)
    L = P.Layer(s)
    rng = np.random.default_rng(4)
    xp = cuda.empty(1024, dtype=cuda.float32).pin_memory()
    yp = cuda.empty(512, dtype=cuda.float32).pin_memory()
    for i in range(6):
        x = rng.standard_normal(1024).astype(np.float32)
        ref = t.matvec(x)
        if i % 2:
            xp.numpy()[:] = x
            y = L.matvec_host(xp.numpy(), out=yp.numpy()).copy()
        else:
            y = L.matvec_host(x)
        assert relative_l2(y, ref) < 1e-5, i
        assert P.last_launch_count() >= 1
    X = rng.standard_normal((2, 1024)).astype(np.float32)  # batch 2: a new graph
    Y = L.matvec_host(X)
    for b in range(2):
        assert relative_l2(Y[b], t.matvec(X[b])) < 1e-5
    X = rng.standard_normal((6, 1024)).astype(np.float32)  # batch 6: gemm_tc stores y to host memory
    Y = L.matvec_host(X)
    for b in range(6):
        assert relative_l2(Y[b], t.matvec(X[b])) < TOL
    x = rng.standard_normal(1024).astype(np.float32)  # back to batch 1
    assert relative_l2(L.matvec_host(x), t.matvec(x)) < 1e-5


def test_host_call_bound_buffers(cuda, oracle_c):
    """Layer.host_call binds matvec_host to one page-locked x / y pair: x is
    re-read and y rewritten every call; wrong buffers are refused up front."""
    s = synth.random_stream(512, 1024, seed=8)
    t = oracle_c.decode(s)
    L = P.Layer(s)
    xp = cuda.empty(1024, dtype=cuda.float32).pin_memory()
    yp = cuda.empty(512, dtype=cuda.float32).pin_memory()
    call = L.host_call(xp.numpy(), yp.numpy())
    rng = np.random.default_rng(9)
    for i in range(4):
        x = rng.standard_normal(1024).astype(np.float32)
        xp.numpy()[:] = x
        call()
        assert relative_l2(yp.numpy(), t.matvec(x)) < 1e-5, i
    with pytest.raises(ValueError):
        L.host_call(np.zeros(1024, np.float64), yp.numpy())
    with pytest.raises(ValueError):
        L.host_call(xp.numpy(), np.zeros(511, np.float32))


def test_deterministic_and_workspace(cuda):
    s = synth.random_stream(1024, 4096, seed=3)
    L = P.Layer(s)
    x = cuda.randn(4096, device="cuda", dtype=cuda.float16)
    y1 = cuda.empty(1024, device="cuda")
    y2 = cuda.empty(1024, device="cuda")
    L.matvec(x, y1)
    ws = cuda.zeros(L.workspace_bytes(1), dtype=cuda.uint8, device="cuda")
    st = cuda.cuda.Stream()
    with cuda.cuda.stream(st):
        L.matvec(x, y2, stream=st, workspace=ws)
    st.synchronize()
    assert cuda.equal(y1, y2)
    for _ in range(3):
        L.matvec(x, y2)
        assert cuda.equal(y1, y2)


def test_device_roundtrip_export(cuda, golden, golden_cases):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        assert P.Layer(s).export_stream() == s, name
    s = synth.random_stream(512, 2048, seed=9, permute=True)
    assert P.Layer(s).export_stream() == s


def test_row_band_layers_concatenate(cuda):
    s = synth.random_stream(512, 1024, seed=4)
    x = cuda.randn(1024, device="cuda", dtype=cuda.float16)
    full = P.Layer(s)
    y = cuda.empty(512, device="cuda")
    full.matvec(x, y)
    parts = []
    for r0 in range(0, 512, 128):
        band = P.Layer(s, rows=(r0, r0 + 128))
        yb = cuda.empty(128, device="cuda")
        band.matvec(x, yb)
        parts.append(yb)
    assert relative_l2(cuda.cat(parts).cpu().numpy(), y.cpu().numpy()) < 1e-6


@pytest.mark.slow
@pytest.mark.parametrize("shape", [(4096, 4096), (11008, 4096), (4096, 11008)])
def test_llama7b_shapes_vs_oracle(cuda, oracle_c, shape):
    s = synth.random_stream(*shape, seed=1)
    L = P.Layer(s)
    t = oracle_c.decode(s)
    x = np.random.default_rng(2).standard_normal(shape[1]).astype(np.float16)
    y = cuda.empty(shape[0], device="cuda")
    L.matvec(_dev(cuda, x), y)
    assert relative_l2(y.cpu().numpy(), t.matvec(x.astype(np.float32))) < TOL
    w = cuda.empty(shape, device="cuda")
    L.dequantize(w)
    assert np.array_equal(w.cpu().numpy().view(np.uint32), t.dequantize_full().view(np.uint32))
    # HBM footprint: the cell records (~ the payload) + offsets + workspace -- no raw stream copy
    assert L.info["device_bytes"] < 1.02 * len(s) + L.workspace_bytes() + 4 * (shape[0] // 32 + 1) * (shape[1] // 256 + 1)


@pytest.mark.slow
@pytest.mark.parametrize("shape", [(8192, 8192), (22016, 8192), (8192, 22016)])
def test_llama65b_shapes_vs_oracle(cuda, oracle_c, shape):
    """BASELINE configs[2]/[3] at full size: the fast kernel (f16 and f32 x)
    against the oracle, plus the size-independent properties -- linearity in x
    and run-to-run bit equality."""
    s = synth.random_stream(*shape, seed=3)
    L = P.Layer(s)
    t = oracle_c.decode(s)
    rng = np.random.default_rng(5)
    x1 = rng.standard_normal(shape[1]).astype(np.float32)
    x2 = rng.standard_normal(shape[1]).astype(np.float32)
    y = cuda.empty(shape[0], device="cuda")
    L.matvec(_dev(cuda, x1), y)
    y1 = y.cpu().numpy()
    assert relative_l2(y1, t.matvec(x1)) < 1e-5  # fp32 x: hi/lo split, fp32 accumulation
    xh = x1.astype(np.float16)
    L.matvec(_dev(cuda, xh), y)
    assert relative_l2(y.cpu().numpy(), t.matvec(xh.astype(np.float32))) < TOL
    L.matvec(_dev(cuda, x2), y)
    y2 = y.cpu().numpy()
    L.matvec(_dev(cuda, x1 + x2), y)
    assert relative_l2(y.cpu().numpy(), y1 + y2) < 1e-5  # linearity
    L.matvec(_dev(cuda, x1), y)
    assert np.array_equal(y.cpu().numpy().view(np.uint32), y1.view(np.uint32))  # deterministic


def test_dense_gemv_f16(cuda):
    W = cuda.randn(300, 1024, device="cuda", dtype=cuda.float16)
    x = cuda.randn(1024, device="cuda", dtype=cuda.float16)
    y = cuda.empty(300, device="cuda")
    P.dense_gemv_f16(W, x, y, 300, 1024)
    ref = (W.float() @ x.float())
    assert float((y - ref).norm() / ref.norm()) < 1e-5


def test_errors_surface(cuda):
    s = synth.random_stream(32, 256, seed=0)
    L = P.Layer(s)
    with pytest.raises(P.SpqrError) as ei:
        L.matvec(cuda.zeros(256, device="cuda"), cuda.empty(32, device="cuda"), batch=0)
    assert ei.value.errc == "shape_mismatch"
    with pytest.raises(P.SpqrError) as ei:
        P.Layer(s[:-3])
    assert ei.value.errc == "malformed_stream"


def test_stacked_layers_match_separate(cuda, oracle_c):
    """spqr_layer_create_stacked: q/k/v-style layers sharing x in one handle;
    y is the row-wise concatenation of the separate products."""
    streams = [P.encode_arrays(synth.make_layer(m, 768, seed=20 + i, outlier_rate=0.02)) for i, m in
               enumerate((96, 64, 50))]
    L = P.Layer.stacked(streams)
    assert L.rows == 96 + 64 + 50 and L.info["fast_path"] == 1
    refs = [oracle_c.decode(s) for s in streams]
    rng = np.random.default_rng(4)
    for batch, dt, tol in ((1, np.float16, 1e-5), (1, np.float32, 1e-5), (8, np.float16, TOL)):
        X = rng.standard_normal((batch, 768)).astype(dt)
        Y = cuda.empty((batch, L.rows), device="cuda")
        L.matvec(_dev(cuda, X), Y, batch=batch)
        got = Y.cpu().numpy()
        for b in range(batch):
            ref = np.concatenate([t.matvec(X[b].astype(np.float32)) for t in refs])
            assert relative_l2(got[b], ref) < tol, (batch, dt)
    with pytest.raises(P.SpqrError):
        L.dequantize(cuda.empty((L.rows, 768), device="cuda"))
    bad = P.encode_arrays(synth.make_layer(64, 512, seed=1))
    with pytest.raises(P.SpqrError):
        P.Layer.stacked([streams[0], bad])


@pytest.mark.parametrize("case", [(96, 544, 3, 0.02, True), (50, 300, 2, 0.05, False), (160, 1000, 4, 0.03, True),
                                  (256, 4096, 3, 0.01, False)])
def test_device_transcode_matches_host(cuda, case):
    """The GPU loader (transcode_dev.cuh) writes byte-identical cell records
    and offsets to the host transcode (transcode.cpp), single and stacked."""
    m, n, bw, rate, perm = case
    a = synth.make_layer(m, n, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=m, permute=perm, outlier_rate=rate)
    s = P.encode_arrays(a)
    host = P.debug_tiled_host(s)
    dev = P.Layer(s).debug_cells()
    assert np.array_equal(dev["cell_off"], host["cell_off"])
    assert np.array_equal(dev["cells"], host["cells"][: dev["cells"].size])
    if m % 32 == 0:
        dh = P.Layer.stacked([s, s], host_transcode=True).debug_cells()
        dd = P.Layer.stacked([s, s]).debug_cells()
        assert np.array_equal(dh["cell_off"], dd["cell_off"]) and np.array_equal(dh["cells"], dd["cells"])


@pytest.mark.parametrize("world", [2, 3])
def test_fused_gather_matches_band_kernels(world):
    """Fused all-gather epilogue (spqr_matvec_gather + spqr_gather_wait): ranks
    sharing cuda:0 over CUDA IPC; full y on every rank, eager and graph-replayed."""
    import os
    import socket
    import subprocess
    import sys

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    here = os.path.dirname(os.path.abspath(__file__))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes", "1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(here, "dist", "fused_gather_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "fused gather ok" in r.stdout


@pytest.mark.parametrize("bw,bs", [(2, 2), (2, 4), (3, 2), (3, 3), (3, 4), (4, 3), (4, 4)])
@pytest.mark.parametrize("shape,perm", [((32, 256), False), ((50, 300), True), ((160, 1000), False),
                                        ((96, 4096), True)])
def test_dequantize_cells_bit_exact(cuda, oracle_c, bw, bs, shape, perm):
    """dequantize_full from the tiled cell records (dequant_cells, one launch)
    == the oracle bit for bit, every fast-path width, ragged shapes, permuted
    columns, 2 % outliers; the fast-path handle holds no raw stream copy."""
    s = P.encode_arrays(synth.make_layer(*shape, weight_bits=bw, scale_bits=bs, zero_bits=bs, outlier_rate=0.02,
                                         seed=bw * 7 + bs + shape[0], permute=perm))
    L = P.Layer(s)
    assert L.info["fast_path"] == 1
    w = cuda.full(shape, float("nan"), device="cuda")
    L.dequantize(w)
    cuda.cuda.synchronize()
    assert P.last_launch_count() == 1
    ref = oracle_c.decode(s).dequantize_full()
    assert np.array_equal(w.cpu().numpy().view(np.uint32), ref.view(np.uint32))
