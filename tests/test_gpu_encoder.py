"""The GPU encoder (spqr_hessian_*, spqr_quantize_layer)
against the UNMODIFIED reference encoder (oracle/ref_encoder.cpp: the
reference's HessianAccumulator, finalize, spqr_quantize, make_spqr_tensor and
encode, built with our functional minimal Eigen).  Same W and calibration X:
the .spqr streams must be identical byte for byte (codes, statistics,
outliers, permutation, header), and the reports (relative layer error,
outlier rate, bits per parameter) agree.  Both run the reference's algorithm
in binary64; the GPU sums its products in a different order (cuBLAS,
cuSOLVER), which can only move a decision sitting within ~1e-12 of a
rounding boundary."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest
import torch

import paper_2306_03078_b200 as P

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))


@pytest.fixture(scope="module")
def ref_encoder():
    import oracle as O

    if not os.path.exists(O.REF_ENC_SO):
        pytest.skip("oracle/_ref/libspqr_ref_enc.so not built")
    return O.ReferenceEncoder()


def _layer(m, n, samples, seed, outlier_cols=0):
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((m, n)) * 0.02).astype(np.float32)
    if outlier_cols:  # a few heavy weights the screen should keep in 16 bits
        idx = rng.integers(0, m * n, size=m * n // 200)
        W.reshape(-1)[idx] *= 8.0
    X = rng.standard_normal((n, samples)).astype(np.float32)
    X[: n // 8] *= 3.0  # uneven activation scales: a non-trivial Hessian
    return W, X


CASES = [
    dict(),
    dict(weight_bits=2, scale_bits=2, zero_bits=2),  # > 5 % outliers: both refuse (outlier_budget_exceeded)
    dict(weight_bits=2, scale_bits=2, zero_bits=2, tau=1.0),
    dict(weight_bits=4, scale_bits=4, zero_bits=4, tau=0.05),
    dict(beta1=32, beta2=32),
    dict(beta2=64, order="act_order"),
    dict(order="act_order", act_order_key="inverse_diag"),
    dict(order="shuffled", seed=7),
    dict(integer_zero=True, weight_bits=3, zero_bits=3),
    dict(full_range_sign=False),
    dict(scale_bits=16, zero_bits=16),
    dict(outliers=False),
    dict(tau=0.5, lambda_rel=0.1),
]


@pytest.mark.parametrize("cfg", CASES, ids=[",".join(f"{k}={v}" for k, v in c.items()) or "default" for c in CASES])
def test_gpu_encoder_matches_reference(cuda, ref_encoder, cfg):
    m, n, samples = 96, 256, 384
    W, X = _layer(m, n, samples, seed=len(str(cfg)), outlier_cols=1)
    H = P.Hessian(n, device=0)
    H.accumulate(torch.from_numpy(X).cuda())
    try:
        s_ref, rep_ref = ref_encoder.quantize(W, X, **cfg)
    except Exception as ex:  # the reference refuses: the GPU encoder must refuse the same way
        with pytest.raises(P.SpqrError) as ei:
            H.quantize(torch.from_numpy(W).cuda(), **cfg)
        assert ei.value.errc == ex.errc
        return
    s_gpu, rep_gpu = H.quantize(torch.from_numpy(W).cuda(), **cfg)
    assert P.validate(s_gpu)["rows"] == m
    assert s_gpu == s_ref
    assert rep_gpu["outlier_rate"] == rep_ref["outlier_rate"]
    assert rep_gpu["bits_per_param"] == rep_ref["bits_per_param"]
    assert abs(rep_gpu["relative_error"] - rep_ref["relative_error"]) <= 1e-9 * max(1.0, rep_ref["relative_error"])


def test_hessian_matches_2xxt(cuda):
    rng = np.random.default_rng(3)
    n = 200
    H = P.Hessian(n, device=0)
    X1 = rng.standard_normal((n, 50)).astype(np.float32)
    X2 = rng.standard_normal((n, 70)).astype(np.float32)
    H.accumulate(torch.from_numpy(X1).cuda())
    H.accumulate(torch.from_numpy(X2).cuda())  # mergeable by addition (hessian.hpp:71-76)
    want = 2.0 * (X1.astype(np.float64) @ X1.T.astype(np.float64) + X2.astype(np.float64) @ X2.T.astype(np.float64))
    got = H.matrix()
    assert np.array_equal(got, got.T)  # the exactly symmetric form
    assert np.max(np.abs(got - want)) <= 1e-9 * np.max(np.abs(want))


def test_encoder_errors(cuda):
    H = P.Hessian(64, device=0)
    W = torch.zeros(16, 64, device="cuda")
    with pytest.raises(P.SpqrError, match="EmptyInput"):
        H.quantize(W)  # no calibration samples (hessian.hpp:140)
    H.accumulate(torch.randn(64, 8, device="cuda"))
    with pytest.raises(P.SpqrError, match="ConfigInvalid"):
        H.quantize(W, weight_bits=9)


def test_gpu_encoder_stream_decodes_and_runs(cuda, ref_encoder):
    """The encoded layer runs on the decode kernels: matvec == the reference
    decode's reconstruction times x."""
    import oracle as O

    W, X = _layer(128, 512, 256, seed=11)
    H = P.Hessian(512, device=0)
    H.accumulate(torch.from_numpy(X).cuda())
    s, rep = H.quantize(torch.from_numpy(W).cuda())
    assert 0.0 < rep["relative_error"] < 0.1
    L = P.Layer(s)
    x = torch.randn(512, generator=torch.Generator().manual_seed(2)).cuda()
    y = torch.empty(128, device="cuda")
    L.matvec(x, y)
    t = O.Oracle().decode(s)
    assert O.relative_l2(y.cpu().numpy(), t.matvec(x.cpu().numpy())) <= 1e-5


@pytest.mark.parametrize("target", [0.002, 0.01, 0.0001])
def test_gpu_tune_tau_matches_reference(cuda, ref_encoder, target):
    """tune_tau (solver.hpp:546-640): same tau, same stream, same verdict."""
    W, X = _layer(64, 256, 256, seed=5, outlier_cols=1)
    s_ref, rep_ref = ref_encoder.quantize(W, X, target_rate=target)
    H = P.Hessian(256, device=0)
    H.accumulate(torch.from_numpy(X).cuda())
    s_gpu, rep_gpu = H.quantize(torch.from_numpy(W).cuda(), target_rate=target)
    assert rep_gpu["tau"] == rep_ref["tau"] and rep_gpu["target_reached"] == rep_ref["target_reached"]
    assert s_gpu == s_ref
