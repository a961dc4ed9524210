"""Pin the oracle: the C restatement against the golden fixtures (made by the
reference itself, tests/golden/make_golden.py) and against the reference
compiled from /root/reference (oracle/_ref) on fresh seeded layers."""
from __future__ import annotations

import numpy as np
import pytest

from golden.make_golden import corruptions
from oracle import OracleError, relative_l2
from paper_2306_03078_b200 import synth


def test_golden_streams_decode_and_reencode(golden, golden_cases, oracle_c):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        t = oracle_c.decode(s)
        assert t.encode() == s, name


def test_golden_dequantize_bit_exact(golden, golden_cases, oracle_c):
    for name in golden_cases:
        t = oracle_c.decode(golden[f"{name}/stream"].tobytes())
        w = t.dequantize_full()
        assert np.array_equal(w.view(np.uint32), golden[f"{name}/w_bits"]), name


def test_golden_matvec(golden, golden_cases, oracle_c):
    for name in golden_cases:
        t = oracle_c.decode(golden[f"{name}/stream"].tobytes())
        for x, y, yn in zip(golden[f"{name}/x"], golden[f"{name}/y"], golden[f"{name}/y_naive"]):
            assert np.array_equal(t.matvec(x).view(np.uint32), y.view(np.uint32)), name
            assert np.array_equal(t.matvec_naive(x).view(np.uint32), yn.view(np.uint32)), name


def test_golden_error_codes(golden, golden_cases, oracle_c):
    for name in golden_cases:
        s = golden[f"{name}/stream"].tobytes()
        m = int(np.frombuffer(s[8:12], np.uint32)[0])
        for cname, bad in corruptions(s, m).items():
            want = int(golden[f"{name}/bad/{cname}/status"][0])
            try:
                oracle_c.decode(bad)
                got = 0
            except OracleError as e:
                got = e.status
            assert got == want, (name, cname, got, want)


def test_appendix_a_bytes(golden, oracle_c):
    """SURVEY Appendix A / SPEC.md:356 -- 116-byte group records, 356-byte stream."""
    s = golden["appendix_a"].tobytes()
    assert len(s) == 356 == 48 + 2 * 116 + 17 * 4 + 2 * 4
    assert s[48:68].hex() == "191400bc00380034" + "88c6fa88c6fa" + "98c3ab98c3ab"
    assert s[68:80].hex() == "88c6fa88c6fa" + "d1581fd1581f"
    t = oracle_c.decode(s)
    w = t.dequantize_full()
    assert np.float32(w[0, 0]) == np.float32(1.25050545e-4)
    rs = np.frombuffer(s[280:348], np.uint32)
    assert rs.tolist() == [0, 1, 1, 1, 2] + [2] * 12
    assert s[348:356].hex() == "05000030" + "140000b8"


def test_size_model_and_avg_bits(golden, oracle_c):
    for row in golden["payload_sizes"]:
        m, n, wb, sb, zb, b1, b2, nnz, hp, want = (int(v) for v in row)
        assert oracle_c.payload_bytes(m, n, wb, sb, zb, b1, b2, nnz, hp) == want
        assert synth.payload_bytes(m, n, wb, sb, zb, b1, b2, nnz, hp) == want
    for row in golden["avg_bits_grid"]:
        got = oracle_c.estimate_avg_bits(*(int(v) for v in row[:5]), float(row[5]))
        np.testing.assert_array_equal(got, row[6:])
    # SPEC.md:372-374 / PAPER Table 10 known answers
    assert abs(oracle_c.estimate_avg_bits(3, 3, 3, 16, 32, 0.004)[0] - 3.63) < 0.01
    assert oracle_c.estimate_avg_bits(3, 3, 3, 4, 4, 0.0)[0] == 8.5
    assert oracle_c.estimate_avg_bits(3, 3, 3, 16, 32, 0.0)[0] == 3.5


def test_fp16_tables(golden, oracle_c):
    tbl = golden["fp16_to_float_bits"]
    for h in list(range(0, 65536, 7)) + [0x7C00, 0xFC00, 0x0001, 0x8001, 0x03FF, 0x7BFF]:
        got = np.float32(oracle_c.fp16_to_float(h)).view(np.uint32)
        assert got == tbl[h] or (h & 0x7C00) == 0x7C00 and (h & 0x3FF), h
    for f, want in zip(golden["fp16_from_float_in"], golden["fp16_from_float_out"]):
        assert oracle_c.fp16_from_float(float(f)) == int(want), f


@pytest.mark.parametrize("seed", [0, 1, 2])
@pytest.mark.parametrize("cfg", [
    dict(m=80, n=160),
    dict(m=67, n=130, permute=True, outlier_rate=0.03),
    dict(m=64, n=128, weight_bits=4, scale_bits=4, zero_bits=4),
    dict(m=45, n=77, beta1=8, beta2=12, weight_bits=5, scale_bits=16, zero_bits=6),
    dict(m=32, n=64, integer_zero=True, outlier_rate=0.0),
])
def test_restatement_matches_reference(reference, oracle_c, cfg, seed):
    cfg = dict(cfg)
    m, n = cfg.pop("m"), cfg.pop("n")
    a = synth.make_layer(m, n, seed=seed, **cfg)
    s = reference.from_arrays(a).encode()
    assert oracle_c.from_arrays(a).encode() == s
    tr, to = reference.decode(s), oracle_c.decode(s)
    assert to.encode() == s
    assert np.array_equal(tr.dequantize_full().view(np.uint32), to.dequantize_full().view(np.uint32))
    x = np.random.default_rng(seed).standard_normal(n).astype(np.float32)
    assert np.array_equal(tr.matvec(x).view(np.uint32), to.matvec(x).view(np.uint32))
    assert relative_l2(to.matvec(x), to.matvec_naive(x)) <= 1e-6  # kernel.hpp:191
