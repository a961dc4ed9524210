"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Run in the dev container (needs /root/reference, via oracle/_ref/libspqr_ref.so):

    python tests/golden/make_golden.py

Every expected output in the fixtures (stream bytes, dequantized weights as
uint32 bit patterns, matvec outputs, error codes, size-model numbers) is
produced by the unmodified reference compiled from /root/reference
(oracle/Makefile).  The C restatement and the CUDA path are checked against
these files; nothing here is produced by our own code.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

from oracle import OracleError, Reference, build  # noqa: E402
from paper_2306_03078_b200 import synth  # noqa: E402

# (name, rows, cols, kwargs) -- small layers covering the edge cases the
# SPEC names: ragged m/n, permutation, raw-16 statistics, integer zero,
# 2/4-bit widths, non-16 group sizes, zero and 5% outlier densities.
CASES = [
    ("base_48x80", 48, 80, {}),
    ("perm_64x96", 64, 96, {"permute": True}),
    ("ragged_37x53_b8x4_w4_s16_z5", 37, 53, {"beta1": 8, "beta2": 4, "weight_bits": 4,
                                             "scale_bits": 16, "zero_bits": 5}),
    ("intzero_40x40", 40, 40, {"integer_zero": True}),
    ("w2_s2_z16_33x70", 33, 70, {"weight_bits": 2, "scale_bits": 2, "zero_bits": 16}),
    ("rate5_64x256", 64, 256, {"outlier_rate": 0.05}),
    ("rate0_96x128", 96, 128, {"outlier_rate": 0.0}),
    ("w4_64x256", 64, 256, {"weight_bits": 4, "scale_bits": 4, "zero_bits": 4}),
    ("raw_both_32x48", 32, 48, {"scale_bits": 16, "zero_bits": 16}),
    ("perm_ragged_50x300", 50, 300, {"permute": True, "outlier_rate": 0.02}),
    ("clustered_32x512", 32, 512, {"clustered": True, "outlier_rate": 0.03}),
    ("fast_128x512", 128, 512, {"permute": True}),
]


def appendix_a(R: Reference) -> bytes:
    """m=16, n=32, 3/3/3, beta 16x16, two outliers."""
    m, n = 16, 32
    r = np.arange(m)[:, None]
    c = np.arange(n)[None, :]
    codes = ((r + c) % 8).astype(np.uint8).reshape(-1)
    sc = np.stack([np.arange(m) % 8] * 2).astype(np.uint8).reshape(-1)
    zc = np.stack([(3 * np.arange(m) + k) % 8 for k in range(2)]).astype(np.uint8).reshape(-1)
    h = R.fp16_from_float
    scal = np.array([[h(0.001), h(-1.0), h(0.5), h(0.25)],
                     [h(0.002), h(-1.0), h(0.5), h(0.25)]], np.uint16).reshape(-1)
    a = {"rows": m, "cols": n, "weight_bits": 3, "scale_bits": 3, "zero_bits": 3, "beta1": 16,
         "beta2": 16, "flags": 0x18, "tau": 0.1, "lambda_rel": 0.01, "order": None,
         "codes": codes, "scale_codes": sc, "zero_codes": zc, "group_scalars": scal,
         "outlier_rows": np.array([0, 3], np.uint32), "outlier_cols": np.array([5, 20], np.uint32),
         "outlier_vals": np.array([h(0.125), h(-0.5)], np.uint16)}
    return R.from_arrays(a).encode()


def corruptions(stream: bytes, m: int) -> dict:
    """Malformed variants of a stream; expected Errc comes from the reference."""
    s = bytearray(stream)
    nnz = int(np.frombuffer(stream[28:32], np.uint32)[0])
    csr = len(stream) - 4 * nnz - 4 * (m + 1)
    out = {
        "truncated": bytes(s[:-1]),
        "trailing": bytes(s + b"\0"),
        "bad_magic": b"XPQR" + bytes(s[4:]),
        "bad_version": bytes(s[:4]) + b"\x02\x00" + bytes(s[6:]),
        "zero_rows": bytes(s[:8]) + b"\0\0\0\0" + bytes(s[12:]),
        "bad_wbits": bytes(s[:16]) + b"\x09" + bytes(s[17:]),
        "bad_sbits": bytes(s[:17]) + b"\x0c" + bytes(s[18:]),
        "short_header": bytes(s[:40]),
    }
    t = bytearray(s)
    t[csr:csr + 4] = (1).to_bytes(4, "little")
    out["csr_nonzero_start"] = bytes(t)
    if nnz >= 2:
        t = bytearray(s)
        rs = np.frombuffer(stream[csr:csr + 4 * (m + 1)], np.uint32).copy()
        i = int(np.argmax(rs > 0))  # first row start > 0
        rs[i] = rs[i] + 1  # now rs[i] > rs[i+1] somewhere or sum mismatch
        t[csr:csr + 4 * (m + 1)] = rs.tobytes()
        out["csr_decreasing"] = bytes(t)
        t = bytearray(s)
        ent = csr + 4 * (m + 1)
        t[ent:ent + 2] = (0xFFFF).to_bytes(2, "little")  # column out of range
        out["csr_col_range"] = bytes(t)
        t = bytearray(s)
        # make the second entry's column equal the first's within one row when possible
        t[ent + 4:ent + 6] = t[ent:ent + 2]
        out["csr_dup_col"] = bytes(t)
    # negative second-level scale in the first record (header + optional perm)
    flags = int(np.frombuffer(stream[6:8], np.uint16)[0])
    sb = stream[17]
    if sb != 16:
        off = 48 + (4 * int(np.frombuffer(stream[12:16], np.uint32)[0]) if flags & 1 else 0)
        t = bytearray(s)
        t[off:off + 2] = (0xBC00).to_bytes(2, "little")  # -1.0
        out["negative_scale_s"] = bytes(t)
    return out


def main() -> None:
    build()
    R = Reference()
    out = {}
    out["appendix_a"] = np.frombuffer(appendix_a(R), np.uint8)
    for name, m, n, kw in CASES:
        a = synth.make_layer(m, n, seed=7, **kw)
        stream = R.from_arrays(a).encode()
        t = R.decode(stream)
        assert t.encode() == stream
        w = t.dequantize_full()
        rng = np.random.default_rng(11)
        xs = rng.standard_normal((3, n)).astype(np.float16).astype(np.float32)
        xs[2] = 0.0
        xs[2, n // 3] = 1.0  # e_j
        ys = np.stack([t.matvec(x) for x in xs])
        yn = np.stack([t.matvec_naive(x) for x in xs])
        out[f"{name}/stream"] = np.frombuffer(stream, np.uint8)
        out[f"{name}/w_bits"] = w.view(np.uint32)
        out[f"{name}/x"] = xs
        out[f"{name}/y"] = ys
        out[f"{name}/y_naive"] = yn
        mb = R.measure_actual_bits(t)
        out[f"{name}/measured_bits"] = mb
        errs = []
        for cname, bad in corruptions(stream, m).items():
            try:
                R.decode(bad)
                code = 0
            except OracleError as e:
                code = e.status
            errs.append((cname, code))
            out[f"{name}/bad/{cname}/status"] = np.array([code], np.int32)
    # size model and average-bits KATs (PAPER Table 10)
    grid = []
    for b1 in (4, 8, 16, 32, 64, 128):
        for b2 in (4, 8, 16, 32, 64, 128):
            for ro in (0.0, 0.004, 0.01):
                grid.append([3, 3, 3, b1, b2, ro] + list(R.estimate_avg_bits(3, 3, 3, b1, b2, ro)))
    out["avg_bits_grid"] = np.array(grid, np.float64)
    sizes = []
    for (m, n, wb, sb, zb, b1, b2, nnz, hp) in [
            (4096, 4096, 3, 3, 3, 16, 16, 167772, 0), (11008, 4096, 3, 3, 3, 16, 16, 450887, 0),
            (4096, 11008, 3, 3, 3, 16, 16, 450887, 0), (8192, 8192, 3, 3, 3, 16, 16, 671088, 0),
            (22016, 8192, 3, 3, 3, 16, 16, 1803550, 0), (8192, 22016, 3, 3, 3, 16, 16, 1803550, 0),
            (8192, 8192, 4, 3, 3, 16, 16, 671088, 0), (37, 53, 4, 16, 5, 8, 4, 12, 1),
            (16, 16, 3, 3, 3, 16, 16, 0, 0)]:
        sizes.append([m, n, wb, sb, zb, b1, b2, nnz, hp, R.payload_bytes(m, n, wb, sb, zb, b1, b2, nnz, hp)])
    out["payload_sizes"] = np.array(sizes, np.int64)
    fp = np.arange(65536, dtype=np.uint32)
    out["fp16_to_float_bits"] = np.array([np.float32(R.fp16_to_float(int(h))).view(np.uint32) for h in fp],
                                         np.uint32)
    probe = np.random.default_rng(5).standard_normal(4000).astype(np.float32) * \
        np.float32(10.0) ** np.random.default_rng(6).integers(-9, 6, 4000).astype(np.float32)
    probe = np.concatenate([probe, np.array([65504, 65519.99, 65520, 1e9, -1e9, 6e-8, 3e-8, 2.9e-8,
                                             np.inf, -np.inf, 0.0, -0.0], np.float32)])
    out["fp16_from_float_in"] = probe
    out["fp16_from_float_out"] = np.array([R.fp16_from_float(float(f)) for f in probe], np.uint16)
    path = os.path.join(HERE, "golden.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({os.path.getsize(path)} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
