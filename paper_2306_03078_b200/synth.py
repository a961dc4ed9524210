"""Synthetic SpQR layers (numpy).

Two generators:

* ``make_layer`` -- a realistic layer: W ~ N(0, 0.02^2), exact-count outliers
  injected at large magnitude, first-level min-max statistics per
  (row, beta1-block) with outliers masked, second-level b_s/b_z-bit
  quantisation over beta2-row groups with binary16 scalars, codes by
  round-half-up.  It follows the reference encoder's statistics rules
  (fit_group_minmax quantizer.hpp:77-97, quant_code :50-56, stat_dequant
  :65-67, fit_statistics_impl solver.hpp:180-266, outlier correction
  solver.hpp:480-483) without GPTQ error feedback (no Hessian here).
  Returns the flat arrays the encoder consumes.

* ``random_stream`` -- a valid .spqr stream with uniform-random codes and
  plausible binary16 scalars, written directly as bytes.  Bytes are identical
  in size to a real layer; used for timing runs where numeric realism does
  not matter.
"""
from __future__ import annotations

import numpy as np

RAW = 16
F_PERM, F_ACT, F_INTZERO, F_FULLRANGE, F_OUTLIERS = 1, 2, 4, 8, 16


def _minmax_fit(v: np.ndarray, bits: int, full_range_sign: bool, integer_zero: bool):
    """fit_group_minmax (quantizer.hpp:77-97) along the last axis, float64."""
    mn = v.min(axis=-1)
    mx = v.max(axis=-1)
    if not full_range_sign:
        mn = np.minimum(mn, 0.0)
        mx = np.maximum(mx, 0.0)
    maxq = float((1 << bits) - 1)
    deg = mx == mn
    s = np.where(deg, 1.0, (mx - mn) / maxq)
    with np.errstate(divide="ignore", invalid="ignore"):
        z = np.where(deg, -mn, -mn / np.where(deg, 1.0, s))
    if integer_zero:
        z = np.clip(np.floor(z + 0.5), 0.0, maxq)
    return s, z


def _quant_code(v, s, z, maxq: int):
    """quant_code (quantizer.hpp:50-56), float64, round half up, clamped."""
    with np.errstate(divide="ignore", invalid="ignore"):
        t = np.floor(v / s + z + 0.5)
    t = np.where(np.logical_not(s > 0.0), 0.0, t)
    t = np.where(np.logical_not(t > 0.0), 0.0, t)
    t = np.minimum(t, float(maxq))
    return t.astype(np.uint8)


def _h2f(h: np.ndarray) -> np.ndarray:
    return h.view(np.float16).astype(np.float32)


def _f2h(f) -> np.ndarray:
    # numpy's float32->float16 is RNE; the reference saturates instead of
    # producing inf (common.hpp:81-83).  Clamp first to match.
    f = np.clip(np.asarray(f, np.float32), -65504.0, 65504.0)
    return f.astype(np.float16).view(np.uint16)


def _stat_dequant(s16, z16, code):
    """stat_dequant (quantizer.hpp:65-67) in binary32."""
    return (_h2f(s16) * (code.astype(np.float32) - _h2f(z16))).astype(np.float32)


def make_layer(m: int, n: int, weight_bits: int = 3, scale_bits: int = 3, zero_bits: int = 3,
               beta1: int = 16, beta2: int = 16, outlier_rate: float = 0.01, seed: int = 0,
               permute: bool = False, integer_zero: bool = False, full_range_sign: bool = True,
               clustered: bool = False, nnz: int | None = None) -> dict:
    rng = np.random.default_rng(seed)
    W = (rng.standard_normal((m, n)) * 0.02).astype(np.float32)
    order = rng.permutation(n).astype(np.uint32) if permute else None
    Wp = W[:, order] if order is not None else W  # solve order
    Wp = Wp.astype(np.float64)

    # exact-count outliers, injected at large magnitude
    k = int(np.floor(outlier_rate * m * n)) if nnz is None else int(nnz)
    orng = np.random.default_rng(seed + 1)
    if k > 0:
        if clustered:  # concentrate in the first quarter of rows (load-balance test)
            rows_hot = max(1, m // 4)
            flat = orng.choice(rows_hot * n, size=min(k, rows_hot * n), replace=False)
            if flat.size < k:
                rest = orng.choice(np.arange(rows_hot * n, m * n), size=k - flat.size, replace=False)
                flat = np.concatenate([flat, rest])
        else:
            flat = orng.choice(m * n, size=k, replace=False)
        flat = np.sort(flat)
        orow, ocol = (flat // n).astype(np.uint32), (flat % n).astype(np.uint32)
        Wp[orow, ocol] += orng.standard_normal(k) * 0.2
    else:
        orow = ocol = np.zeros(0, np.uint32)
    mask = np.zeros((m, n), bool)
    mask[orow, ocol] = True

    nb = (n + beta1 - 1) // beta1
    ng = (m + beta2 - 1) // beta2
    maxq = (1 << weight_bits) - 1
    codes = np.zeros((m, n), np.uint8)
    base = np.zeros((m, n), np.float32)
    sc = np.zeros((nb, m), np.uint8) if scale_bits != RAW else None
    zc = np.zeros((nb, m), np.uint8) if zero_bits != RAW else None
    rs = np.zeros((nb, m), np.float32) if scale_bits == RAW else None
    rz = np.zeros((nb, m), np.float32) if zero_bits == RAW else None
    anyq = scale_bits != RAW or zero_bits != RAW
    scal = np.zeros((nb, ng, 4), np.uint16)
    scal[:, :, 0] = 0x3C00
    scal[:, :, 2] = 0x3C00

    for kb in range(nb):
        c0, c1 = kb * beta1, min(n, kb * beta1 + beta1)
        blk = np.where(mask[:, c0:c1], 0.0, Wp[:, c0:c1])
        s1, z1 = _minmax_fit(blk, weight_bits, full_range_sign, integer_zero)
        # scales
        if scale_bits == RAW:
            rs[kb] = s1.astype(np.float32)
            scale = rs[kb]
        else:
            scale = np.zeros(m, np.float32)
            for g in range(ng):
                r0, r1 = g * beta2, min(m, g * beta2 + beta2)
                ss, zs = _minmax_fit(s1[r0:r1], scale_bits, True, False)
                s16, z16 = _f2h(np.float32(ss)), _f2h(np.float32(zs))
                scal[kb, g, 0], scal[kb, g, 1] = s16, z16
                code = _quant_code(s1[r0:r1], float(_h2f(s16)), float(_h2f(z16)), (1 << scale_bits) - 1)
                sc[kb, r0:r1] = code
                scale[r0:r1] = _stat_dequant(s16, z16, code)
        # zeros
        if zero_bits == RAW:
            rz[kb] = z1.astype(np.float32)
            zero = rz[kb]
        elif integer_zero:
            zc[kb] = z1.astype(np.uint8)
            zero = zc[kb].astype(np.float32)
        else:
            zero = np.zeros(m, np.float32)
            for g in range(ng):
                r0, r1 = g * beta2, min(m, g * beta2 + beta2)
                sz, zz = _minmax_fit(z1[r0:r1], zero_bits, True, False)
                s16, z16 = _f2h(np.float32(sz)), _f2h(np.float32(zz))
                scal[kb, g, 2], scal[kb, g, 3] = s16, z16
                code = _quant_code(z1[r0:r1], float(_h2f(s16)), float(_h2f(z16)), (1 << zero_bits) - 1)
                zc[kb, r0:r1] = code
                zero[r0:r1] = _stat_dequant(s16, z16, code)
        s64 = scale.astype(np.float64)[:, None]
        z64 = zero.astype(np.float64)[:, None]
        q = _quant_code(Wp[:, c0:c1], s64, z64, maxq)
        codes[:, c0:c1] = q
        base[:, c0:c1] = scale[:, None] * (q.astype(np.float32) - zero[:, None])  # dequant_value

    oval = _f2h((Wp[orow, ocol] - base[orow, ocol].astype(np.float64)).astype(np.float32)) \
        if k > 0 else np.zeros(0, np.uint16)
    flags = (F_FULLRANGE if full_range_sign else 0) | F_OUTLIERS | (F_INTZERO if integer_zero else 0)
    if permute:
        flags |= F_ACT
    return {
        "rows": m, "cols": n, "weight_bits": weight_bits, "scale_bits": scale_bits,
        "zero_bits": zero_bits, "beta1": beta1, "beta2": beta2, "flags": flags,
        "tau": 0.1, "lambda_rel": 0.01, "order": order, "codes": codes.reshape(-1),
        "scale_codes": None if sc is None else sc.reshape(-1),
        "zero_codes": None if zc is None else zc.reshape(-1),
        "raw_scales": None if rs is None else rs.reshape(-1),
        "raw_zeros": None if rz is None else rz.reshape(-1),
        "group_scalars": scal.reshape(-1) if anyq else None,
        "outlier_rows": orow, "outlier_cols": ocol, "outlier_vals": oval,
    }


def payload_bytes(m, n, wb, sb, zb, b1, b2, nnz, has_perm) -> int:
    """stream_payload_bytes (layout.hpp:47-64), closed form."""
    def pk(c, b):
        return (c * b + 7) // 8

    def rec(gr, bw):
        b = (4 + pk(gr, sb)) if sb <= 8 else 4 * gr
        b += (4 + pk(gr, zb)) if zb <= 8 else 4 * gr
        return b + pk(gr * bw, wb)

    nb_full, lastw = divmod(n, b1)
    ng_full, lastr = divmod(m, b2)
    per_col = ng_full * rec(b2, b1) + (rec(lastr, b1) if lastr else 0)
    total = nb_full * per_col
    if lastw:
        total += ng_full * rec(b2, lastw) + (rec(lastr, lastw) if lastr else 0)
    return (4 * n if has_perm else 0) + total + 4 * (m + 1) + 4 * nnz


def random_stream(m: int, n: int, weight_bits: int = 3, scale_bits: int = 3, zero_bits: int = 3,
                  outlier_rate: float = 0.01, seed: int = 0, permute: bool = False, beta1: int = 16,
                  beta2: int = 16) -> bytes:
    """A valid stream with random codes (timing workloads): full beta1 x beta2
    group records (m % beta2 == 0, n % beta1 == 0)."""
    assert m % beta2 == 0 and n % beta1 == 0
    for b in (weight_bits, scale_bits, zero_bits):
        assert (beta2 * b) % 8 == 0 and 1 <= b <= 8
    rng = np.random.default_rng(seed)
    nb, ng = n // beta1, m // beta2
    nnz = int(np.floor(outlier_rate * m * n))
    rec = 8 + (beta2 * scale_bits + beta2 * zero_bits + beta1 * beta2 * weight_bits) // 8
    hdr = np.zeros(48, np.uint8)
    hdr[0:4] = np.frombuffer(b"SPQR", np.uint8)
    hdr[4:6] = np.array([1], np.uint16).view(np.uint8)
    flags = F_FULLRANGE | F_OUTLIERS | (F_PERM | F_ACT if permute else 0)
    hdr[6:8] = np.array([flags], np.uint16).view(np.uint8)
    hdr[8:16] = np.array([m, n], np.uint32).view(np.uint8)
    hdr[16:20] = [weight_bits, scale_bits, zero_bits, 0]
    hdr[20:32] = np.array([beta1, beta2, nnz], np.uint32).view(np.uint8)
    hdr[32:40] = np.array([0.1, 0.01], np.float32).view(np.uint8)
    parts = [hdr]
    if permute:
        parts.append(rng.permutation(n).astype(np.uint32).view(np.uint8))
    recs = rng.integers(0, 256, size=(nb * ng, rec), dtype=np.uint8)
    # plausible second-level scalars: scale_s ~ 1e-3 (>= 0), scale_z ~ -0.5,
    # zero_s ~ 0.5, zero_z ~ 0
    sc = np.empty((nb * ng, 4), np.float32)
    sc[:, 0] = rng.uniform(2e-4, 2e-3, nb * ng)
    sc[:, 1] = rng.uniform(-1.0, 0.0, nb * ng)
    sc[:, 2] = rng.uniform(0.3, 1.2, nb * ng)
    sc[:, 3] = rng.uniform(-0.5, 0.5, nb * ng)
    recs[:, 0:8] = _f2h(sc).view(np.uint8).reshape(nb * ng, 8)
    parts.append(recs.reshape(-1))
    # CSR: exactly nnz unique positions, sorted by (row, col)
    if nnz:
        flat = np.unique(rng.integers(0, m * n, size=int(nnz * 1.05) + 16, dtype=np.int64))
        while flat.size < nnz:
            flat = np.unique(np.concatenate([flat, rng.integers(0, m * n, size=nnz, dtype=np.int64)]))
        flat = np.sort(rng.choice(flat, size=nnz, replace=False))
        rows, cols = flat // n, flat % n
    else:
        rows = cols = np.zeros(0, np.int64)
    rstarts = np.zeros(m + 1, np.uint32)
    np.cumsum(np.bincount(rows, minlength=m), out=rstarts[1:])
    parts.append(rstarts.view(np.uint8))
    ent = np.empty((nnz, 2), np.uint16)
    ent[:, 0] = cols.astype(np.uint16)
    ent[:, 1] = _f2h(rng.standard_normal(nnz).astype(np.float32) * 0.05)
    parts.append(ent.reshape(-1).view(np.uint8))
    out = np.concatenate(parts).tobytes()
    assert len(out) == 48 + payload_bytes(m, n, weight_bits, scale_bits, zero_bits, beta1, beta2, nnz, permute)
    return out


def random_x(n: int, batch: int = 1, seed: int = 2, dtype=np.float16) -> np.ndarray:
    """x ~ N(0,1), fp16 by default (the north-star benchmark input)."""
    rng = np.random.default_rng(seed)
    return rng.standard_normal((batch, n)).astype(dtype)
