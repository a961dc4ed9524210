"""Bit-level numpy model of the tiled GEMV kernel (gemv_tiled / xprep_tiled).

Test infrastructure: it reads the tiled HBM image the C++ loader produces
(spqr_debug_tiled_host) and replays, lane by lane, exactly what the CUDA kernel
does -- window selection (even byte / PRMT / shift), the single LOP3 mask, the
binary16-subnormal interpretation, the per-column 2^-p pre-scale of x, the
per-block power-of-two scaling, and the fp32 epilogue -- so the layout logic is
checked on the CPU before any GPU time is spent.
"""
from __future__ import annotations

import numpy as np

import paper_2306_03078_b200 as P


def cw_of(bw):
    return 3 if bw == 3 else 1


def mpc_of(bw):
    return {3: 4, 4: 1, 2: 2}[bw]


def column_prescale(bw, k, cc):
    m = (k % 8) % mpc_of(bw)
    return (bw * (2 * m + cc // 8)) & 7


def _window(w, B, CW):
    if B % 2 == 0:
        return int(w[B // 2])
    if B // 2 + 1 < CW:
        a, b = int(w[B // 2]), int(w[B // 2 + 1])
        # __byte_perm(a, b, 0x6341): bytes [a.b1, b.b0, a.b3, b.b2]
        return ((a >> 8) & 0xFF) | ((b & 0xFF) << 8) | (((a >> 24) & 0xFF) << 16) | (((b >> 16) & 0xFF) << 24)
    return int(w[B // 2]) >> 8


def extract_codes(stream: bytes):
    """Replay the kernel's A-fragment extraction; returns (codes m_pad x n_pad,
    prescale exponent per element) recovered from the tiled image."""
    info = P.validate(stream)
    bw, bs, bz = info["weight_bits"], info["scale_bits"], info["zero_bits"]
    t = P.debug_tiled_host(stream)
    Gn, Pn, cb = t["Gn"], t["Pn"], t["cell_bytes"]
    CW, MPC = cw_of(bw), mpc_of(bw)
    NP = 16 * CW // bw
    MASK = (1 << bw) - 1
    unit = cb // 2
    codes = np.zeros((Gn * 32, Pn * 256), np.int64)
    pre = np.full((Gn * 32, Pn * 256), -1, np.int64)
    cells = t["cells"]
    for G in range(Gn):
        for Pp in range(Pn):
            base = int(t["cell_off"][G * Pn + Pp])
            for u in range(2):
                ub = base + u * unit
                for lane in range(32):
                    g, tt = lane >> 2, lane & 3
                    words = cells[ub + lane * 16 * bw: ub + (lane + 1) * 16 * bw].view(np.uint32)
                    for mu in range(16):
                        c, mm = mu // MPC, mu % MPC
                        w = words[CW * c: CW * c + CW]
                        for r in range(4):
                            rho, kh = r & 1, r >> 1
                            qq = 2 * mm + kh
                            i = rho * (NP // 2) + qq
                            B, pp = (bw * i) >> 3, (bw * i) & 7
                            a = _window(w, B, CW) & ((MASK << pp) * 0x00010001)
                            row = 32 * G + 16 * u + g + 8 * rho
                            col = 256 * Pp + 16 * mu + 2 * tt + 8 * kh
                            for e, half in ((0, a & 0xFFFF), (1, a >> 16)):
                                # binary16 subnormal value = half * 2^-24 = code * 2^(pp-24)
                                assert half & 0x7C00 == 0, "window escaped the mantissa"
                                assert half % (1 << pp) == 0
                                codes[row, col + e] = half >> pp
                                pre[row, col + e] = pp
    return codes, pre


def model_matvec(stream: bytes, x: np.ndarray, xlo: bool = True) -> np.ndarray:
    """y = W x as the tiled kernel computes it (float32 epilogue, float64 MMA)."""
    info = P.validate(stream)
    a = P.decode_arrays(stream)
    bw, bs, bz = info["weight_bits"], info["scale_bits"], info["zero_bits"]
    m, n = info["rows"], info["cols"]
    codes, pre = extract_codes(stream)
    n_pad = codes.shape[1]
    nblk = n_pad // 16
    order = a["order"] if a["order"] is not None else np.arange(n)
    xs = np.zeros(n_pad, np.float32)
    xs[:n] = np.asarray(x, np.float32)[order]
    # xprep
    eff = np.zeros(n_pad, np.float64)   # effective scaled x (what the MMA multiplies, times 2^p)
    SC = np.zeros(nblk, np.float32)
    XX = np.zeros(nblk, np.float32)
    for k in range(nblk):
        v = xs[16 * k:16 * k + 16]
        mx = float(np.max(np.abs(v)))
        e = 15 - int(np.frexp(mx)[1]) if mx > 0 else 0
        Xs = np.zeros(16, np.float32)
        for cc in range(16):
            p = column_prescale(bw, k, cc)
            assert pre[:, 16 * k + cc].min() in (p, -1) and pre[:, 16 * k + cc].max() == p
            s = np.float32(np.ldexp(np.float64(v[cc]), e - p))
            hi = np.float16(s)
            ef = np.float32(hi)
            if xlo:
                lo = np.float16(np.float32(s - ef))
                ef = np.float32(ef + np.float32(lo))
            eff[16 * k + cc] = np.ldexp(np.float64(ef), p)
            Xs[cc] = np.float32(np.ldexp(np.float64(ef), p))
        for d in (1, 2, 4, 8):  # xprep's butterfly order
            Xs = (Xs + Xs[np.arange(16) ^ d]).astype(np.float32)
        X = Xs[0]
        SC[k] = np.float32(2.0 ** (24 - e))
        XX[k] = np.float32(-X * np.float32(5.9604644775390625e-08))
    # "MMA": C = sum code * 2^(p-24) * eff * 2^-p  (exact in float64)
    D = (codes.reshape(codes.shape[0], nblk, 16) * eff.reshape(1, nblk, 16)).sum(-1) * 2.0 ** -24
    D = D.astype(np.float32)
    nb = (n + 15) // 16
    ng = (m + 15) // 16
    sc = a["scale_codes"].reshape(nb, m)
    zc = a["zero_codes"].reshape(nb, m)
    scal = a["group_scalars"].reshape(nb, ng, 4).view(np.float16).astype(np.float32)
    y = np.zeros(m, np.float32)
    for k in range(nb):
        Ss, Zs, Sz, Zz = (scal[k, np.arange(m) // 16, i] for i in range(4))
        A1 = (Ss * SC[k]).astype(np.float32)
        A0 = (-A1 * Zs).astype(np.float32)
        B0 = (-Sz * Zz).astype(np.float32)
        shat = (A1 * sc[k].astype(np.float32) + A0).astype(np.float32)
        zhat = (Sz * zc[k].astype(np.float32) + B0).astype(np.float32)
        tt = (zhat * XX[k] + D[:m, k]).astype(np.float32)
        y = (y + shat * tt).astype(np.float32)
    # outliers
    for r, c, v in zip(a["outlier_rows"], a["outlier_cols"], a["outlier_vals"]):
        y[r] += np.float32(np.uint16(v).view(np.float16)) * xs[c]
    return y
