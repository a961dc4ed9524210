"""ctypes loaders for the parity checkers.  TEST INFRASTRUCTURE ONLY.

Two interchangeable back ends with the same Python surface:

* ``Oracle``  -- oracle/liboracle.so, the plain-C restatement (spqr_oracle.c).
* ``Reference`` -- oracle/_ref/libspqr_ref.so, the unmodified reference headers
  compiled by oracle/Makefile (built in the dev container where
  /root/reference exists; the prebuilt .so travels to the GPU box).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspqr_ref.so")
REF_ENC_SO = os.path.join(HERE, "_ref", "libspqr_ref_enc.so")

ERRC = [
    "malformed_header", "shape_mismatch", "non_finite_value", "io_failure", "parse_error",
    "missing_file", "empty_input", "not_positive_definite", "dimension_mismatch",
    "config_invalid", "column_index_overflow", "malformed_stream", "version_unsupported",
    "corrupt_csr", "ill_conditioned", "outlier_budget_exceeded",
]


class OracleError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.errc = ERRC[status - 1] if 1 <= status <= len(ERRC) else f"status{status}"
        super().__init__(f"{where}: {self.errc}")


def build(force: bool = False) -> None:
    """Build liboracle.so (and _ref when the reference is present)."""
    if force or not os.path.exists(ORACLE_SO) or (
        os.path.getmtime(ORACLE_SO) < os.path.getmtime(os.path.join(HERE, "spqr_oracle.c"))
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, ORACLE_SO])
    if os.path.isdir("/root/reference/proj/include/spqr") and (
        force or not os.path.exists(REF_SO) or not os.path.exists(REF_ENC_SO)
        or os.path.getmtime(REF_SO) < os.path.getmtime(os.path.join(HERE, "ref_shim.cpp"))
        or os.path.getmtime(REF_ENC_SO) < os.path.getmtime(os.path.join(HERE, "ref_encoder.cpp"))
    ):
        subprocess.check_call(["make", "-s", "-C", HERE, "ref"])


_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def _arr(a, dt):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=dt)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _Backend:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.lib = C.CDLL(path)
        p = self.prefix
        L = self.lib
        self._decode = getattr(L, p + "decode")
        self._decode.argtypes = [C.c_void_p, C.c_size_t, C.POINTER(C.c_void_p)]
        self._free = getattr(L, p + "free")
        self._free.argtypes = [C.c_void_p]
        self._encode = getattr(L, p + "encode")
        self._encode.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t)]
        self._deq = getattr(L, p + "dequantize_full")
        self._deq.argtypes = [C.c_void_p, C.c_void_p]
        self._naive = getattr(L, p + "matvec_naive")
        self._naive.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        self._from = getattr(L, p + "from_arrays")
        self._from.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint32,
                               C.c_uint32, C.c_uint16, C.c_float, C.c_float] + [C.c_void_p] * 7 + [
                                   C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p,
                                   C.POINTER(C.c_void_p)]
        self._pb = getattr(L, p + "payload_bytes")
        self._pb.restype = C.c_size_t
        self._pb.argtypes = [C.c_uint32, C.c_uint32, C.c_int, C.c_int, C.c_int, C.c_uint32,
                             C.c_uint32, C.c_uint32, C.c_int]
        self._est = getattr(L, p + "estimate_avg_bits")
        self._est.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_double,
                              C.c_void_p]
        self._h2f = getattr(L, p + "fp16_to_float")
        self._h2f.restype = C.c_float
        self._h2f.argtypes = [C.c_uint16]
        self._f2h = getattr(L, p + "fp16_from_float")
        self._f2h.restype = C.c_uint16
        self._f2h.argtypes = [C.c_float]

    # -- tensors --------------------------------------------------------
    def decode(self, stream: bytes) -> "Tensor":
        buf = np.frombuffer(stream, dtype=np.uint8)
        h = C.c_void_p()
        rc = self._decode(_ptr(buf), buf.size, C.byref(h))
        if rc:
            raise OracleError(rc, "decode")
        return Tensor(self, h, stream)

    def from_arrays(self, a: dict) -> "Tensor":
        h = C.c_void_p()
        keep = {
            "order": _arr(a.get("order"), np.uint32), "codes": _arr(a["codes"], np.uint8),
            "scodes": _arr(a.get("scale_codes"), np.uint8), "zcodes": _arr(a.get("zero_codes"), np.uint8),
            "raw_s": _arr(a.get("raw_scales"), np.float32), "raw_z": _arr(a.get("raw_zeros"), np.float32),
            "scal": _arr(a.get("group_scalars"), np.uint16), "orow": _arr(a["outlier_rows"], np.uint32),
            "ocol": _arr(a["outlier_cols"], np.uint32), "oval": _arr(a["outlier_vals"], np.uint16),
        }
        rc = self._from(a["rows"], a["cols"], a["weight_bits"], a["scale_bits"], a["zero_bits"],
                        a["beta1"], a["beta2"], a.get("flags", 0x18), a.get("tau", 0.0),
                        a.get("lambda_rel", 0.0), _ptr(keep["order"]), _ptr(keep["codes"]),
                        _ptr(keep["scodes"]), _ptr(keep["zcodes"]), _ptr(keep["raw_s"]),
                        _ptr(keep["raw_z"]), _ptr(keep["scal"]), int(keep["orow"].size),
                        _ptr(keep["orow"]), _ptr(keep["ocol"]), _ptr(keep["oval"]), C.byref(h))
        if rc:
            raise OracleError(rc, "from_arrays")
        return Tensor(self, h, None)

    def payload_bytes(self, rows, cols, wb, sb, zb, b1, b2, nnz, has_perm) -> int:
        return int(self._pb(rows, cols, wb, sb, zb, b1, b2, nnz, int(bool(has_perm))))

    def estimate_avg_bits(self, bw, bs, bz, b1, b2, ro):
        out = np.zeros(5, np.float64)
        rc = self._est(bw, bs, bz, b1, b2, ro, _ptr(out))
        if rc:
            raise OracleError(rc, "estimate_avg_bits")
        return out

    def fp16_to_float(self, h: int) -> float:
        return float(self._h2f(h))

    def fp16_from_float(self, f: float) -> int:
        return int(self._f2h(f))


class Tensor:
    """A decoded tensor held by one of the back ends."""

    def __init__(self, be: _Backend, h, stream):
        self.be, self.h, self.stream = be, h, stream
        hdr = np.frombuffer(stream, np.uint8) if stream is not None else None
        self.rows = self.cols = None
        if hdr is not None:
            self.rows = int(hdr[8:12].view(np.uint32)[0])
            self.cols = int(hdr[12:16].view(np.uint32)[0])

    def __del__(self):
        try:
            if self.h:
                self.be._free(self.h)
        except Exception:
            pass

    def _dims(self):
        if self.rows is None:
            s = self.encode()
            hdr = np.frombuffer(s, np.uint8)
            self.rows = int(hdr[8:12].view(np.uint32)[0])
            self.cols = int(hdr[12:16].view(np.uint32)[0])
        return self.rows, self.cols

    def encode(self) -> bytes:
        n = C.c_size_t()
        rc = self.be._encode(self.h, None, 0, C.byref(n))
        if rc and rc != 4:  # io_failure = buffer too small for the C oracle
            raise OracleError(rc, "encode")
        out = np.empty(n.value, np.uint8)
        rc = self.be._encode(self.h, _ptr(out), out.size, C.byref(n))
        if rc:
            raise OracleError(rc, "encode")
        if self.rows is None:
            self.rows = int(out[8:12].view(np.uint32)[0])
            self.cols = int(out[12:16].view(np.uint32)[0])
        return out.tobytes()

    def dequantize_full(self) -> np.ndarray:
        m, n = self._dims()
        out = np.empty((m, n), np.float32)
        rc = self.be._deq(self.h, _ptr(out))
        if rc:
            raise OracleError(rc, "dequantize_full")
        return out

    def matvec(self, x) -> np.ndarray:
        m, n = self._dims()
        x = _arr(x, np.float32)
        y = np.empty(m, np.float32)
        rc = self.be._mv(self.h, x, y)
        if rc:
            raise OracleError(rc, "matvec")
        return y

    def matvec_naive(self, x) -> np.ndarray:
        m, n = self._dims()
        x = _arr(x, np.float32)
        y = np.empty(m, np.float32)
        rc = self.be._naive(self.h, _ptr(x), _ptr(y))
        if rc:
            raise OracleError(rc, "matvec_naive")
        return y


class Oracle(_Backend):
    """The C restatement (oracle/spqr_oracle.c)."""

    prefix = "oracle_"

    def __init__(self, path: str = ORACLE_SO):
        super().__init__(path)
        f = self.lib.oracle_matvec
        f.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint32]
        self._mv_raw = f
        self.lib.oracle_relative_l2.restype = C.c_double
        self.lib.oracle_relative_l2.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t]

    def _mv(self, h, x, y):
        return self._mv_raw(h, _ptr(x), _ptr(y), 64)

    def relative_l2(self, a, b) -> float:
        a = _arr(a, np.float32)
        b = _arr(b, np.float32)
        return float(self.lib.oracle_relative_l2(_ptr(a), _ptr(b), a.size))


class Reference(_Backend):
    """The unmodified reference, compiled into oracle/_ref/libspqr_ref.so."""

    prefix = "ref_"

    def __init__(self, path: str = REF_SO):
        super().__init__(path)
        L = self.lib
        L.ref_matvec.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_matvec_bands.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.ref_bench_matvec.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
        L.ref_measure_actual_bits.argtypes = [C.c_void_p, C.c_void_p]
        L.ref_slice_rows.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.POINTER(C.c_void_p)]

    def _mv(self, h, x, y):
        return self.lib.ref_matvec(h, _ptr(x), _ptr(y))

    def slice_rows(self, t: Tensor, r0: int, r1: int) -> Tensor:
        """Rows [r0, r1) of a decoded tensor as a reference tensor (ref_slice_rows)."""
        h = C.c_void_p()
        rc = self.lib.ref_slice_rows(t.h, r0, r1, C.byref(h))
        if rc:
            raise OracleError(rc, "slice_rows")
        band = Tensor(self, h, None)
        band.rows, band.cols = r1 - r0, t._dims()[1]
        return band

    def matvec_bands(self, tensors, x, nthreads: int) -> np.ndarray:
        """Multi-core harness: the reference's own matvec on disjoint row bands."""
        x = _arr(x, np.float32)
        m = sum(t._dims()[0] for t in tensors)
        y = np.empty(m, np.float32)
        hs = (C.c_void_p * len(tensors))(*[t.h for t in tensors])
        rc = self.lib.ref_matvec_bands(hs, len(tensors), _ptr(x), _ptr(y), nthreads)
        if rc:
            raise OracleError(rc, "matvec_bands")
        return y

    def bench_matvec(self, t: Tensor, x, repeats: int):
        out = np.zeros(3, np.float64)
        x = _arr(x, np.float32)
        rc = self.lib.ref_bench_matvec(t.h, _ptr(x), repeats, _ptr(out))
        if rc:
            raise OracleError(rc, "bench_matvec")
        return out

    def measure_actual_bits(self, t: Tensor):
        out = np.zeros(3, np.float64)
        rc = self.lib.ref_measure_actual_bits(t.h, _ptr(out))
        if rc:
            raise OracleError(rc, "measure_actual_bits")
        return out


class ReferenceEncoder:
    """The unmodified reference encoder (HessianAccumulator, finalize,
    spqr_quantize, make_spqr_tensor + encode) in oracle/_ref/libspqr_ref_enc.so,
    built with our functional minimal Eigen (oracle/eigen_min)."""

    def __init__(self, path: str = REF_ENC_SO):
        self.lib = C.CDLL(path)
        self.lib.ref_enc_quantize.restype = C.c_int
        self.lib.ref_enc_quantize.argtypes = [C.c_void_p, C.c_uint32, C.c_uint32, C.c_void_p, C.c_uint32,
                                              C.c_void_p, C.c_double, C.c_double, C.c_uint64, C.c_double,
                                              C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t), C.c_void_p]

    def quantize(self, W, X, weight_bits=3, scale_bits=3, zero_bits=3, beta1=16, beta2=16, order="natural",
                 act_order_key="hessian_diag", outliers=True, integer_zero=False, full_range_sign=True, tau=0.1,
                 lambda_rel=0.01, seed=0, target_rate=None):
        """W: m x n fp32; X: n x samples fp32 -> (stream bytes, report dict)."""
        W = _arr(W, np.float32)
        X = _arr(X, np.float32)
        m, n = W.shape
        cfg = np.array([weight_bits, scale_bits, zero_bits, beta1, beta2,
                        {"natural": 0, "act_order": 1, "shuffled": 2}[order],
                        {"hessian_diag": 0, "inverse_diag": 1}[act_order_key], int(outliers), int(integer_zero),
                        int(full_range_sign)], np.int32)
        cap = 48 + 4 * n + 2 * m * n + 64 * m * n // max(1, beta1) + 4 * (m + 1) + 4 * (m * n // 20 + 1) + 4096
        out = np.empty(cap, np.uint8)
        ln = C.c_size_t()
        rep = np.zeros(5, np.float64)
        rc = self.lib.ref_enc_quantize(_ptr(W), m, n, _ptr(X), X.shape[1], _ptr(cfg), tau, lambda_rel, seed,
                                       float(target_rate or 0.0), _ptr(out), cap, C.byref(ln), _ptr(rep))
        if rc:
            raise OracleError(rc, "ref_enc_quantize")
        r = {"relative_error": float(rep[0]), "outlier_rate": float(rep[1]), "bits_per_param": float(rep[2])}
        if target_rate:
            r.update(tau=float(rep[3]), target_reached=bool(rep[4]))
        return out[: ln.value].tobytes(), r


def relative_l2(a, b) -> float:
    """kernel.hpp:154-163 semantics, in numpy float64."""
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    num = float(np.sum((a - b) ** 2))
    den = float(np.sum(b * b))
    return float(np.sqrt(num)) if den == 0.0 else float(np.sqrt(num / den))
