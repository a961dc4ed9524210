"""paper_2306_03078_b200 -- B200-native SpQR decode path (y = W x, W in SpQR format).

Python face of the C ABI in include/spqr_cuda.h (libspqr_b200.so, built in-tree
by ``paper_2306_03078_b200.build``).  Mirrors the reference's decode-path API
(/root/reference/proj/include/spqr: format.hpp encode/decode/save/load,
kernel.hpp dequantize_full/matvec) with the same error codes.

There is no CPU fallback: the compute calls launch sm_100a kernels, and the
module raises if the library is missing.  Device buffers are passed as raw
pointers (torch tensors are accepted for convenience: torch is plumbing for
device memory and streams here, never the compute path).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPQR_LIB") or os.path.join(PKG, "libspqr_b200.so")

ERRC = [
    "malformed_header", "shape_mismatch", "non_finite_value", "io_failure", "parse_error",
    "missing_file", "empty_input", "not_positive_definite", "dimension_mismatch",
    "config_invalid", "column_index_overflow", "malformed_stream", "version_unsupported",
    "corrupt_csr", "ill_conditioned", "outlier_budget_exceeded",
]
F16, F32 = 0, 1


class SpqrError(RuntimeError):
    """spqr::Error across the C ABI: .status (1 + Errc) and .errc name."""

    def __init__(self, status: int, msg: str):
        self.status = status
        if 1 <= status <= len(ERRC):
            self.errc = ERRC[status - 1]
        elif status == 100:
            self.errc = "cuda"
        elif status == 101:
            self.errc = "buffer_too_small"
        else:
            self.errc = f"status{status}"
        super().__init__(msg or self.errc)


class LayerInfo(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("weight_bits", C.c_int32),
                ("scale_bits", C.c_int32), ("zero_bits", C.c_int32), ("beta1", C.c_uint32),
                ("beta2", C.c_uint32), ("outlier_count", C.c_uint32), ("flags", C.c_uint32),
                ("has_permutation", C.c_int32), ("tau", C.c_float), ("lambda_rel", C.c_float),
                ("payload_bytes", C.c_uint64), ("device_bytes", C.c_uint64),
                ("fast_path", C.c_int32), ("device", C.c_int32)]

    def as_dict(self) -> dict:
        return {k: getattr(self, k) for k, _ in self._fields_}


class LayoutSpec(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("weight_bits", C.c_int32),
                ("scale_bits", C.c_int32), ("zero_bits", C.c_int32), ("beta1", C.c_uint32),
                ("beta2", C.c_uint32), ("outlier_count", C.c_uint32), ("has_permutation", C.c_int32)]


class TensorArrays(C.Structure):
    _fields_ = [("rows", C.c_uint32), ("cols", C.c_uint32), ("weight_bits", C.c_int32),
                ("scale_bits", C.c_int32), ("zero_bits", C.c_int32), ("beta1", C.c_uint32),
                ("beta2", C.c_uint32), ("flags", C.c_uint32), ("tau", C.c_float),
                ("lambda_rel", C.c_float), ("order", C.c_void_p), ("codes", C.c_void_p),
                ("scale_codes", C.c_void_p), ("zero_codes", C.c_void_p), ("raw_scales", C.c_void_p),
                ("raw_zeros", C.c_void_p), ("group_scalars", C.c_void_p),
                ("outlier_count", C.c_uint32), ("outlier_rows", C.c_void_p),
                ("outlier_cols", C.c_void_p), ("outlier_vals", C.c_void_p)]


class EncoderCfg(C.Structure):
    _fields_ = [("weight_bits", C.c_int32), ("scale_bits", C.c_int32), ("zero_bits", C.c_int32),
                ("beta1", C.c_uint32), ("beta2", C.c_uint32), ("order", C.c_int32), ("act_order_key", C.c_int32),
                ("outliers_enabled", C.c_int32), ("integer_zero", C.c_int32), ("full_range_sign", C.c_int32),
                ("tau", C.c_double), ("lambda_rel", C.c_double), ("seed", C.c_uint64)]


class LayerOpts(C.Structure):
    _fields_ = [("device", C.c_int32), ("force_generic", C.c_int32), ("keep_stream", C.c_int32),
                ("row_begin", C.c_uint32), ("row_end", C.c_uint32), ("host_transcode", C.c_int32)]


_lib = None

# every symbol include/spqr_cuda.h declares (tests check the .so exports them)
EXPORTS = [
    "spqr_last_error", "spqr_version", "spqr_stream_validate", "spqr_decode_arrays",
    "spqr_encode_arrays", "spqr_payload_bytes", "spqr_estimate_avg_bits",
    "spqr_measure_actual_bits", "spqr_stream_slice_rows", "spqr_transcode_roundtrip_host",
    "spqr_layer_create", "spqr_layer_destroy", "spqr_layer_get_info", "spqr_layer_export_stream",
    "spqr_layer_set_exact", "spqr_dequantize", "spqr_workspace_bytes", "spqr_matvec", "spqr_matvec_ws", "spqr_matvec_host",
    "spqr_dense_gemv_f16", "spqr_last_launch_count", "spqr_debug_tiled_host",
    "spqr_matvec_stage", "spqr_bench_layer", "spqr_dev_alloc", "spqr_dev_free",
    "spqr_dev_copy_to_host", "spqr_dev_copy_to_device",
]


def lib() -> C.CDLL:
    """Load libspqr_b200.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2306_03078_b200.build`")
    L = C.CDLL(LIB_PATH)
    vp, sz, u32, i32 = C.c_void_p, C.c_size_t, C.c_uint32, C.c_int
    sig = {
        "spqr_last_error": (C.c_char_p, []),
        "spqr_version": (C.c_char_p, []),
        "spqr_stream_validate": (i32, [vp, sz, C.POINTER(LayerInfo)]),
        "spqr_decode_arrays": (i32, [vp, sz, C.POINTER(TensorArrays)]),
        "spqr_encode_arrays": (i32, [C.POINTER(TensorArrays), vp, sz, C.POINTER(C.c_size_t)]),
        "spqr_payload_bytes": (C.c_uint64, [C.POINTER(LayoutSpec)]),
        "spqr_estimate_avg_bits": (i32, [i32, i32, i32, u32, u32, C.c_double, vp]),
        "spqr_measure_actual_bits": (i32, [vp, sz, vp]),
        "spqr_stream_slice_rows": (i32, [vp, sz, u32, u32, vp, sz, C.POINTER(C.c_size_t)]),
        "spqr_transcode_roundtrip_host": (i32, [vp, sz, vp, sz, C.POINTER(C.c_size_t)]),
        "spqr_layer_create": (i32, [vp, sz, C.POINTER(LayerOpts), C.POINTER(vp)]),
        "spqr_layer_destroy": (None, [vp]),
        "spqr_layer_create_stacked": (i32, [C.POINTER(vp), C.POINTER(sz), i32, C.POINTER(LayerOpts), C.POINTER(vp)]),
        "spqr_debug_layer_cells": (i32, [vp, vp, sz, C.POINTER(C.c_size_t), vp]),
        "spqr_layer_get_info": (i32, [vp, C.POINTER(LayerInfo)]),
        "spqr_layer_set_exact": (i32, [vp, i32]),
        "spqr_layer_export_stream": (i32, [vp, vp, sz, C.POINTER(C.c_size_t)]),
        "spqr_dequantize": (i32, [vp, vp, vp]),
        "spqr_workspace_bytes": (C.c_uint64, [vp, i32]),
        "spqr_matvec": (i32, [vp, vp, i32, vp, i32, vp]),
        "spqr_matvec_ws": (i32, [vp, vp, i32, vp, i32, vp, C.c_uint64, vp]),
        "spqr_matvec_host": (i32, [vp, vp, vp, i32]),
        "spqr_dense_gemv_f16": (i32, [vp, vp, vp, u32, u32, vp]),
        "spqr_last_launch_count": (i32, []),
        "spqr_debug_tiled_host": (i32, [vp, sz, vp, vp, vp, vp]),
        "spqr_matvec_stage": (i32, [vp, vp, i32, vp, i32, i32, vp]),
        "spqr_bench_layer": (i32, [vp, i32, vp]),
        "spqr_gather_create": (i32, [i32, u32, i32, i32, C.POINTER(vp)]),
        "spqr_gather_handle": (i32, [vp, vp]),
        "spqr_gather_open": (i32, [vp, vp, vp]),
        "spqr_gather_y": (vp, [vp]),
        "spqr_matvec_gather": (i32, [vp, vp, i32, vp, vp]),
        "spqr_gather_wait": (i32, [vp, vp]),
        "spqr_gather_destroy": (None, [vp]),
        "spqr_row_bands": (i32, [u32, u32, i32, vp]),
        "spqr_hessian_create": (i32, [u32, i32, C.POINTER(vp)]),
        "spqr_hessian_accumulate": (i32, [vp, vp, u32, vp]),
        "spqr_hessian_read": (i32, [vp, vp]),
        "spqr_hessian_destroy": (None, [vp]),
        "spqr_quantize_layer": (i32, [vp, vp, u32, C.POINTER(EncoderCfg), vp, sz, C.POINTER(C.c_size_t), vp]),
        "spqr_quantize_layer_tuned": (i32, [vp, vp, u32, C.POINTER(EncoderCfg), C.c_double, vp, sz,
                                            C.POINTER(C.c_size_t), vp]),
        "spqr_nccl_unique_id": (i32, [vp]),
        "spqr_nccl_comm_init": (i32, [vp, i32, i32, i32, C.POINTER(vp)]),
        "spqr_nccl_comm_destroy": (i32, [vp]),
        "spqr_sharded_create": (i32, [C.POINTER(vp), C.POINTER(sz), i32, i32, i32, vp, C.POINTER(LayerOpts),
                                      C.POINTER(vp)]),
        "spqr_sharded_band": (i32, [vp, C.POINTER(u32), C.POINTER(u32), C.POINTER(u32), C.POINTER(vp)]),
        "spqr_sharded_matvec": (i32, [vp, vp, i32, vp, i32, vp]),
        "spqr_sharded_destroy": (None, [vp]),
        "spqr_dev_alloc": (i32, [C.POINTER(vp), sz]),
        "spqr_dev_free": (None, [vp]),
        "spqr_dev_copy_to_host": (i32, [vp, vp, sz]),
        "spqr_dev_copy_to_device": (i32, [vp, vp, sz]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L


def _check(rc: int) -> None:
    if rc:
        raise SpqrError(rc, lib().spqr_last_error().decode())


def _buf(stream: bytes):
    a = np.frombuffer(stream, dtype=np.uint8)
    return a, a.ctypes.data_as(C.c_void_p), a.size


def _ptr(x):
    """Raw pointer of a torch tensor / numpy array / int."""
    if x is None:
        return None
    if isinstance(x, int):
        return C.c_void_p(x)
    if hasattr(x, "data_ptr"):
        return C.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        return x.ctypes.data_as(C.c_void_p)
    raise TypeError(type(x))


def _stream_ptr(stream):
    if stream is None:
        return None
    if hasattr(stream, "cuda_stream"):
        return C.c_void_p(stream.cuda_stream)
    return C.c_void_p(int(stream))


# ---------------------------------------------------------------- format --
def validate(stream: bytes) -> dict:
    """decode()'s validation (format.hpp:354-500); returns the header info."""
    _, p, n = _buf(stream)
    info = LayerInfo()
    _check(lib().spqr_stream_validate(p, n, C.byref(info)))
    return info.as_dict()


def decode_arrays(stream: bytes) -> dict:
    """decode() (format.hpp:354) into flat numpy arrays (SpqrTensor fields)."""
    info = validate(stream)
    m, n = info["rows"], info["cols"]
    nb = (n + info["beta1"] - 1) // info["beta1"]
    ng = (m + info["beta2"] - 1) // info["beta2"]
    sb, zb = info["scale_bits"], info["zero_bits"]
    out = {
        "order": np.zeros(n, np.uint32), "codes": np.zeros(m * n, np.uint8),
        "scale_codes": np.zeros(nb * m, np.uint8) if sb != 16 else None,
        "zero_codes": np.zeros(nb * m, np.uint8) if zb != 16 else None,
        "raw_scales": np.zeros(nb * m, np.float32) if sb == 16 else None,
        "raw_zeros": np.zeros(nb * m, np.float32) if zb == 16 else None,
        "group_scalars": np.zeros(nb * ng * 4, np.uint16) if (sb != 16 or zb != 16) else None,
        "outlier_rows": np.zeros(info["outlier_count"], np.uint32),
        "outlier_cols": np.zeros(info["outlier_count"], np.uint32),
        "outlier_vals": np.zeros(info["outlier_count"], np.uint16),
    }
    ta = TensorArrays()
    for k, v in out.items():
        setattr(ta, k, None if v is None else v.ctypes.data)
    _, p, nn = _buf(stream)
    _check(lib().spqr_decode_arrays(p, nn, C.byref(ta)))
    for k in ("rows", "cols", "weight_bits", "scale_bits", "zero_bits", "beta1", "beta2", "flags",
              "tau", "lambda_rel"):
        out[k] = getattr(ta, k)
    if not (out["flags"] & 1):
        out["order"] = None
    out["flags"] &= ~1
    return out


def encode_arrays(a: dict) -> bytes:
    """encode() (format.hpp:269) of a tensor given as flat arrays."""
    keep = {}

    def arr(key, dt):
        v = a.get(key)
        if v is None:
            return None
        keep[key] = np.ascontiguousarray(v, dtype=dt)
        return keep[key].ctypes.data

    ta = TensorArrays(rows=a["rows"], cols=a["cols"], weight_bits=a["weight_bits"],
                      scale_bits=a["scale_bits"], zero_bits=a["zero_bits"], beta1=a["beta1"],
                      beta2=a["beta2"], flags=a.get("flags", 0x18), tau=a.get("tau", 0.0),
                      lambda_rel=a.get("lambda_rel", 0.0))
    ta.order = arr("order", np.uint32)
    ta.codes = arr("codes", np.uint8)
    ta.scale_codes = arr("scale_codes", np.uint8)
    ta.zero_codes = arr("zero_codes", np.uint8)
    ta.raw_scales = arr("raw_scales", np.float32)
    ta.raw_zeros = arr("raw_zeros", np.float32)
    ta.group_scalars = arr("group_scalars", np.uint16)
    ta.outlier_rows = arr("outlier_rows", np.uint32)
    ta.outlier_cols = arr("outlier_cols", np.uint32)
    ta.outlier_vals = arr("outlier_vals", np.uint16)
    ta.outlier_count = int(np.asarray(a["outlier_rows"]).size)
    n = C.c_size_t()
    rc = lib().spqr_encode_arrays(C.byref(ta), None, 0, C.byref(n))
    if rc not in (0, 101):
        _check(rc)
    out = np.empty(n.value, np.uint8)
    _check(lib().spqr_encode_arrays(C.byref(ta), out.ctypes.data_as(C.c_void_p), out.size, C.byref(n)))
    return out.tobytes()


def payload_bytes(rows, cols, weight_bits, scale_bits, zero_bits, beta1, beta2, outlier_count,
                  has_permutation) -> int:
    """stream_payload_bytes (layout.hpp:47-64): the algorithmic bytes."""
    ls = LayoutSpec(rows, cols, weight_bits, scale_bits, zero_bits, beta1, beta2, outlier_count,
                    int(bool(has_permutation)))
    return int(lib().spqr_payload_bytes(C.byref(ls)))


def estimate_avg_bits(b_w, b_s, b_z, beta1, beta2, r_o) -> np.ndarray:
    out = np.zeros(5, np.float64)
    _check(lib().spqr_estimate_avg_bits(b_w, b_s, b_z, beta1, beta2, r_o, out.ctypes.data_as(C.c_void_p)))
    return out


def measure_actual_bits(stream: bytes) -> np.ndarray:
    out = np.zeros(3, np.float64)
    _, p, n = _buf(stream)
    _check(lib().spqr_measure_actual_bits(p, n, out.ctypes.data_as(C.c_void_p)))
    return out


def _sized_call(f, *args) -> bytes:
    n = C.c_size_t()
    rc = f(*args, None, 0, C.byref(n))
    if rc not in (0, 101):
        _check(rc)
    out = np.empty(max(n.value, 1), np.uint8)
    _check(f(*args, out.ctypes.data_as(C.c_void_p), out.size, C.byref(n)))
    return out[: n.value].tobytes()


def slice_rows(stream: bytes, r0: int, r1: int) -> bytes:
    """Rows [r0, r1) as a standalone stream (row-sharding helper)."""
    a, p, n = _buf(stream)
    return _sized_call(lib().spqr_stream_slice_rows, p, n, r0, r1)


def transcode_roundtrip_host(stream: bytes) -> bytes:
    a, p, n = _buf(stream)
    return _sized_call(lib().spqr_transcode_roundtrip_host, p, n)


def debug_tiled_host(stream: bytes) -> dict:
    """The tiled HBM image (host copy) -- test hook for the kernel model."""
    a, p, n = _buf(stream)
    dims = np.zeros(4, np.uint32)
    _check(lib().spqr_debug_tiled_host(p, n, dims.ctypes.data_as(C.c_void_p), None, None, None))
    Gn, Pn, cb, total = (int(v) for v in dims)
    cells = np.zeros(total, np.uint8)
    off = np.zeros(Gn * Pn + 1, np.uint32)
    _check(lib().spqr_debug_tiled_host(p, n, dims.ctypes.data_as(C.c_void_p), cells.ctypes.data_as(C.c_void_p),
                                       off.ctypes.data_as(C.c_void_p), None))
    return {"Gn": Gn, "Pn": Pn, "cell_bytes": cb, "cells": cells, "cell_off": off}


# ---------------------------------------------------------------- device --
class Layer:
    """A layer resident in HBM (spqr_layer_create: decode + plan + upload)."""

    def __init__(self, stream: bytes, device: int = -1, force_generic: bool = False,
                 rows: tuple[int, int] | None = None, host_transcode: bool = False, keep_stream: bool = False):
        a, p, n = _buf(stream)
        opts = LayerOpts(device=device, force_generic=int(force_generic), keep_stream=int(keep_stream),
                         row_begin=rows[0] if rows else 0, row_end=rows[1] if rows else 0,
                         host_transcode=int(host_transcode))
        h = C.c_void_p()
        _check(lib().spqr_layer_create(p, n, C.byref(opts), C.byref(h)))
        self._h = h
        info = LayerInfo()
        _check(lib().spqr_layer_get_info(h, C.byref(info)))
        self.info = info.as_dict()
        self.rows, self.cols = self.info["rows"], self.info["cols"]

    @classmethod
    def stacked(cls, streams: list, device: int = -1, host_transcode: bool = False) -> "Layer":
        """Several layers sharing their input (q/k/v, gate/up) stacked row-wise
        in one handle (spqr_layer_create_stacked): one launch, y = [y_0; y_1; ...]."""
        bufs = [_buf(s) for s in streams]
        ptrs = (C.c_void_p * len(bufs))(*[b[1] for b in bufs])
        sizes = (C.c_size_t * len(bufs))(*[b[2] for b in bufs])
        opts = LayerOpts(device=device, force_generic=0, keep_stream=0, row_begin=0, row_end=0,
                         host_transcode=int(host_transcode))
        h = C.c_void_p()
        _check(lib().spqr_layer_create_stacked(ptrs, sizes, len(bufs), C.byref(opts), C.byref(h)))
        self = cls.__new__(cls)
        self._h = h
        info = LayerInfo()
        _check(lib().spqr_layer_get_info(h, C.byref(info)))
        self.info = info.as_dict()
        self.rows, self.cols = self.info["rows"], self.info["cols"]
        return self

    def close(self):
        if getattr(self, "_owner", None) is not None:  # a view of a handle owned elsewhere
            self._h = self._owner = None
        if getattr(self, "_h", None):
            lib().spqr_layer_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self):
        return self._h

    @property
    def exact(self) -> bool:
        """Batched-decode precision mode (spqr_layer_set_exact): False (default)
        runs batch >= 5 on gemm_tc (fp16 weights, ~1e-4), True keeps every
        batch on exact-code kernels (gemv_cta pairs, gemm_bm / gemm_ex for batch >= 7)."""
        return getattr(self, "_exact", False)

    @exact.setter
    def exact(self, on: bool) -> None:
        _check(lib().spqr_layer_set_exact(self._h, int(bool(on))))
        self._exact = bool(on)

    def matvec(self, x, y, batch: int = 1, stream=None, workspace=None) -> None:
        """y (batch x rows, fp32, device) = W x (batch x cols, f16/f32, device)."""
        dt = F16 if str(getattr(x, "dtype", "")).endswith("float16") else F32
        if workspace is None:
            _check(lib().spqr_matvec(self._h, _ptr(x), dt, _ptr(y), batch, _stream_ptr(stream)))
        else:
            _check(lib().spqr_matvec_ws(self._h, _ptr(x), dt, _ptr(y), batch, _ptr(workspace),
                                        workspace.numel() * workspace.element_size(), _stream_ptr(stream)))

    def matvec_stage(self, x, y, stage: int, batch: int = 1, stream=None) -> None:
        """Launch only the x preparation (1), only the fused product (2), or both (0)."""
        dt = F16 if str(getattr(x, "dtype", "")).endswith("float16") else F32
        _check(lib().spqr_matvec_stage(self._h, _ptr(x), dt, _ptr(y), batch, stage, _stream_ptr(stream)))

    def bench(self, repeats: int = 20) -> np.ndarray:
        """ns per op: fused matvec, dequantize_full, dense fp16 GEMV (CUDA events)."""
        out = np.zeros(3, np.float64)
        _check(lib().spqr_bench_layer(self._h, repeats, out.ctypes.data_as(C.c_void_p)))
        return out

    def matvec_host(self, x: np.ndarray, out: np.ndarray | None = None) -> np.ndarray:
        """Drop-in matvec(t, x) with host buffers (kernel.hpp:126).  Page-locked
        x / out (e.g. numpy views of pinned torch tensors) are copied directly;
        pageable ones go through the layer's pinned staging."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        batch = x.size // self.cols
        y = np.empty(batch * self.rows, np.float32) if out is None else out
        if y.dtype != np.float32 or not y.flags.c_contiguous or y.size != batch * self.rows:
            raise ValueError("out must be a contiguous float32 array of batch * rows elements")
        # raw addresses through __array_interface__ (ndarray.ctypes costs ~1 us per access)
        rc = _lib.spqr_matvec_host(self._h, x.__array_interface__["data"][0], y.__array_interface__["data"][0],
                                   batch)
        if rc:
            _check(rc)
        return y.reshape(batch, self.rows) if batch > 1 else y

    def host_call(self, x: np.ndarray, out: np.ndarray):
        """matvec_host(x, out) bound to these two buffers: a zero-argument
        callable for decode loops that refill the same (page-locked) x and read
        the same y every step -- the argument checks and pointer lookups run
        once here, not per call.  x and out must be contiguous float32 arrays
        that outlive the callable."""
        for a, what in ((x, "x"), (out, "out")):
            if not isinstance(a, np.ndarray) or a.dtype != np.float32 or not a.flags.c_contiguous:
                raise ValueError(f"{what} must be a contiguous float32 ndarray")
        batch = x.size // self.cols
        if batch < 1 or x.size != batch * self.cols or out.size != batch * self.rows:
            raise ValueError("x must hold batch * cols and out batch * rows elements")
        fn, h = _lib.spqr_matvec_host, self._h
        xa, ya = x.__array_interface__["data"][0], out.__array_interface__["data"][0]

        def call() -> None:
            rc = fn(h, xa, ya, batch)
            if rc:
                _check(rc)

        call.buffers = (x, out)  # keep the arrays alive with the callable
        return call

    def dequantize(self, w, stream=None) -> None:
        """dequantize_full (kernel.hpp:17) into a rows x cols fp32 device buffer."""
        _check(lib().spqr_dequantize(self._h, _ptr(w), _stream_ptr(stream)))

    def debug_cells(self) -> dict:
        """The device-resident cell records and record offsets (test hook)."""
        n = C.c_size_t()
        ncell = ((self.rows + 31) // 32) * ((self.cols + 255) // 256)
        off = np.zeros(ncell + 1, np.uint32)
        _check(lib().spqr_debug_layer_cells(self._h, None, 0, C.byref(n), off.ctypes.data_as(C.c_void_p)))
        cells = np.zeros(n.value, np.uint8)
        _check(lib().spqr_debug_layer_cells(self._h, cells.ctypes.data_as(C.c_void_p), n.value, C.byref(n), None))
        return {"cells": cells, "cell_off": off}

    def workspace_bytes(self, batch: int = 1) -> int:
        return int(lib().spqr_workspace_bytes(self._h, batch))

    def export_stream(self) -> bytes:
        return _sized_call(lib().spqr_layer_export_stream, self._h)


GATHER_HANDLE_BYTES = 64


class Gather:
    """Full-y target of the fused all-gather (spqr_gather_*): every rank's
    band matvec stores its rows into every rank's buffer over P2P and signals
    a per-rank round counter; wait() blocks the stream until all ranks'
    rows of this round have landed."""

    def __init__(self, device: int, rows: int, world: int, rank: int):
        h = C.c_void_p()
        _check(lib().spqr_gather_create(device, rows, world, rank, C.byref(h)))
        self._h, self.rows, self.world, self.rank = h, rows, world, rank

    def handle(self) -> bytes:
        buf = (C.c_uint8 * GATHER_HANDLE_BYTES)()
        _check(lib().spqr_gather_handle(self._h, buf))
        return bytes(buf)

    def open(self, handles: list, row_base: list) -> None:
        """handles[j] = rank j's handle() bytes; row_base[j] = first row of rank j's band."""
        hb = b"".join(handles)
        rb = np.ascontiguousarray(row_base, dtype=np.uint32)
        _check(lib().spqr_gather_open(self._h, C.c_char_p(hb), rb.ctypes.data_as(C.c_void_p)))

    def y_ptr(self) -> int:
        return int(lib().spqr_gather_y(self._h))

    def matvec(self, layer: "Layer", x, stream=None) -> None:
        dt = F16 if str(getattr(x, "dtype", "")).endswith("float16") else F32
        _check(lib().spqr_matvec_gather(layer.handle, _ptr(x), dt, self._h, _stream_ptr(stream)))

    def wait(self, stream=None) -> None:
        _check(lib().spqr_gather_wait(self._h, _stream_ptr(stream)))

    def close(self):
        if getattr(self, "_h", None):
            lib().spqr_gather_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Hessian:
    """H = 2 X X^T accumulated on the GPU in binary64 (spqr_hessian_*,
    hessian.hpp:52-85); quantize() runs the GPU encoder against it."""

    def __init__(self, n: int, device: int = -1):
        h = C.c_void_p()
        _check(lib().spqr_hessian_create(n, device, C.byref(h)))
        self._h, self.n = h, n

    def accumulate(self, x, stream=None) -> None:
        """x: n x samples fp32 on the device (calibration inputs, one column per sample)."""
        if x.dim() != 2 or x.shape[0] != self.n:
            raise ValueError("x must be n x samples")
        _check(lib().spqr_hessian_accumulate(self._h, _ptr(x.contiguous()), x.shape[1], _stream_ptr(stream)))

    def matrix(self) -> np.ndarray:
        out = np.empty((self.n, self.n), np.float64)
        _check(lib().spqr_hessian_read(self._h, out.ctypes.data_as(C.c_void_p)))
        return out

    def quantize(self, w, weight_bits=3, scale_bits=3, zero_bits=3, beta1=16, beta2=16, order="natural",
                 act_order_key="hessian_diag", outliers=True, integer_zero=False, full_range_sign=True,
                 tau=0.1, lambda_rel=0.01, seed=0, target_rate=None):
        """spqr_quantize + encode on the GPU: (stream bytes, report dict).
        target_rate: tune_tau (solver.hpp:546) instead of a fixed tau."""
        cfg = EncoderCfg(weight_bits, scale_bits, zero_bits, beta1, beta2,
                         {"natural": 0, "act_order": 1, "shuffled": 2}[order],
                         {"hessian_diag": 0, "inverse_diag": 1}[act_order_key], int(outliers), int(integer_zero),
                         int(full_range_sign), float(tau), float(lambda_rel), int(seed))
        w = w.contiguous()
        m = w.shape[0]
        rep = np.zeros(3, np.float64)
        n = C.c_size_t()
        # upper bound of the stream: header, permutation, records with 16-bit
        # statistics, CSR with the 5 % outlier cap
        nb, ng = -(-self.n // beta1), -(-m // beta2)
        cap = 48 + 4 * self.n + nb * ng * (8 + 8 * beta2 + beta1 * beta2) + 4 * (m + 1) + 4 * (m * self.n // 20 + 1)
        buf = np.empty(cap, np.uint8)
        if target_rate is not None:
            rep = np.zeros(5, np.float64)
            _check(lib().spqr_quantize_layer_tuned(self._h, _ptr(w), m, C.byref(cfg), float(target_rate),
                                                   buf.ctypes.data_as(C.c_void_p), buf.size, C.byref(n),
                                                   rep.ctypes.data_as(C.c_void_p)))
            return buf[: n.value].tobytes(), {"relative_error": float(rep[0]), "outlier_rate": float(rep[1]),
                                              "bits_per_param": float(rep[2]), "tau": float(rep[3]),
                                              "target_reached": bool(rep[4])}
        _check(lib().spqr_quantize_layer(self._h, _ptr(w), m, C.byref(cfg), buf.ctypes.data_as(C.c_void_p),
                                         buf.size, C.byref(n), rep.ctypes.data_as(C.c_void_p)))
        return buf[: n.value].tobytes(), {"relative_error": float(rep[0]), "outlier_rate": float(rep[1]),
                               "bits_per_param": float(rep[2])}

    def close(self):
        if getattr(self, "_h", None):
            lib().spqr_hessian_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


NCCL_ID_BYTES = 128


def c_row_bands(rows: int, beta2: int, world: int) -> list[tuple[int, int]]:
    """The C ABI's band edges (spqr_row_bands; sharded.row_bands is the same rule)."""
    e = np.zeros(world + 1, np.uint32)
    _check(lib().spqr_row_bands(rows, beta2, world, e.ctypes.data_as(C.c_void_p)))
    return [(int(e[i]), int(e[i + 1])) for i in range(world)]


def nccl_unique_id() -> bytes:
    """ncclGetUniqueId through the C ABI (spqr_nccl_unique_id): broadcast the
    bytes to every rank by any transport, then NcclComm(id, world, rank)."""
    buf = (C.c_uint8 * NCCL_ID_BYTES)()
    _check(lib().spqr_nccl_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """An NCCL communicator created through the C ABI (spqr_nccl_comm_init)."""

    def __init__(self, uid: bytes, world: int, rank: int, device: int):
        h = C.c_void_p()
        _check(lib().spqr_nccl_comm_init(C.c_char_p(uid), world, rank, device, C.byref(h)))
        self._h, self.world, self.rank, self.device = h, world, rank, device

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            _check(lib().spqr_nccl_comm_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class ShardedNccl:
    """This rank's row band of one layer (or of layers stacked row-wise) plus
    the NCCL all-gather of y, entirely behind the C ABI (spqr_sharded_*):
    matvec(x, y) leaves the full y (batch x rows) on every rank."""

    def __init__(self, streams, comm: NcclComm, device: int = -1):
        streams = [streams] if isinstance(streams, (bytes, bytearray)) else list(streams)
        bufs = [_buf(s) for s in streams]
        ptrs = (C.c_void_p * len(bufs))(*[b[1] for b in bufs])
        sizes = (C.c_size_t * len(bufs))(*[b[2] for b in bufs])
        opts = LayerOpts(device=device, force_generic=0, keep_stream=0, row_begin=0, row_end=0, host_transcode=0)
        h = C.c_void_p()
        _check(lib().spqr_sharded_create(ptrs, sizes, len(bufs), comm.rank, comm.world, comm.handle,
                                         C.byref(opts), C.byref(h)))
        self._h, self.comm = h, comm
        rows, a, b = C.c_uint32(), C.c_uint32(), C.c_uint32()
        _check(lib().spqr_sharded_band(h, C.byref(rows), C.byref(a), C.byref(b), None))
        self.rows, self.band = rows.value, (a.value, b.value)

    def band_layer(self) -> "Layer":
        """This rank's band as a Layer view (owned by this handle: valid while it lives)."""
        h = C.c_void_p()
        _check(lib().spqr_sharded_band(self._h, None, None, None, C.byref(h)))
        L = Layer.__new__(Layer)
        L._h, L._owner = h, self
        info = LayerInfo()
        _check(lib().spqr_layer_get_info(h, C.byref(info)))
        L.info = info.as_dict()
        L.rows, L.cols = L.info["rows"], L.info["cols"]
        return L

    def matvec(self, x, y, batch: int = 1, stream=None) -> None:
        dt = F16 if str(getattr(x, "dtype", "")).endswith("float16") else F32
        _check(lib().spqr_sharded_matvec(self._h, _ptr(x), dt, _ptr(y), batch, _stream_ptr(stream)))

    def close(self):
        if getattr(self, "_h", None):
            lib().spqr_sharded_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def dense_gemv_f16(w, x, y, rows: int, cols: int, stream=None) -> None:
    _check(lib().spqr_dense_gemv_f16(_ptr(w), _ptr(x), _ptr(y), rows, cols, _stream_ptr(stream)))


def last_launch_count() -> int:
    return int(lib().spqr_last_launch_count())
