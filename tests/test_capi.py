"""The drop-in boundary: the C-ABI library loads, exports every symbol
include/spqr_cuda.h declares, and the C++ drop-in headers compile and work
(format half on CPU; device half under the gpu marker)."""
from __future__ import annotations

import os
import re
import subprocess

import numpy as np
import pytest

import paper_2306_03078_b200 as P

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "spqr_cuda.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spqr_[a-z0-9_]+)\s*\(", src)))


def test_header_symbols_exported():
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (spqr_[a-z0-9_]+)$", out, flags=re.M))
    declared = _declared()
    assert declared, "no declarations parsed"
    missing = [s for s in declared if s not in exported]
    assert not missing, missing
    assert set(P.EXPORTS) <= set(declared)


def test_library_loads_without_gpu():
    L = P.lib()
    assert b"sm_100a" in L.spqr_version()
    assert L.spqr_last_error() == b""


def test_kernels_are_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", P.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _build_cpp(tmp_path, src_name):
    exe = tmp_path / src_name.replace(".cpp", "")
    cmd = ["g++", "-std=c++20", "-O1", f"-I{ROOT}/include", os.path.join(ROOT, "tests", "cpp", src_name),
           "-o", str(exe), f"-L{os.path.dirname(P.LIB_PATH)}", "-lspqr_b200",
           f"-Wl,-rpath,{os.path.dirname(P.LIB_PATH)}"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_dropin_format_api(tmp_path, golden):
    """A caller written against the reference's format.hpp API, recompiled
    against include/spqr/*.hpp, round-trips the golden streams."""
    exe = _build_cpp(tmp_path, "dropin_format.cpp")
    for name in ("base_48x80", "perm_64x96", "ragged_37x53_b8x4_w4_s16_z5"):
        f = tmp_path / f"{name}.spqr"
        f.write_bytes(golden[f"{name}/stream"].tobytes())
        r = subprocess.run([str(exe), str(f), str(tmp_path / "out.spqr")], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        assert (tmp_path / "out.spqr").read_bytes() == f.read_bytes()
    r = subprocess.run([str(exe), str(tmp_path / "missing.spqr"), "x"], capture_output=True, text=True)
    assert r.returncode == 3 and "MissingFile: " in r.stdout


@pytest.mark.gpu
def test_cpp_dropin_kernel_api(tmp_path, golden, cuda):
    exe = _build_cpp(tmp_path, "dropin_kernel.cpp")
    for name in ("base_48x80", "perm_ragged_50x300", "w2_s2_z16_33x70"):
        f = tmp_path / f"{name}.spqr"
        f.write_bytes(golden[f"{name}/stream"].tobytes())
        x = golden[f"{name}/x"][0]
        (tmp_path / "x.bin").write_bytes(x.astype(np.float32).tobytes())
        r = subprocess.run([str(exe), str(f), str(tmp_path / "x.bin"), str(tmp_path / "w.bin"),
                            str(tmp_path / "y.bin")], capture_output=True, text=True)
        assert r.returncode == 0, r.stdout + r.stderr
        w = np.fromfile(tmp_path / "w.bin", np.uint32)
        assert np.array_equal(w, golden[f"{name}/w_bits"].reshape(-1))
        y = np.fromfile(tmp_path / "y.bin", np.float32)
        ref = golden[f"{name}/y"][0]
        assert float(np.linalg.norm(y - ref) / np.linalg.norm(ref)) < 1e-5


def test_gather_api_validates_without_gpu():
    """spqr_gather_create rejects bad world/rank before touching the device
    (the fused all-gather's host-side contract)."""
    import pytest as _pytest

    for world, rank in ((0, 0), (9, 0), (2, 2), (2, -1)):
        with _pytest.raises(P.SpqrError) as e:
            P.Gather(0, 1024, world, rank)
        assert e.value.errc == "config_invalid"
        assert "gather" in str(e.value)
