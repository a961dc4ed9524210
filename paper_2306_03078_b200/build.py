"""Build libspqr_b200.so in-tree (host C++ with g++, kernels with nvcc for sm_100a).

    python -m paper_2306_03078_b200.build [--force] [--verbose]

The .so lands next to this file so it travels with the gpurun snapshot.  No
torch involvement: the library is a plain C ABI over CUDA.
"""
from __future__ import annotations

import argparse
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INC = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "obj")
LIB = os.path.join(PKG, "libspqr_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]
CXXFLAGS = ["-std=c++20", "-O3", "-fPIC", "-ffp-contract=off", "-march=x86-64-v3", "-Wall",
            "-Wno-unused-function", f"-I{INC}", f"-I{CSRC}"]
NVFLAGS = ["-std=c++20", "-O3", "-lineinfo", *GENCODE, "-Xcompiler", "-fPIC,-ffp-contract=off",
           "--fmad=true", f"-I{INC}", f"-I{CSRC}", "-Xptxas", "-warn-spills"]


def _sources():
    cpp = sorted(glob.glob(os.path.join(CSRC, "*.cpp")))
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    hdr = sorted(glob.glob(os.path.join(CSRC, "*.hpp")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                 glob.glob(os.path.join(INC, "*.h")) + glob.glob(os.path.join(INC, "spqr", "*.hpp")))
    return cpp, cu, hdr


def _run(cmd, verbose):
    if verbose:
        print(" ".join(cmd), flush=True)
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if verbose and (r.stdout or r.stderr):
        print(r.stdout + r.stderr)
    return r


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    cpp, cu, hdr = _sources()
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in cpp + cu + hdr)


def build(force: bool = False, verbose: bool = False, ptxas_info: bool = False, out: str | None = None,
          defines: tuple = ()) -> str:
    """Compile the library.  `out`/`defines` build an experimental variant
    (e.g. -DSPQR_MAX_NW=16) next to the default one; the loader picks it up
    through $SPQR_LIB."""
    lib_path = out or LIB
    if not force and out is None and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    cpp, cu, _ = _sources()
    objs = []
    procs = []
    for src in cpp:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        cmd = ["g++", *CXXFLAGS, "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    for src in cu:
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        extra = ["-Xptxas", "-v"] if ptxas_info else []
        cmd = [NVCC, *NVFLAGS, *extra, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True)))
        objs.append(obj)
    failed = False
    for cmd, p in procs:
        out, err = p.communicate()
        if verbose:
            print(" ".join(cmd))
        if p.returncode != 0:
            failed = True
            sys.stderr.write(out + err)
        elif verbose or ptxas_info:
            if out or err:
                print(out + err)
    if failed:
        raise RuntimeError("compilation failed")
    _run([NVCC, *GENCODE, "-shared", "-o", lib_path, *objs, "-lpthread"], verbose)
    return lib_path


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--verbose", action="store_true")
    ap.add_argument("--ptxas-info", action="store_true")
    ap.add_argument("--out")
    ap.add_argument("-D", dest="defines", action="append", default=[])
    a = ap.parse_args()
    print(build(force=a.force, verbose=a.verbose, ptxas_info=a.ptxas_info, out=a.out, defines=tuple(a.defines)))
