"""Build the in-tree CUDA library libglsgpu.so for sm_100a (nvcc, no JIT cache, no torch extension).

    python -m paper_2510_14471_b200.build

Flags: -gencode arch=compute_100a,code=sm_100a, -lineinfo (ncu source view), -fmad=false (no FMA
contraction: the element-wise updates round as the reference's x86-64 build).
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libglsgpu.so")
SOURCES = [os.path.join(CSRC, "glsgpu.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("kernels.cuh", "ne.cuh", "gemm.cuh", "cqr.cuh")] + [
    os.path.join(ROOT, "include", "glsgpu.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-fmad=false",
    "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr",
]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return LIB
    cmd = [NVCC, *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB, *SOURCES]
    p = subprocess.run(cmd, capture_output=True, text=True)
    if verbose or p.returncode != 0:
        sys.stderr.write(p.stdout + p.stderr)
    if p.returncode != 0:
        raise RuntimeError(f"nvcc failed ({p.returncode}): {' '.join(cmd)}")
    with open(os.path.join(PKG, "ptxas_report.txt"), "w") as f:
        f.write(p.stderr)
    return LIB


CPP_TESTS = os.path.join(ROOT, "tests", "cpp")
REF_INCLUDE = "/root/reference/proj/include"


CPP_DEPS = [os.path.join(ROOT, "include", "glsgpu.h"), os.path.join(ROOT, "include", "gls_b200", "gls_b200.hpp"),
            os.path.join(ROOT, "integration", "gls_gpu_adapter.hpp"), os.path.join(CPP_TESTS, "test_header_api.cpp"),
            os.path.join(CPP_TESTS, "test_reference_adapter.cpp"), os.path.join(ROOT, "include", "gls_b200", "io.hpp"),
            os.path.join(CPP_TESTS, "test_io.cpp"), os.path.join(CPP_TESTS, "ref_io.cpp")]


def cpp_deps_digest() -> str:
    """Content hash of the headers / sources the C++ test binaries are compiled from."""
    import hashlib
    h = hashlib.sha256()
    for d in CPP_DEPS:
        h.update(open(d, "rb").read() if os.path.exists(d) else b"-")
    return h.hexdigest()


def build_cpp_tests(verbose: bool = False) -> list:
    """The C++ host-API test (always) and the reference-adapter test (when the reference headers are
    present -- i.e. here, not on the GPU box; the binary travels).  rpath $ORIGIN-relative so the
    binaries find libglsgpu.so / the oracle libraries inside the snapshot."""
    out = os.path.join(CPP_TESTS, "bin")
    os.makedirs(out, exist_ok=True)
    rpath = "-Wl,-rpath,$ORIGIN/../../../paper_2510_14471_b200:$ORIGIN/../../../oracle:$ORIGIN/../../../oracle/_ref"
    cmds = [[
        "g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(CPP_TESTS, "test_header_api.cpp"),
        "-L", PKG, "-lglsgpu", "-L", os.path.join(ROOT, "oracle"), "-loracle", rpath,
        "-o", os.path.join(out, "test_header_api"),
    ]]
    cmds.append([
        "g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(CPP_TESTS, "test_io.cpp"),
        "-L", PKG, "-lglsgpu", rpath, "-o", os.path.join(out, "test_io"),
    ])
    if os.path.isdir(REF_INCLUDE) and os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libglsref.so")):
        cmds.append([
            "g++", "-std=c++20", "-O2", "-I", REF_INCLUDE, os.path.join(CPP_TESTS, "ref_io.cpp"),
            "-L", os.path.join(ROOT, "oracle", "_ref"), "-lglsref", rpath, "-o", os.path.join(out, "ref_io"),
        ])
        cmds.append([
            "g++", "-std=c++20", "-O2", "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "include"), "-I",
            os.path.join(ROOT, "integration"), os.path.join(CPP_TESTS, "test_reference_adapter.cpp"),
            "-L", os.path.join(ROOT, "oracle", "_ref"), "-lglsref", "-L", PKG, "-lglsgpu", rpath,
            "-o", os.path.join(out, "test_reference_adapter"),
        ])
    built = []
    for cmd in cmds:
        p = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or p.returncode != 0:
            sys.stderr.write(p.stdout + p.stderr)
        if p.returncode != 0:
            raise RuntimeError(f"g++ failed: {' '.join(cmd)}")
        built.append(cmd[cmd.index("-o") + 1])
    with open(os.path.join(out, "deps.sha256"), "w") as f:
        f.write(cpp_deps_digest())
    return built


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(LIB)
