"""Build every native artefact in-tree (no cmake, no JIT cache):

* paper_2204_05496_b200/lib/libheinfer_b200.so — the product: sm_100a CUDA +
  the C ABI (nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo).
* oracle/liboracle.so — the C restatement (test infrastructure, gcc).
* oracle/_ref/libheiref.so — the unmodified reference compiled in place,
  only when /root/reference exists (this container, not the GPU box).
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2204_05496_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "lib", "libheinfer_b200.so")
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
    "-diag-suppress", "177",
]
SOURCES = ["heinfer_b200.cu"]


def _nvcc() -> str:
    for c in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_product(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "heinfer_b200.h")]
    if force or _stale(LIB, deps):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES]]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(verbose: bool = False) -> None:
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "all"], check=True)
    if os.path.isdir("/root/reference/proj/src"):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "oracle"), "ref"], check=True)
        if os.path.exists(LIB):  # drop-in parity binary: reference + C++ adapter + product
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "dropin"], check=True)


def build_all(force: bool = False, verbose: bool = False) -> None:
    build_product(force=force, verbose=verbose)
    build_oracle(verbose=verbose)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv, verbose=True)
