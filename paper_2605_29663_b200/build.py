"""Build recipe of libexm_b200.so (nvcc, sm_100a only) and of the test oracle."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libexm_b200.so")
SOURCES = ["exm_kernels.cu", "exm_abi.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall", "-shared"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, s) for s in SOURCES] + [
        os.path.join(CSRC, "exm_common.cuh"), os.path.join(ROOT, "include", "exm_b200.h")]
    if force or _stale(LIB, deps):
        os.makedirs(os.path.dirname(LIB), exist_ok=True)
        cmd = ["nvcc", *NVCC_FLAGS, "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES], "-ldl"]
        if verbose:
            print(" ".join(cmd))
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(with_reference: bool | None = None) -> None:
    """Test infrastructure: oracle/lib (C restatement) always; oracle/_ref (the reference's own
    sources) when the reference tree is present (dev container only)."""
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "all"], check=True)
    ref = os.environ.get("REF_DIR", "/root/reference/proj")
    if with_reference is None:
        with_reference = os.path.isdir(os.path.join(ref, "src"))
    if with_reference:
        subprocess.run(["make", "-s", "-C", odir, "ref", f"REF_DIR={ref}"], check=True)


def build_dropin() -> None:
    """C++ link-time drop-in demo (needs the reference tree: dev container only)."""
    ref = os.environ.get("REF_DIR", "/root/reference/proj")
    if os.path.isdir(os.path.join(ref, "src")):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "host"), f"REF_DIR={ref}", "all",
                        "acceptance"], check=True)


if __name__ == "__main__":
    build_library(force=True, verbose=True)
    build_oracle()
    build_dropin()
