"""Build recipe of libexm_b200.so (nvcc, sm_100a only) and of the test oracle."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "lib", "libexm_b200.so")
SOURCES = ["exm_kernels.cu", "exm_dynamics.cu", "exm_world.cu", "exm_exact64.cu", "exm_abi.cu"]
HEADERS = ["exm_common.cuh", "exm_device.cuh"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]
# Per-unit flags: the FP64 dynamics round every product and sum separately, as the reference's
# x86-64 build does (no FMA contraction); the FP32 signed-distance kernels fuse explicitly.
UNIT_FLAGS = {"exm_dynamics.cu": ["-fmad=false"], "exm_world.cu": ["-fmad=false"],
              "exm_exact64.cu": ["-fmad=false"]}
# Unit-private headers (a change rebuilds only the units that include them).
UNIT_DEPS = {"exm_dynamics.cu": ["exm_exact64.cuh"], "exm_exact64.cu": ["exm_exact64.cuh"],
             "exm_abi.cu": ["exm_exact64.cuh"]}
# exm_kernels.cu is compiled as this many units (-DEXM_PART=k): its signed-distance kernel
# instantiations (footprint kind x edge count x mode) are split between them and compile in
# parallel. The unit holding the 64-edge polygon (the fully unrolled every-pair kernel of
# config 4) takes ~8.5 minutes, the others under one minute.
KERNEL_PARTS = 4


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_library(force: bool = False, verbose: bool = False, lib: str = LIB,
                  defines: tuple = ()) -> str:
    """Compile the stale objects (source or a shared header newer than the object) in
    parallel, then link when any object changed. `lib` / `defines`: A/B variant builds
    (tools/ab_variants.py: e.g. -DEXM_SDF_RMAJOR into abtest/<name>/libexm_b200.so, selected at
    run time with EXM_LIB_PATH); the product is the default build."""
    from concurrent.futures import ThreadPoolExecutor

    LIB_ = lib
    common = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "exm_b200.h")]
    objdir = os.path.join(os.path.dirname(LIB_), "obj")
    os.makedirs(objdir, exist_ok=True)
    jobs, objs = [], []
    units = []  # (source, object, extra flags): the SDF kernels' instantiations in KERNEL_PARTS
    for src in SOURCES:
        if src == "exm_kernels.cu":
            for k in range(KERNEL_PARTS):
                units.append((src, src.replace(".cu", f"_p{k}.o"),
                              [f"-DEXM_PART={k}", f"-DEXM_NPARTS={KERNEL_PARTS}"]))
        else:
            units.append((src, src.replace(".cu", ".o"), []))
    # the longest compiles first (the kernel parts), so the pool's tail is short
    units.sort(key=lambda u: u[0] != "exm_kernels.cu")
    for src, oname, extra in units:
        obj = os.path.join(objdir, oname)
        objs.append(obj)
        deps = [os.path.join(CSRC, d) for d in UNIT_DEPS.get(src, [])]
        if force or _stale(obj, [os.path.join(CSRC, src), *common, *deps]):
            jobs.append(["nvcc", *NVCC_FLAGS, *UNIT_FLAGS.get(src, []), *extra, *defines, "-c",
                         "-o", obj, os.path.join(CSRC, src)])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)

    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), max(os.cpu_count() or 1, 1))) as ex:
            list(ex.map(run, jobs))
    if force or jobs or _stale(LIB_, objs):
        run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", LIB_, *objs,
             "-ldl"])
    return LIB_


def build_oracle(with_reference: bool | None = None) -> None:
    """Test infrastructure: oracle/lib (C restatement) always; oracle/_ref (the reference's own
    sources) when the reference tree is present (dev container only)."""
    odir = os.path.join(ROOT, "oracle")
    subprocess.run(["make", "-s", "-C", odir, "all"], check=True)
    ref = os.environ.get("REF_DIR", "/root/reference/proj")
    if with_reference is None:
        with_reference = os.path.isdir(os.path.join(ref, "src"))
    if with_reference:
        subprocess.run(["make", "-s", "-C", odir, "ref", "refunit", f"REF_DIR={ref}"], check=True)


def build_dropin() -> None:
    """C++ link-time drop-in demo (needs the reference tree: dev container only)."""
    ref = os.environ.get("REF_DIR", "/root/reference/proj")
    if os.path.isdir(os.path.join(ref, "src")):
        subprocess.run(["make", "-s", "-C", os.path.join(HERE, "host"), f"REF_DIR={ref}", "all",
                        "acceptance", "scaling", "episode", "hybridcheck", "refunit"],
                       check=True)


if __name__ == "__main__":
    build_library(force=True, verbose=True)
    build_oracle()
    build_dropin()
