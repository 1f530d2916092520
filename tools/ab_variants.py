"""A/B variant builds of libexm_b200.so and an interleaved benchmark over them.

  python tools/ab_variants.py build NAME=-DFLAG[,-DFLAG2] ...      (here: nvcc cross-compiles)
  python tools/ab_variants.py bench CFG ROUNDS NAME ...            (on the GPU box)

Variants live in abtest/<NAME>/libexm_b200.so; `base` is the product build. The benchmark runs
bench.py once per variant per round (EXM_LIB_PATH selects the library) and prints device
ms/step, SDF ms and e2e steps/s of each."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def lib_of(name):
    if name == "base":
        return os.path.join(ROOT, "paper_2605_29663_b200", "lib", "libexm_b200.so")
    return os.path.join(ROOT, "abtest", name, "libexm_b200.so")


def build(specs):
    from paper_2605_29663_b200 import build as b
    for spec in specs:
        name, _, flags = spec.partition("=")
        defines = tuple(f for f in flags.split(",") if f)
        os.makedirs(os.path.join(ROOT, "abtest", name), exist_ok=True)
        b.build_library(lib=lib_of(name), defines=defines)
        print("built", name, defines)


def bench(cfg, rounds, names, extra=()):
    os.makedirs(os.path.join(ROOT, "gpurun_out", "ab"), exist_ok=True)
    for r in range(rounds):
        for name in names:
            env = dict(os.environ, EXM_LIB_PATH=lib_of(name))
            out = subprocess.run([sys.executable, "bench.py", "--config", cfg, "--steps", "100",
                                  "--warmup", "10", "--no-cpu-baseline", "--no-sdf-batch", *extra],
                                 cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
            try:
                d = json.loads(out.stdout.strip().splitlines()[-1])
                print(f"[{name:12s}] {cfg} step {d['ms_per_step']:.4f} p50 {d['ms_per_step_p50']:.4f}"
                      f" sdf {d['roofline']['sdf_kernel_ms']:.4f} e2e {d['e2e']['value']:.0f}", flush=True)
            except Exception:
                print(f"[{name:12s}] {cfg} FAILED: {out.stderr[-500:]}", flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "build":
        build(sys.argv[2:])
    else:
        bench(sys.argv[2], int(sys.argv[3]), sys.argv[4:])
