"""The reference's evaluator benchmark (scaling_benchmark, proj/src/bench.cpp:55-113; CLI `bench`)
re-run with B200 rows, in the reference's CSV schema
`footprint,evaluator,queries,trials,mean_us,std_us,median_us,threads` (bench.cpp:57).

Rows per (footprint, query count):
  threads=1 / threads=<nproc>  the unmodified reference's batch_signed_distance (oracle/_ref),
                               wall clock per call, exactly its protocol (3 warm-ups)
  threads=b200-kernel          k_sdf_pairs on device-resident queries, CUDA events per launch
  threads=b200-call            exm_batch_signed_distance host->host (pipelined FP32 staging, H2D,
                               kernel, D2H), wall clock per call from Python — the analogue of
                               the paper's per-call JAX timing (L 0.09/0.29 ms,
                               T 0.09/0.32, F 0.15/0.30 at 1e5)
  threads=b200-dropin-P(T)     the reference's OWN scaling_benchmark (bench.cpp, compiled where it
                               lies) with batch_signed_distance redirected to the B200 by
                               host/geometry_sdf_b200.cpp (lib/exm_scaling_b200), T host threads,
                               P = fp64 (the drop-in's default) or fp32 (EXM_DROPIN_SDF_FP32=1)

  python tools/scaling_benchmark.py [--trials 100] [--counts 100,1000,10000,100000,1000000]
"""
import argparse
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402
from tests import oracle_bindings as ob  # noqa: E402

NAMES = ["l_shape", "l_shape_rect", "t_shape", "t_shape_rect", "f_shape", "f_shape_rect"]


def stats(samples_us):
    m = statistics.fmean(samples_us)
    sd = statistics.pstdev(samples_us)
    return m, sd, statistics.median(samples_us)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--trials", type=int, default=100)
    ap.add_argument("--counts", default="100,1000,10000,100000,1000000")
    ap.add_argument("--cpu-max", type=int, default=100000, help="largest count for CPU rows")
    ap.add_argument("--seed", type=int, default=0)
    args = ap.parse_args()
    counts = [int(c) for c in args.counts.split(",")]
    nproc = os.cpu_count() or 1
    base = W.cfg1(K=8, T=2)
    print("footprint,evaluator,queries,trials,mean_us,std_us,median_us,threads")
    for name in NAMES:
        fp = W.footprint(name)
        evaluator = "polygon" if fp.is_polygon() else "rect_cover"
        eng = Engine(base.model, base.limits, fp, base.params, n_cap=16, guide_cap=4)
        ref = ob.Reference(fp, base.model, base.limits, base.params) if ob.reference_available() else None
        for n in counts:
            q = np.ascontiguousarray(
                W.benchmark_queries(n, 50.0, int(W.hash_combine(args.seed, n))))
            rows = []
            if ref is not None and n <= args.cpu_max:
                for th in sorted({1, nproc}):
                    for _ in range(3):
                        ref.batch_signed_distance(q, th)
                    s = []
                    for _ in range(args.trials):
                        t0 = time.perf_counter()
                        ref.batch_signed_distance(q, th)
                        s.append(1e6 * (time.perf_counter() - t0))
                    rows.append((str(th), stats(s)))
            # device-resident kernel time
            eng.sdf_stage(np.zeros((1, 3)), q)
            eng.sdf_run_resident(3, True)
            eng.step_stats()
            s = []
            for _ in range(args.trials):
                eng.sdf_run_resident(1, True)
                s.append(1e3 * eng.step_stats()["sdf_ms"])
            rows.append(("b200-kernel", stats(s)))
            # host -> host per call through the C ABI
            for _ in range(3):
                eng.batch_signed_distance(q)
            s = []
            for _ in range(args.trials):
                t0 = time.perf_counter()
                eng.batch_signed_distance(q)
                s.append(1e6 * (time.perf_counter() - t0))
            rows.append(("b200-call", stats(s)))
            for th, (m, sd, med) in rows:
                print(f"{name},{evaluator},{n},{args.trials},{m:.3f},{sd:.3f},{med:.3f},{th}",
                      flush=True)
    dropin_rows(counts, args.trials, nproc)


def dropin_rows(counts, trials, nproc):
    """The reference's scaling_benchmark itself, every batch_signed_distance call on the B200."""
    import subprocess
    import tempfile
    binary = os.path.join(ROOT, "paper_2605_29663_b200", "lib", "exm_scaling_b200")
    if not os.path.exists(binary):
        return
    with tempfile.TemporaryDirectory() as d:
        subprocess.run([sys.executable, os.path.join(ROOT, "tools", "write_fixtures.py"), d],
                       check=True, capture_output=True)
        # the drop-in's default is FP64 (EXM_OPT_SDF_FP64, the reference's arithmetic);
        # EXM_DROPIN_SDF_FP32=1 rows time the FP32 kernel through the same call
        for prec, fp32 in (("fp64", "0"), ("fp32", "1")):
            env = dict(os.environ, EXM_DROPIN_SDF_FP32=fp32)
            for th in sorted({1, min(8, nproc)}):
                out = subprocess.run([binary, d, str(trials), str(th), *map(str, counts)],
                                     check=True, capture_output=True, text=True, env=env).stdout
                for line in out.strip().splitlines()[1:]:
                    f = line.split(",")
                    print(",".join(f[:7] + [f"b200-dropin-{prec}({f[7]})"]), flush=True)


if __name__ == "__main__":
    main()
