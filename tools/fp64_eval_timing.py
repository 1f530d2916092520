"""Wall time of one exm_evaluate_rollouts call (host buffers in and out, config-2 and config-1
full size) with the FP32 culled minima and with EXM_OPT_SDF_FP64 (FP64 brute force in the
reference's arithmetic), beside the unmodified reference's evaluate_rollouts on all host threads.

  python tools/fp64_eval_timing.py
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402
from tests import oracle_bindings as ob  # noqa: E402


def timed(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts)) * 1e3, out


def main():
    for name, f in (("cfg1", W.cfg1), ("cfg2", W.cfg2)):
        wl = f()
        eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
        ref = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params, threads=os.cpu_count())
        D = wl.model.control_dim()
        eps = ref.sample_perturbations(3, 1)
        nom, up = 0.2 * np.ones(wl.params.horizon * D), np.full(3, 0.05)
        obs = wl.obstacles()
        call = lambda: eng.evaluate_rollouts(wl.q0, nom, eps, obs, wl.guidance, up)  # noqa: E731
        eng.set_sdf_fp64(False)
        t32, g32 = timed(call, 10)
        eng.set_sdf_fp64(True)
        t64, g64 = timed(call, 5)
        tr, want = timed(lambda: ref.evaluate_rollouts(wl.q0, nom, eps, wl.cloud, None,
                                                       wl.guidance, up), 2)
        e32 = np.max(np.abs(g32.d_min - want["d_min"]))
        e64 = np.max(np.abs(g64.d_min - want["d_min"]))
        print(f"{name} K={wl.params.rollouts} T={wl.params.horizon} N={wl.n_points}: "
              f"fp32 {t32:.2f} ms (max |dd| {e32:.2e}), fp64 {t64:.2f} ms (max |dd| {e64:.2e}), "
              f"reference {tr:.1f} ms on {os.cpu_count()} threads", flush=True)


if __name__ == "__main__":
    main()
