#!/usr/bin/env python
"""Config 5 per-snapshot device step: the e2e leg of bench.py cycles through 8 moving-obstacle
snapshots (cycle = 10 j); this times resident steps on each one separately (CUDA events on the
library's stream), with the SDF kernel time and the cull counters.

  python tools/cfg5_snapshots.py [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    wl = W.cfg5()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8, device=0)
    ext = torch.cuda.ExternalStream(eng.stream_ptr())
    for j in range(8):
        obs = W.cfg5(cycle=10 * j).obstacles()
        nom, up = wl.zero_state()
        eng.stage(wl.q0, obs, wl.guidance, nom, up, 0)
        eng.run_resident(5)
        torch.cuda.synchronize()
        eng.step_stats()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(ext):
            a.record(ext)
        eng.run_resident(steps)
        with torch.cuda.stream(ext):
            b.record(ext)
        torch.cuda.synchronize()
        st = eng.step_stats()
        c = eng.sdf_work_stats()
        poses = wl.params.rollouts * wl.params.horizon
        per = {k: round(v / poses, 1) for k, v in c.items()}
        print(f"snapshot {j}: step {a.elapsed_time(b) / steps:.3f} ms  sdf {st['sdf_ms']:.3f} ms  "
              f"per pose {per}", flush=True)


if __name__ == "__main__":
    main()
