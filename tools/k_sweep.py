"""Device ms per resident config-2 step (and SDF ms) for K = 4096 ... 512: the per-rank share
of the rollouts at 1, 2, 4, 8 GPUs (the sharded step without the all-gather), config 1, and
config 5 at K = 65,536 ... 8,192.
Usage (on the box): python tools/k_sweep.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

cases = ([("cfg2", K) for K in (4096, 2048, 1024, 512)] + [("cfg1", 1024)] +
         [("cfg5", K) for K in (65536, 32768, 16384, 8192)])
for name, K in cases:
    wl = getattr(W, name)(K=K)
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    if os.environ.get("SDF_MAP"):
        eng.set_sdf_map(os.environ["SDF_MAP"])
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(30)
    torch.cuda.synchronize()
    eng.step_stats()
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    ext = torch.cuda.ExternalStream(eng.stream_ptr())
    with torch.cuda.stream(ext):
        s.record(ext)
    n = 200 if name != "cfg5" else 40
    eng.run_resident(n)
    with torch.cuda.stream(ext):
        e.record(ext)
    torch.cuda.synchronize()
    st = eng.step_stats()
    print(f"{name} K={K:5d} T={wl.params.horizon} ms/step {s.elapsed_time(e) / n:.4f} "
          f"sdf {st['sdf_ms']:.4f} path {eng.last_sdf_path()[0]}")
    eng.close()
