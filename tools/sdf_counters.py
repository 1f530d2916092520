"""SDF work counters and kernel time of the rollout signed distance for configs (one line each):
  EXM_LIB_PATH=... python tools/sdf_counters.py cfg2 cfg3 cfg5"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402,F401  (CUDA context + libnccl for the library)

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402
import bench  # noqa: E402

for cfg in sys.argv[1:]:
    wl = {"cfg1": W.cfg1, "cfg2": W.cfg2, "cfg3": W.cfg3, "cfg5": W.cfg5}[cfg]()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    if os.environ.get("SDF_MODE"):  # A/B of the kernel choice: thread / warp / cta / persist
        eng.set_sdf_mode(os.environ["SDF_MODE"])
    if os.environ.get("SDF_THRESHOLD") == "0":
        eng.set_sdf_threshold(False)
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(10)
    eng.step_stats()
    eng.run_resident(20)
    st = eng.step_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.run_resident(50)  # whole resident steps (graph launches back to back), wall clock
    torch.cuda.synchronize()
    step_ms = (time.perf_counter() - t0) / 50 * 1e3
    c = eng.sdf_work_stats()
    ops, _ = bench.executed_ops(c, wl.footprint)
    poses = wl.params.rollouts * wl.params.horizon
    per_pose = {k: round(v / poses, 2) for k, v in c.items()}
    eff = c["point_tests"] / (32.0 * c["point_iters_warp"]) if c["point_iters_warp"] else None
    print(json.dumps({"cfg": cfg, "lib": os.environ.get("EXM_LIB_PATH", "base"), "mode": os.environ.get("SDF_MODE", "auto"),
                      "sdf_ms": round(st["sdf_ms"], 4), "step_ms": round(step_ms, 4), "tflops_exec": round(ops / st["sdf_ms"] / 1e9, 2),
                      "lane_eff_points": eff and round(eff, 3), "path": eng.last_sdf_path()[0],
                      "per_pose": per_pose}), flush=True)
