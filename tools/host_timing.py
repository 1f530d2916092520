"""Host-side phases of exm_control_cycle (EXM_OPT_HOST_TIMING) and the Python per-call time, cfg2."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402,F401
from paper_2605_29663_b200 import _abi, workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine, ObstacleSet  # noqa: E402

wl = W.cfg2()
eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
obst = wl.obstacles()
if len(sys.argv) > 1 and sys.argv[1] == "pinned":
    obst = ObstacleSet.pinned(obst.points, obst.mask)
nom, up = wl.zero_state()
for c in range(20):
    eng.control_cycle_raw(wl.q0, obst, wl.guidance, nom, up, c)
eng.set_option(_abi.OPT_HOST_TIMING, 1)
t0 = time.perf_counter()
n = 300
for c in range(n):
    eng.control_cycle_raw(wl.q0, obst, wl.guidance, nom, up, 100 + c)
dt = (time.perf_counter() - t0) / n
print({"per_call_us": 1e6 * dt, **eng.host_timing()})
