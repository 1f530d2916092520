"""Cross-check of the SDF kernel time: event-timed inside the step graph (step_stats) against
the whole resident step, with the d_safe threshold on and off (config 2). Run it plain and
under ncu's launch list to compare the per-kernel durations:
  python tools/sdf_timing_check.py [on|off|both]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
for thr in ([True, False] if which == "both" else [which == "on"]):
    wl = W.cfg2()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    eng.set_sdf_threshold(thr)
    if os.environ.get("SDF_MAP"):
        eng.set_sdf_map(os.environ["SDF_MAP"])
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(10)
    torch.cuda.synchronize()
    eng.step_stats()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    eng.run_resident(30)
    b.record()
    torch.cuda.synchronize()
    st = eng.step_stats()
    print(f"threshold={thr} step_ms={a.elapsed_time(b) / 30:.4f} sdf_event_ms={st['sdf_ms']:.4f} "
          f"path={eng.last_sdf_path()[0]}", flush=True)
    eng.close()
