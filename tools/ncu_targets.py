"""Small, deterministic launch sequences for ncu captures (never a bench number).

  python tools/ncu_targets.py step [n]    n resident MPPI steps of config 2 (k_sdf_grid et al.)
  python tools/ncu_targets.py pairs [n]   n launches of k_sdf_pairs on config 4 (10^9 pairs)
  python tools/ncu_targets.py cfgX [n]    n resident steps of config X (1, 3, 5)
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402


# The lane mapping the live tuner picks per config (bench.py's sdf_path.hmajor). Under ncu every
# kernel is serialised and replayed, so the tuner's event timings mean nothing there: pin it.
LIVE_MAP = {"cfg1": "rmajor", "cfg2": "rmajor", "cfg3": "rmajor", "cfg5": "rmajor"}


def steps(wl, n, cfg="cfg2"):
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    eng.set_sdf_map(os.environ.get("SDF_MAP", LIVE_MAP[cfg]))
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(n)
    print(eng.step_stats(), eng.read_resident().argmin)


def pairs(n, want_pairs=False):
    fp, poses, pts = W.cfg4()
    wl = W.cfg1(K=8, T=2)
    eng = Engine(wl.model, wl.limits, fp, wl.params, n_cap=16, guide_cap=4)
    eng.sdf_stage(poses, pts)
    eng.sdf_run_resident(n, want_pairs)
    print(eng.step_stats())


if __name__ == "__main__":
    what = sys.argv[1]
    n = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    if what == "step":
        steps(W.cfg2(), n, "cfg2")
    elif what == "pairs":
        pairs(n)
    elif what == "pairs_out":
        pairs(n, True)
    else:
        steps({"cfg1": W.cfg1, "cfg3": W.cfg3, "cfg5": W.cfg5}[what](), n, what)
