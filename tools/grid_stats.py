"""Cull statistics (point tests, exact SDF evaluations) of the grid kernel on a config."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    wl = getattr(W, name)()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(1)
    print(name, os.environ.get("EXM_GRID_VARIANT"), eng.cull_stats())
