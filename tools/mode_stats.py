"""Cull statistics per pose (tests, exact evaluations) for grid-kernel modes on configs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

modes = os.environ.get("MODES", "thread,share").split(",")
for name in sys.argv[1:]:
    wl = getattr(W, name)()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(2)
    n = wl.params.rollouts * wl.params.horizon
    for m in modes:
        os.environ["EXM_GRID_MODE"] = m
        a = eng.cull_stats()
        print(name, m, "tests/evals per pose %.1f %.1f" % (a[0] / n, a[1] / n))
    os.environ["EXM_GRID_MODE"] = ""
