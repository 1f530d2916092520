"""Cull statistics per pose after a few resident steps (caps from the previous step in place)
versus uncapped (EXM_GRID_MODE=nocap)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

for name in sys.argv[1:]:
    wl = getattr(W, name)()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(3)
    n = wl.params.rollouts * wl.params.horizon
    a = eng.cull_stats()
    os.environ["EXM_GRID_MODE"] = "nocap"
    b = eng.cull_stats()
    os.environ["EXM_GRID_MODE"] = ""
    print(name, "capped tests/evals per pose %.1f %.1f" % (a[0] / n, a[1] / n),
          " uncapped %.1f %.1f" % (b[0] / n, b[1] / n))
