"""Distribution of the per-pose minimum signed distance of a config's first cycle (GPU)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

for name in sys.argv[1:]:
    wl = getattr(W, name)()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    nom, up = wl.zero_state()
    eps = eng.sample_perturbations(wl.params.seed, 0)
    b = eng.evaluate_rollouts(wl.q0, nom, eps, wl.obstacles(), wl.guidance, up)
    d = b.d_min.reshape(-1)
    q = np.percentile(d, [0, 1, 10, 50, 90, 99, 100])
    print(name, "R=%.3f" % wl.footprint.bounding_radius(), "neg=%.3f" % (d < 0).mean(),
          "pct[0,1,10,50,90,99,100]=", np.round(q, 3))
    s = b.states[:, :-1, :2].reshape(-1, 2)
    print("   pose spread x", np.round(np.percentile(s[:, 0], [1, 50, 99]), 2), "y",
          np.round(np.percentile(s[:, 1], [1, 50, 99]), 2), "q0", wl.q0)
