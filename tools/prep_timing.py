"""Phase timestamps of k_cloud_prep (diagnostic build with -DEXM_TIMING via EXM_LIB_PATH)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import _abi  # noqa: E402
from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

for name in sys.argv[1:] or ["cfg2"]:
    wl = getattr(W, name)()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    nom, up = wl.zero_state()
    eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
    eng.run_resident(3)
    eng.read_resident()
    buf = (C.c_longlong * 16)()
    _abi.load_library().exm_debug_probes_prep(buf)
    t = list(buf)
    names = ["start", "load+bbox", "gridmeta", "zero+hist", "scan", "scatter"]
    print(name, " ".join(f"{names[i]}={t[i] - t[i - 1]}" for i in range(1, 6)), "total", t[5] - t[0])
