"""Phase timestamps of k_update (diagnostic build with -DEXM_TIMING; EXM_LIB_PATH points at it)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import _abi  # noqa: E402
from paper_2605_29663_b200 import workloads as W  # noqa: E402
from paper_2605_29663_b200.api import Engine  # noqa: E402

wl = W.cfg2()
eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
nom, up = wl.zero_state()
eng.stage(wl.q0, wl.obstacles(), wl.guidance, nom, up, 0)
eng.run_resident(3)
eng.read_resident()
buf = (C.c_longlong * 16)()
lib = _abi.load_library()
lib.exm_debug_probes(buf)
t = list(buf)
names = ["start", "beta", "S/A", "U+sync", "val: staged", "clamp", "heading", "sincos+xy", "x/y chain", "end"]
for i in range(1, 10):
    print(f"{names[i]:14s} {t[i] - t[i - 1]:8d} cycles")
print("total", t[9] - t[0], "cycles")
