"""Write the footprint fixtures the reference's acceptance suite loads (FIXTURES_DIR/footprints)
from this repo's own transcription (paper_2605_29663_b200/workloads.py) — used to run the
reference's acceptance_main.cpp against the B200 drop-in on a box without the reference tree.

  python tools/write_fixtures.py <dir>
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2605_29663_b200 import workloads as W  # noqa: E402


def main(out):
    fdir = os.path.join(out, "footprints")
    os.makedirs(fdir, exist_ok=True)
    for name, verts in W.FOOTPRINTS.items():
        with open(os.path.join(fdir, f"{name}.json"), "w") as f:
            json.dump({"name": name, "kind": "polygon", "vertices": verts}, f)
    for name, (cs, hs) in W.RECT_FOOTPRINTS.items():
        rects = [{"center": c, "half_extent": h} for c, h in zip(cs, hs)]
        with open(os.path.join(fdir, f"{name}.json"), "w") as f:
            json.dump({"name": name, "kind": "rectangles", "rectangles": rects}, f)
    print(out)


if __name__ == "__main__":
    main(sys.argv[1])
