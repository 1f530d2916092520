"""CPU tests of the body-frame cull geometry (exm_footprint_cull_boxes): the boxes the SDF
kernels bound with must contain the footprint, or the culling would not be exact. The polygon
inside test is the oracle's signed distance (oracle/exm_oracle.c, geometry.cpp:273-295)."""
import numpy as np
import pytest

from tests.oracle_bindings import Oracle
from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import FootprintSpec, KinematicLimits, MotionModel, MppiParams


def _footprints():
    out = [(n, W.footprint(n)) for n in W.GALLERY]
    out += [("l_shape_12", W.l12_footprint()), ("star64", W.star64_footprint()),
            ("forklift", W.forklift_footprint())]
    out += [(n, FootprintSpec.rect_cover(*W.RECT_FOOTPRINTS[n], n)) for n in W.RECT_FOOTPRINTS]
    return out


def _in_boxes(p, boxes, slack):
    inside = np.zeros(len(p), bool)
    for cx, cy, hx, hy in boxes:
        inside |= (np.abs(p[:, 0] - cx) <= hx + slack) & (np.abs(p[:, 1] - cy) <= hy + slack)
    return inside


@pytest.mark.parametrize("name,fp", _footprints(), ids=[n for n, _ in _footprints()])
def test_cover_contains_footprint(name, fp):
    aabb, boxes = fp.cull_boxes()
    assert 1 <= len(boxes) <= 3
    o = Oracle(fp, MotionModel.diff(), KinematicLimits.unbounded(), MppiParams(rollouts=1, horizon=1))
    rng = np.random.default_rng(7)
    r = fp.bounding_radius()
    p = rng.uniform(-r, r, size=(20000, 2))
    sd = o.batch_signed_distance(p)
    inside = p[sd <= 0.0]
    assert inside.shape[0] > 100
    assert _in_boxes(inside, boxes, 1e-6).all()
    # every boundary point (vertices, edge samples) as well
    v = fp.all_vertices()
    if fp.is_polygon():
        t = np.linspace(0.0, 1.0, 33)[:, None, None]
        seg = (v[None] * (1 - t) + np.roll(v, -1, axis=0)[None] * t).reshape(-1, 2)
        assert _in_boxes(seg, boxes, 1e-6).all()
    # and the boxes stay inside the AABB
    for cx, cy, hx, hy in boxes:
        assert cx - hx >= aabb[0] - 1e-5 and cx + hx <= aabb[1] + 1e-5
        assert cy - hy >= aabb[2] - 1e-5 and cy + hy <= aabb[3] + 1e-5


@pytest.mark.parametrize("fp", [W.footprint("l_shape"), W.l12_footprint()], ids=["L6", "L12"])
def test_l_cover_is_exact(fp):
    """The L (2.0 x 2.0, 0.4 m legs) is covered exactly by its two legs: total box area equals
    the polygon area (1.44 m^2) up to the 2.4e-4 m slack per side, so the notch is culled."""
    _, boxes = fp.cull_boxes()
    area = sum(4 * hx * hy for _, _, hx, hy in boxes)
    assert len(boxes) == 2
    assert area == pytest.approx(1.44, abs=3e-3)
