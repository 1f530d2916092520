"""Exactness of the culled grid SDF (GPU): every cull (ring, cell, chunk, point bounds with the
rounding margin) may only skip points that cannot lower the minimum, so the culled per-pose
minimum must equal, bit for bit, the same kernel with every bound disabled (EXM_SDF_BRUTE:
every valid point evaluated with identical FP32 arithmetic). Covers both kernels (thread- and
warp-per-pose), polygons (L12, L6, star) and rectangle covers (1 and 3 boxes), clouds with
obstacles overlapping the footprint (negative minima) and far obstacles (large minima)."""
import dataclasses
import math

import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine, FootprintSpec

pytestmark = pytest.mark.gpu

def _nonagon() -> FootprintSpec:
    """A 9-vertex concave polygon: no compile-time edge count (the generic NB=0 kernels)."""
    a = 2 * math.pi * np.arange(9) / 9
    r = np.where(np.arange(9) % 2 == 0, 1.0, 0.55)
    return FootprintSpec.polygon(np.stack([r * np.cos(a), r * np.sin(a)], 1), "nonagon")


def _wide_scene():
    """Config 2's clutter plus 2,000 points on a ring 90 m out: a 180 m extent, so the grid's
    per-axis cell cap (kGridMax) binds and the cells are far coarser than the density asks."""
    wl = W.cfg2(K=2048, T=40, N=10_000)
    a = 2 * math.pi * np.arange(2000) / 2000
    ring = wl.q0[:2] + 90.0 * np.stack([np.cos(a), np.sin(a)], 1)
    return dataclasses.replace(wl, cloud=np.concatenate([wl.cloud, ring]))


CASES = {
    "cfg2_wide_capped_grid": _wide_scene,
    "cfg2_star64": lambda: dataclasses.replace(W.cfg2(K=2048, T=40, N=10_000),
                                               footprint=W.star64_footprint()),
    "cfg2_nonagon": lambda: dataclasses.replace(W.cfg2(K=2048, T=40, N=10_000),
                                                footprint=_nonagon()),
    "cfg2_L12": lambda: W.cfg2(K=2048, T=40, N=10_000),
    "cfg3_forklift": lambda: W.cfg3(K=2048, T=40, N=20_000),
    "cfg5_L6_overlap": lambda: W.cfg5(K=1024, T=80, N=30_000),
    "cfg1_rect_far": lambda: W.cfg1(K=2560, T=30),
}


def _dmin(wl, mode, caps=None):
    """Per-step minima of two pose sets with the SDF kernel forced to `mode` (exm_set_option
    EXM_OPT_SDF_MODE: brute, thread, warp, cta, nochunk, persist = thread per pose with the
    persistent work counter at any size)."""
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    eng.set_sdf_mode(mode)
    if caps is not None:
        eng.set_sdf_caps(caps)
    nom, up = wl.zero_state()
    eps = eng.sample_perturbations(wl.params.seed, 0)
    # a few cycles' worth of distinct pose sets: nominal offsets
    out = []
    for scale in (0.0, 0.3):
        b = eng.evaluate_rollouts(wl.q0, nom + scale, eps, wl.obstacles(), wl.guidance, up)
        out.append(b.d_min.copy())
    path = eng.last_sdf_path()[0]
    want_kernel = {"thread": 0, "brute": 0, "nochunk": 0, "persist": 0, "warp": 1, "cta": 2}[mode]
    assert path["kernel"] == want_kernel, (mode, path)
    if mode == "persist":
        assert path["persistent"] == 1
    eng.close()
    return np.concatenate([o.reshape(-1) for o in out])


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("mode", ["thread", "warp", "cta", "nochunk", "persist"])
def test_culled_minimum_is_bitwise_brute_force(case, mode):
    wl = CASES[case]()
    want = _dmin(wl, "brute")
    got = _dmin(wl, mode)
    assert got.shape == want.shape
    bad = np.flatnonzero(got != want)
    assert bad.size == 0, f"{bad.size} poses differ, e.g. {bad[:5]}: {got[bad[:5]]} vs {want[bad[:5]]}"


@pytest.mark.parametrize("case", ["cfg2_L12", "cfg3_forklift", "cfg5_L6_overlap"])
def test_capped_minimum_is_bitwise_brute_force(case):
    """Caps (per-step hints) only prune: caps far below, around and above the true minima, and
    a per-step mix, all give the brute-force minima bit for bit."""
    wl = CASES[case]()
    want = _dmin(wl, "brute")
    T = wl.params.horizon
    per_step = np.quantile(want.reshape(-1, T), 0.5, axis=0).astype(np.float32)  # half resolve
    for caps in (-1.0, 0.05, 0.3, 5.0, per_step):
        got = _dmin(wl, "thread", caps)
        bad = np.flatnonzero(got != want)
        assert bad.size == 0, (caps, bad.size)


@pytest.mark.parametrize("case", ["cfg2_L12", "cfg3_forklift"])
def test_lane_mapping_does_not_change_minima(case):
    """Both lane <-> pose mappings of the thread-per-pose kernel (a rollout's steps per warp /
    rollouts at one step per warp) and the tuned choice give the same minima bit for bit, and
    the resident steps after tuning equal the untuned host-API steps."""
    wl = CASES[case]()
    outs = {}
    for mapping in ("rmajor", "hmajor"):
        eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
        eng.set_sdf_mode("thread")
        eng.set_sdf_map(mapping)
        nom, up = wl.zero_state()
        eps = eng.sample_perturbations(wl.params.seed, 0)
        outs[mapping] = eng.evaluate_rollouts(wl.q0, nom, eps, wl.obstacles(), wl.guidance, up).d_min
        assert eng.last_sdf_path()[0]["hmajor"] == (mapping == "hmajor")
        eng.close()
    assert np.array_equal(outs["rmajor"], outs["hmajor"])
    tuned = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    plain = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    plain.set_sdf_map("rmajor")
    n1, u1 = wl.zero_state()
    n2, u2 = wl.zero_state()
    for cyc in range(8):  # the first 6 steps of `tuned` alternate the mappings outside a graph
        a = tuned.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, n1, u1, cyc)
        b = plain.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, n2, u2, cyc)
        assert np.array_equal(a.command, b.command) and a.argmin == b.argmin
        assert np.array_equal(n1, n2)
    print(case, "tuned mapping:", tuned.last_sdf_path()[0])
