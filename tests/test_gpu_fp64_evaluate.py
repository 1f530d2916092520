"""EXM_OPT_SDF_FP64: exm_evaluate_rollouts with FP64 minima (the reference's own arithmetic,
csrc/exm_exact64.cu) against the unmodified reference's evaluate_rollouts (oracle/_ref,
proj/src/controller.cpp:138-220) on the same injected noise. Minima and costs must agree at the
reference's own batch-vs-scalar tolerance, 1e-9 (proj/tests/acceptance_main.cpp:260-300,
proj/tests/test_controller.cpp:206-245); the only differences left are CUDA's vs glibc's
cos / sin / tan ulps in the states."""
import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine, FootprintSpec
from tests import oracle_bindings as ob

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not ob.reference_available(), reason="oracle/_ref not built")]

TOL = 1e-9

CASES = {
    "cfg1_rect": lambda: W.cfg1(K=256, T=16),
    "cfg2_l12": lambda: W.cfg2(K=256, T=20, N=3000),
    "cfg3_forklift": lambda: W.cfg3(K=256, T=20, N=4000),
    "cfg5_omni": lambda: W.cfg5(K=256, T=16, N=4000),
}


def _run(wl, masked):
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=max(wl.n_points, 1),
                 guide_cap=max(8, wl.guidance.path.shape[0]))
    eng.set_sdf_fp64(True)
    ref = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params, threads=8)
    D = wl.model.control_dim()
    eps = ref.sample_perturbations(3, 1)
    nom = 0.2 * np.ones(wl.params.horizon * D)
    up = np.full(3, 0.05)
    obs = wl.obstacles()
    pts, mask = obs.points, obs.mask.copy()
    if masked:  # every third point masked out
        mask[::3] = 0
        obs = type(obs)(pts, mask)
    got = eng.evaluate_rollouts(wl.q0, nom, eps, obs, wl.guidance, up)
    want = ref.evaluate_rollouts(wl.q0, nom, eps, pts, mask, wl.guidance, up)
    return got, want


@pytest.mark.parametrize("masked", [False, True])
@pytest.mark.parametrize("case", list(CASES))
def test_fp64_minima_and_costs_match_reference(case, masked):
    got, want = _run(CASES[case](), masked)
    assert np.array_equal(got.controls, want["controls"])
    assert np.max(np.abs(got.d_min - want["d_min"])) <= TOL
    rel = np.abs(got.costs - want["costs"]) / np.maximum(np.abs(want["costs"]), 1.0)
    assert np.max(rel) <= TOL
    assert np.array_equal(got.unsafe, want["unsafe"])


def test_fp64_empty_cloud_and_option_off():
    wl = W.cfg2(K=256, T=12, N=500)
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    ref = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params)
    eps = ref.sample_perturbations(5, 0)
    nom, up = np.zeros(wl.params.horizon * 2), np.zeros(3)
    obs = wl.obstacles()
    none = type(obs)(obs.points, np.zeros_like(obs.mask))
    eng.set_sdf_fp64(True)
    got = eng.evaluate_rollouts(wl.q0, nom, eps, none, wl.guidance, up)
    assert np.all(got.d_min == 1e6)  # kEmptyMaskDistance (geometry.hpp:37)
    fp64 = eng.evaluate_rollouts(wl.q0, nom, eps, obs, wl.guidance, up)
    eng.set_sdf_fp64(False)  # back to the FP32 culled kernels: within the 1e-5 m north star
    fp32 = eng.evaluate_rollouts(wl.q0, nom, eps, obs, wl.guidance, up)
    assert np.max(np.abs(fp32.d_min - fp64.d_min) / np.maximum(np.abs(fp64.d_min), 1.0)) <= 1e-5
    assert not np.array_equal(fp32.d_min, fp64.d_min)  # the FP32 path really ran


@pytest.mark.parametrize("fp_name", ["l12", "star64", "forklift", "box"])
@pytest.mark.parametrize("n", [1, 1000, 300_000])
def test_fp64_batch_signed_distance_matches_reference(fp_name, n):
    """batch_signed_distance (geometry.cpp:298-318) under EXM_OPT_SDF_FP64, through the chunked
    host pipeline (n = 300k: several chunks over the three staging slots), against the reference
    at its own 1e-12 (proj/tests/test_geometry.cpp:307-320)."""
    fp = {"l12": W.l12_footprint, "star64": W.star64_footprint, "forklift": W.forklift_footprint,
          "box": lambda: FootprintSpec.rect_cover([[0, 0]], [[0.5, 0.25]])}[fp_name]()
    wl = W.cfg2(K=256, T=4, N=16)
    eng = Engine(wl.model, wl.limits, fp, wl.params, n_cap=16, guide_cap=8)
    eng.set_sdf_fp64(True)
    ref = ob.Reference(fp, wl.model, wl.limits, wl.params)
    q = np.random.default_rng(n).uniform(-3.0, 3.0, size=(n, 2))
    got, want = eng.batch_signed_distance(q), ref.batch_signed_distance(q)
    assert np.all(np.abs(got - want) <= 1e-12 * (1.0 + np.maximum(np.abs(got), np.abs(want))))
    eng.set_sdf_fp64(False)
    f32 = eng.batch_signed_distance(q)
    assert np.max(np.abs(f32 - want) / np.maximum(np.abs(want), 1.0)) <= 1e-5
