"""Pins the C restatement bit-for-bit against the UNMODIFIED reference compiled from its own
sources (oracle/_ref/libexm_ref.so, built by oracle/Makefile). CPU only."""
import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import MppiParams
from tests import oracle_bindings as ob

pytestmark = pytest.mark.skipif(not ob.reference_available(), reason="oracle/_ref not built")


def both(wl):
    args = (wl.footprint, wl.model, wl.limits, wl.params)
    return ob.Oracle(*args), ob.Reference(*args)


@pytest.mark.parametrize("name", W.GALLERY + list(W.RECT_FOOTPRINTS) + ["l12", "star64", "forklift"])
def test_sd_bitwise(name):
    fp = {"l12": W.l12_footprint, "star64": W.star64_footprint,
          "forklift": W.forklift_footprint}.get(name, lambda: W.footprint(name))()
    wl = W.cfg1(K=4, T=3)
    wl.footprint = fp
    o, r = both(wl)
    assert o.radius() == r.radius()
    q = W.benchmark_queries(5000, 8.0, 17)
    assert np.array_equal(o.batch_signed_distance(q), r.batch_signed_distance(q))


def test_min_sd_at_bitwise():
    wl = W.cfg2(K=8, T=4, N=2000)
    o, r = both(wl)
    mask = (np.arange(wl.n_points) % 7 != 3).astype(np.uint8)
    poses = np.concatenate([W.cfg4_poses(300)[:, :2] * 1.5, W.cfg4_poses(300)[:, 2:]], 1)
    r.set_cloud(wl.cloud, mask)
    want = r.min_sd_at(poses)
    got = o.sdf_batch(poses, wl.cloud, mask)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2", "cfg3", "cfg5"])
def test_rollouts_bitwise(cfg):
    wl = {"cfg1": lambda: W.cfg1(K=32, T=10), "cfg2": lambda: W.cfg2(K=32, T=12, N=1500),
          "cfg3": lambda: W.cfg3(K=32, T=12, N=1500), "cfg5": lambda: W.cfg5(K=32, T=10, N=1500)}[cfg]()
    o, r = both(wl)
    eps_o, eps_r = o.sample_perturbations(1, 3), r.sample_perturbations(1, 3)
    assert np.array_equal(eps_o, eps_r)
    nom = 0.1 * np.ones(wl.params.horizon * wl.model.control_dim())
    args = (wl.q0, nom, eps_o, wl.cloud, None, wl.guidance, np.full(3, 0.05))
    a, b = o.evaluate_rollouts(*args), r.evaluate_rollouts(*args)
    for k in ("controls", "states", "d_min", "costs", "unsafe"):
        assert np.array_equal(a[k], b[k]), k


def test_weights_bitwise():
    c = W.uniform_range(5, np.arange(300, dtype=np.uint64), 0, -10, 10)
    wl = W.cfg1(K=4, T=3)
    _, r = both(wl)
    assert np.array_equal(ob.oracle_weights(c, 0.7), r.weights_from_costs(c, 0.7))


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_control_cycle_sequence_bitwise(cfg):
    """Three consecutive MppiController::control_cycle calls of a fresh reference controller vs
    the oracle's explicit-state cycle (device-style noise drawn from (seed, cycle))."""
    wl = W.cfg1(K=64, T=12) if cfg == "cfg1" else W.cfg2(K=64, T=12, N=1500)
    o, r = both(wl)
    nom, up = wl.zero_state()
    q = wl.q0.copy()
    for cyc in range(3):
        want = r.controller_cycle(q, wl.cloud, None, wl.guidance)
        got = o.control_cycle(q, wl.cloud, None, wl.guidance, nom, up, cyc)
        for k in ("command", "validated", "best_cost", "weight_entropy", "nominal_cost"):
            assert np.array_equal(got[k], want[k]), (cyc, k)
        assert np.array_equal(got["nominal_d_min"], want["nominal_d_min"])
        assert np.array_equal(nom, want["nominal"])
        q = o.step(q, got["command"][: wl.model.control_dim()])


def test_validation_errors_match():
    wl = W.cfg1(K=4, T=3)
    bad = MppiParams(rollouts=0)
    for cls in (ob.Oracle, ob.Reference):
        with pytest.raises(ValueError, match="rollouts must be >= 1"):
            cls(wl.footprint, wl.model, wl.limits, bad)
