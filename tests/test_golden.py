"""Committed golden vectors (tests/golden/*.npz, produced by tests/golden/make_golden.py from the
unmodified reference): the oracle must reproduce them bit for bit (CPU), the B200 path within
the north-star tolerances (GPU)."""
import os

import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine
from tests import oracle_bindings as ob
from tests.golden.make_golden import FOOTPRINTS, SMALL

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLD, name))


def rel_err(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    return float(np.max(np.abs(got - want) / np.maximum(np.abs(want), 1.0)))


# ----------------------------------------------------------------- oracle (CPU, bitwise)
@pytest.mark.parametrize("name", list(FOOTPRINTS))
def test_oracle_sd_golden(name):
    g = load("sd_footprints.npz")
    base = W.cfg1(K=4, T=2)
    o = ob.Oracle(FOOTPRINTS[name](), base.model, base.limits, base.params)
    assert np.array_equal(o.batch_signed_distance(g["queries"]), g[name])


def test_oracle_min_sd_golden():
    g = load("min_sd_cfg2.npz")
    wl = W.cfg2(K=4, T=2, N=2000)
    assert np.array_equal(wl.cloud, g["cloud"])  # the generator is itself pinned
    o = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
    assert np.array_equal(o.sdf_batch(g["poses"], g["cloud"], g["mask"]), g["d_min"])


@pytest.mark.parametrize("cfg", list(SMALL))
def test_oracle_rollouts_golden(cfg):
    g = load(f"rollouts_{cfg}.npz")
    wl = SMALL[cfg]()
    o = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
    assert np.array_equal(o.sample_perturbations(wl.params.seed, 0), g["eps"])
    out = o.evaluate_rollouts(wl.q0, g["nominal"], g["eps"], wl.cloud, None, wl.guidance, g["u_prev"])
    for k in ("controls", "states", "d_min", "costs", "unsafe"):
        assert np.array_equal(out[k], g[k]), k


@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_oracle_cycles_golden(cfg):
    g = load(f"cycles_{cfg}.npz")
    wl = SMALL[cfg]()
    o = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
    nom, up = wl.zero_state()
    for c in range(3):
        d = o.control_cycle(g["q"][c], wl.cloud, None, wl.guidance, nom, up, c)
        assert np.array_equal(d["command"], g["command"][c])
        assert np.array_equal(nom, g["nominal"][c])
        assert d["best_cost"] == g["best_cost"][c] and d["nominal_cost"] == g["nominal_cost"][c]


# ----------------------------------------------------------------- B200 (GPU, tolerance)
@pytest.mark.gpu
def test_gpu_sd_golden():
    g = load("sd_footprints.npz")
    base = W.cfg1(K=4, T=2)
    for name, mk in FOOTPRINTS.items():
        eng = Engine(base.model, base.limits, mk(), base.params, n_cap=16, guide_cap=4)
        got = eng.batch_signed_distance(g["queries"])
        assert rel_err(got, g[name]) <= 1e-5, name
        m = np.abs(g[name]) >= 1e-5
        assert np.all((got[m] < 0) == (g[name][m] < 0)), name


@pytest.mark.gpu
def test_gpu_min_sd_golden():
    g = load("min_sd_cfg2.npz")
    wl = W.cfg2(K=4, T=2, N=2000)
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=2000, guide_cap=4)
    assert rel_err(eng.sdf_batch(g["poses"], g["cloud"], g["mask"]), g["d_min"]) <= 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", list(SMALL))
def test_gpu_rollouts_golden(cfg):
    g = load(f"rollouts_{cfg}.npz")
    wl = SMALL[cfg]()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    assert np.allclose(eng.sample_perturbations(wl.params.seed, 0), g["eps"], rtol=1e-12, atol=1e-14)
    r = eng.evaluate_rollouts(wl.q0, g["nominal"], g["eps"], wl.obstacles(), wl.guidance, g["u_prev"])
    assert rel_err(r.d_min, g["d_min"]) <= 1e-5
    assert np.allclose(r.states, g["states"], rtol=1e-9, atol=1e-9)
    deg = ((np.abs(g["d_min"]) < 1e-5) | (np.abs(g["d_min"] - wl.params.d_safe) < 1e-5)).any(1)
    assert rel_err(r.costs[~deg], g["costs"][~deg]) <= 1e-5
    assert np.array_equal(r.unsafe[~deg], g["unsafe"][~deg])


@pytest.mark.gpu
@pytest.mark.parametrize("cfg", ["cfg1", "cfg2"])
def test_gpu_cycles_golden(cfg):
    g = load(f"cycles_{cfg}.npz")
    wl = SMALL[cfg]()
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
    nom, up = wl.zero_state()
    D = wl.model.control_dim()
    for c in range(3):
        d = eng.control_cycle_raw(g["q"][c], wl.obstacles(), wl.guidance, nom, up, c)
        assert d.validated == bool(g["validated"][c])
        assert np.max(np.abs(d.command - g["command"][c][:D])) <= 1e-5
        assert np.max(np.abs(nom - g["nominal"][c])) <= 1e-5
        nom[:] = g["nominal"][c]
        up[:] = 0.0
        up[:D] = g["command"][c][:D]
