"""Hybrid mode families: every family's MPPI step in one device call
(exm_hybrid_cycle), checked (a) against the same families stepped one by one through
exm_control_cycle — bit for bit — and (b) end to end against the reference's own
HybridController (oracle/_ref: hybrid.cpp over the reference MppiControllers)."""
import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import (Engine, HybridController, HybridParams, MotionModel,
                                       ObstacleSet, deadzone_correct, project_to_mode)
from tests import oracle_bindings as ob


def test_projection_and_deadzone():  # hybrid.cpp:18-78 (host logic, CPU)
    hp = HybridParams()
    assert np.allclose(project_to_mode(np.array([0.3, 0.2]), MotionModel.spin()), [0.2])
    assert np.allclose(project_to_mode(np.array([0.3, -0.1, 0.2]), MotionModel.parallel()), [-0.1])
    assert np.allclose(project_to_mode(np.array([0.3, 0.2]), MotionModel.ackermann(0.5)), [0.3, 0.2])
    assert np.allclose(deadzone_correct(np.array([0.03]), MotionModel.spin(), hp), [0.05])
    assert np.allclose(deadzone_correct(np.array([-0.005]), MotionModel.spin(), hp), [-0.005])
    assert np.allclose(deadzone_correct(np.array([0.02, 0.3]), MotionModel.diff(), hp), [0.05, 0.3])
    with pytest.raises(ValueError):
        HybridParams(noise_deadzone_v=0.06).validate()


@pytest.mark.gpu
def test_batched_families_equal_single_family_steps():
    fp, modes, params, hp, q0, cloud, g = W.trap_hybrid()
    hc = HybridController(modes, fp, params, hp, n_cap=cloud.shape[0], guide_cap=8)
    obst = ObstacleSet(cloud, np.ones(cloud.shape[0], np.uint8))
    singles = []
    for m, mode in enumerate(modes):
        p = W.MppiParams(**{**params.__dict__})
        p.seed = params.seed ^ ((0x9E3779B97F4A7C15 * (m + 1)) & 0xFFFFFFFFFFFFFFFF)
        singles.append(Engine(mode.model, mode.limits, fp, p, n_cap=cloud.shape[0], guide_cap=8))
    noms = [np.zeros(params.horizon * m.model.control_dim()) for m in modes]
    ups = [np.zeros(3) for _ in modes]
    for cyc in range(3):
        fam = hc.family_cycles(q0, obst, g)
        for m in range(len(modes)):
            d = singles[m].control_cycle_raw(q0, obst, g, noms[m], ups[m], cyc)
            assert np.array_equal(d.command, fam[m].command), (cyc, m)
            assert d.validated == fam[m].validated and d.argmin == fam[m].argmin
            assert np.array_equal(noms[m].reshape(-1), fam[m].nominal.reshape(-1))
            assert d.nominal_cost == fam[m].nominal_cost


@pytest.mark.gpu
@pytest.mark.skipif(not ob.reference_available(), reason="oracle/_ref not built")
def test_hybrid_controller_vs_reference():
    fp, modes, params, hp, q0, cloud, g = W.trap_hybrid()
    hc = HybridController(modes, fp, params, hp, n_cap=cloud.shape[0], guide_cap=8)
    ref = ob.ReferenceHybrid(fp, modes, params, hp)
    obst = ObstacleSet(cloud, np.ones(cloud.shape[0], np.uint8))
    q = q0.copy()
    for cyc in range(8):
        got = hc.hybrid_cycle(q, obst, g)
        want = ref.hybrid_cycle(q, cloud, None, g)
        assert got.mode_index == want["mode_index"], cyc
        assert got.validated == want["validated"], cyc
        D = modes[got.mode_index].model.control_dim()
        assert np.max(np.abs(got.command - want["command"][:D])) <= 1e-5, cyc
        fin = np.isfinite(want["mode_costs"])
        assert np.array_equal(np.isfinite(got.mode_costs), fin)
        assert np.allclose(np.array(got.mode_costs)[fin], want["mode_costs"][fin], rtol=1e-5)
        # advance with the reference's command under the selected mode's model (run_episode)
        orc = ob.Oracle(fp, modes[got.mode_index].model, modes[got.mode_index].limits, params)
        q = orc.step(q, want["command"][:D])
