"""GPU parity: libexm_b200.so (through the C ABI) vs the CPU oracle (oracle/exm_oracle.c, itself
pinned bit-for-bit to the reference) on identical seeded inputs.

Tolerances (BASELINE.json north_star):
  signed distance   |d - d_ref| <= 1e-5 * max(|d_ref|, 1 m)         (FP32 kernel)
  signs             exact wherever |d_ref| >= 1e-5 m
  rollout cost      1e-5 relative, rollouts with a cost-cliff-degenerate step excluded
                    (|d_ref| < 1e-5 or |d_ref - d_safe| < 1e-5)
  argmin            exact unless degenerate
  command/nominal   |delta| <= 1e-5
  FP64-only parts   states/controls/noise: 1e-9 relative (reference's batch/scalar KAT)
"""
import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine, FootprintSpec, Guidance, MppiParams
from tests import oracle_bindings as ob

pytestmark = pytest.mark.gpu

SD_TOL = 1e-5
DEG = 1e-5


def sd_close(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    err = np.abs(got - want) / np.maximum(np.abs(want), 1.0)
    return float(np.max(err)) if err.size else 0.0


def sign_mismatch(got, want):
    m = np.abs(want) >= DEG
    return int(np.count_nonzero((got[m] < 0) != (want[m] < 0)))


def engine_and_oracle(wl, n_cap=None):
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params,
                 n_cap=n_cap or max(wl.n_points, 1), guide_cap=max(8, wl.guidance.path.shape[0]))
    orc = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
    return eng, orc


ALL_FP = W.GALLERY + list(W.RECT_FOOTPRINTS) + ["l12", "star64", "forklift", "box"]


def get_fp(name):
    return {"l12": W.l12_footprint, "star64": W.star64_footprint,
            "forklift": W.forklift_footprint,
            "box": lambda: FootprintSpec.rect_cover([[0, 0]], [[0.5, 0.25]])}.get(
        name, lambda: W.footprint(name))()


@pytest.mark.parametrize("name", ALL_FP)
def test_sdf_pairs_every_footprint(name):
    wl = W.cfg1(K=4, T=2)
    wl.footprint = get_fp(name)
    eng, orc = engine_and_oracle(wl)
    poses = W.cfg4_poses(40) * np.array([0.5, 0.5, 1.0])
    pts = W.benchmark_queries(3000, 8.0, 11)
    mins, pairs = eng.sdf_batch(poses, pts, per_pair=True)
    omins, opairs = orc.sdf_batch(poses, pts, per_pair=True)
    assert sd_close(pairs, opairs) <= SD_TOL
    assert sign_mismatch(pairs.astype(np.float64), opairs) == 0
    assert sd_close(mins, omins) <= SD_TOL


def test_sdf_mask_and_empty():
    wl = W.cfg2(K=4, T=2, N=500)
    eng, orc = engine_and_oracle(wl)
    poses = W.cfg4_poses(16)
    mask = (np.arange(wl.n_points) % 3 == 0).astype(np.uint8)
    mins, pairs = eng.sdf_batch(poses, wl.cloud, mask, per_pair=True)
    assert np.all(np.isinf(pairs[:, mask == 0]))
    assert sd_close(mins, orc.sdf_batch(poses, wl.cloud, mask)) <= SD_TOL
    empty = eng.sdf_batch(poses, wl.cloud, np.zeros(wl.n_points, np.uint8))
    assert np.all(empty == 1e6)  # kEmptyMaskDistance


def test_batch_signed_distance_body_frame():
    wl = W.cfg1(K=4, T=2)
    wl.footprint = W.footprint("f_shape")
    eng, orc = engine_and_oracle(wl)
    q = W.benchmark_queries(20000, 6.0, 70)
    got, want = eng.batch_signed_distance(q), orc.batch_signed_distance(q)
    assert sd_close(got, want) <= SD_TOL and sign_mismatch(got, want) == 0


def degenerate_rows(dmin_ref, d_safe):
    bad = (np.abs(dmin_ref) < DEG) | (np.abs(dmin_ref - d_safe) < DEG)
    return bad.any(axis=1)


SMALL = {
    "cfg1": lambda: W.cfg1(K=300, T=16),
    "cfg2": lambda: W.cfg2(K=512, T=20, N=3000),
    "cfg3": lambda: W.cfg3(K=256, T=20, N=4000),
    "cfg5": lambda: W.cfg5(K=256, T=16, N=4000),
    # a horizon whose lane-per-rollout tiles exceed shared memory: the warp-per-rollout kernel
    "cfg5_long": lambda: W.cfg5(K=64, T=600, N=2000),
}


@pytest.mark.parametrize("cfg", list(SMALL))
def test_evaluate_rollouts_injected_noise(cfg):
    wl = SMALL[cfg]()
    eng, orc = engine_and_oracle(wl)
    D = wl.model.control_dim()
    eps = orc.sample_perturbations(1, 0)
    nom = 0.2 * np.ones(wl.params.horizon * D)
    up = np.full(3, 0.05)
    got = eng.evaluate_rollouts(wl.q0, nom, eps, wl.obstacles(), wl.guidance, up)
    want = orc.evaluate_rollouts(wl.q0, nom, eps, wl.cloud, None, wl.guidance, up)
    # FP64 dynamics rounded exactly as the reference (exm_dynamics.cu, no FMA contraction):
    # clamped controls bit-identical; states differ only by CUDA vs glibc sin/cos/tan ulps
    assert np.array_equal(got.controls, want["controls"])
    assert np.allclose(got.states, want["states"], rtol=1e-12, atol=1e-12)
    assert sd_close(got.d_min, want["d_min"]) <= SD_TOL
    assert sign_mismatch(got.d_min, want["d_min"]) == 0
    deg = degenerate_rows(want["d_min"], wl.params.d_safe)
    ok = ~deg
    rel = np.abs(got.costs - want["costs"]) / np.maximum(np.abs(want["costs"]), 1.0)
    assert np.max(rel[ok]) <= 1e-5
    assert np.array_equal(got.unsafe[ok], want["unsafe"][ok])


def test_device_noise_matches_reference_keying():
    wl = W.cfg5(K=64, T=10, N=100)
    eng, orc = engine_and_oracle(wl)
    for seed, cyc in ((1, 0), (42, 3), (2 ** 40 + 7, 11)):
        got, want = eng.sample_perturbations(seed, cyc), orc.sample_perturbations(seed, cyc)
        assert np.allclose(got, want, rtol=1e-12, atol=1e-14)


@pytest.mark.parametrize("cfg", list(SMALL))
@pytest.mark.parametrize("injected", [True, False])
def test_control_cycle_vs_oracle(cfg, injected):
    wl = SMALL[cfg]()
    eng, orc = engine_and_oracle(wl)
    D = wl.model.control_dim()
    nom_g, up_g = wl.zero_state()
    nom_o, up_o = nom_g.copy(), up_g.copy()
    q = wl.q0.copy()
    for cyc in range(3):
        eps = orc.sample_perturbations(wl.params.seed, cyc) if injected else None
        # cost-cliff degeneracy of this step (oracle rollouts on the same noise and state)
        e_used = eps if eps is not None else orc.sample_perturbations(wl.params.seed, cyc)
        roll = orc.evaluate_rollouts(q, nom_o, e_used, wl.cloud, None, wl.guidance, up_o)
        deg = degenerate_rows(roll["d_min"], wl.params.d_safe)
        g = eng.control_cycle_raw(q, wl.obstacles(), wl.guidance, nom_g, up_g, cyc, eps)
        o = orc.control_cycle(q, wl.cloud, None, wl.guidance, nom_o, up_o, cyc, eps)
        if deg[o["argmin"]]:
            pytest.skip(f"cycle {cyc}: argmin rollout is boundary-degenerate")
        assert g.validated == o["validated"], cyc
        assert g.argmin == o["argmin"], (cyc, g.argmin, o["argmin"])
        assert np.max(np.abs(g.command - o["command"][:D])) <= 1e-5
        assert np.max(np.abs(nom_g - nom_o)) <= 1e-5
        assert abs(g.best_cost - o["best_cost"]) <= 1e-5 * max(1.0, abs(o["best_cost"]))
        assert abs(g.weight_entropy - o["weight_entropy"]) <= 1e-5 * max(1.0, o["weight_entropy"])
        assert abs(g.nominal_cost - o["nominal_cost"]) <= 1e-5 * max(1.0, abs(o["nominal_cost"]))
        assert sd_close(g.nominal_d_min, o["nominal_d_min"]) <= SD_TOL
        q = orc.step(q, g.command)
        # keep the oracle on the GPU's state so a last-bit divergence cannot compound
        nom_o[:] = nom_g
        up_o[:] = up_g


def test_validate_nominal_vs_oracle():
    wl = W.cfg2(K=64, T=20, N=3000)
    eng, orc = engine_and_oracle(wl)
    D = wl.model.control_dim()
    for v in (0.0, 0.5, 1.5):
        nom = np.tile([v, 0.1], wl.params.horizon)[: wl.params.horizon * D]
        g = eng.validate_nominal(nom, wl.q0, wl.obstacles(), wl.guidance, np.zeros(3))
        o = orc.validate_nominal(nom, wl.q0, wl.cloud, None, wl.guidance, np.zeros(3))
        assert g[0] == o[0]
        assert sd_close(g[1], o[1]) <= SD_TOL
        assert abs(g[2] - o[2]) <= 1e-5 * max(1.0, abs(o[2]))


def test_resident_steps_equal_host_api_steps():
    """exm_run_resident (CUDA graph on resident inputs) == repeated exm_control_cycle calls."""
    wl = W.cfg2(K=512, T=16, N=2000)
    eng, _ = engine_and_oracle(wl)
    nom, up = wl.zero_state()
    for cyc in range(4):
        d = eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom, up, cyc)
    eng2, _ = engine_and_oracle(wl)
    n2, u2 = wl.zero_state()
    eng2.stage(wl.q0, wl.obstacles(), wl.guidance, n2, u2, 0)
    eng2.run_resident(4)
    r = eng2.read_resident()
    assert np.array_equal(r.command, d.command)
    assert np.array_equal(r.nominal.reshape(-1), nom)
    assert r.argmin == d.argmin and r.best_cost == d.best_cost


def test_bitwise_determinism():
    wl = W.cfg3(K=512, T=12, N=3000)
    eng, _ = engine_and_oracle(wl)
    outs = []
    for _ in range(3):
        nom, up = wl.zero_state()
        d = eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom, up, 5)
        outs.append((d.command.copy(), nom.copy(), d.best_cost, d.weight_entropy, d.argmin))
    for o in outs[1:]:
        for a, b in zip(o, outs[0]):
            assert np.array_equal(a, b)


def test_edge_cases():
    # K not a multiple of the 256-rollout block, T=1, single guidance point, one obstacle point
    wl = W.cfg1(K=300, T=1)
    wl.guidance = Guidance([[1.0, 0.0]], [2.0, 0.0, 0.0])
    wl.cloud = np.array([[-5.0, 0.4]])
    eng, orc = engine_and_oracle(wl)
    nom_g, up_g = wl.zero_state()
    nom_o, up_o = nom_g.copy(), up_g.copy()
    g = eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom_g, up_g, 0)
    o = orc.control_cycle(wl.q0, wl.cloud, None, wl.guidance, nom_o, up_o, 0)
    assert g.argmin == o["argmin"] and g.validated == o["validated"]
    assert np.max(np.abs(g.command - o["command"][:2])) <= 1e-5
    # all points masked: every clearance is kEmptyMaskDistance, nothing unsafe
    wl2 = W.cfg2(K=256, T=8, N=400)
    eng2, orc2 = engine_and_oracle(wl2)
    eps = orc2.sample_perturbations(1, 0)
    from paper_2605_29663_b200.api import ObstacleSet
    masked = ObstacleSet(wl2.cloud, np.zeros(wl2.n_points, np.uint8))
    r = eng2.evaluate_rollouts(wl2.q0, np.zeros(16), eps, masked, wl2.guidance, np.zeros(3))
    assert np.all(r.d_min == 1e6) and np.all(r.unsafe == 0)


def test_safe_stop_enclosed():  # test_controller.cpp:338-355 on the device
    from tests.test_oracle_kat import diff_limits, square
    p = MppiParams(rollouts=256, horizon=10, d_safe=0.1, seed=9)
    eng = Engine(W.MotionModel.diff(), diff_limits(), square(0.4), p, n_cap=64, guide_cap=4)
    a = 2 * np.pi * np.arange(32) / 32
    ring = np.stack([0.45 * np.cos(a), 0.45 * np.sin(a)], 1)
    nom, up = np.zeros(20), np.zeros(3)
    d = eng.control_cycle_raw([0, 0, 0], ring, Guidance([[0, 0], [3, 0]], [3, 0, 0]), nom, up, 0)
    assert not d.validated and np.all(d.command == 0) and np.all(nom == 0)


def test_full_size_cfg2_sampled_parity():
    """Full config-2 shapes (K=4096, T=50, N=10k): every d_min is checked on a seeded sample of
    poses against the oracle, the softmax/argmin against the oracle's weights on the GPU costs."""
    wl = W.cfg2()
    eng, orc = engine_and_oracle(wl)
    D = wl.model.control_dim()
    eps = orc.sample_perturbations(1, 0)
    nom, up = wl.zero_state()
    r = eng.evaluate_rollouts(wl.q0, nom, eps, wl.obstacles(), wl.guidance, up)
    rng = np.random.default_rng(0)
    idx = rng.choice(wl.params.rollouts * wl.params.horizon, 600, replace=False)
    st = r.states[:, :-1, :].reshape(-1, 3)[idx]
    want = orc.sdf_batch(st, wl.cloud)
    assert sd_close(r.d_min.reshape(-1)[idx], want) <= SD_TOL
    nom2, up2 = wl.zero_state()
    d = eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom2, up2, 0, eps)
    aug = r.costs + wl.params.w_inf * r.unsafe
    assert d.argmin == int(np.argmin(aug))
    assert abs(d.best_cost - aug.min()) <= 1e-9 * max(1.0, abs(aug.min()))


def test_pregenerated_noise_is_the_drawn_noise():
    """The next cycle's noise is generated in the tail of each step (k_noise_pregen) and used
    by the next rollout when its cycle matches: consecutive device-noise cycles, a jump in the
    cycle sequence (no pregenerated match) and a repeat after injected noise must all equal the
    same cycles run with that cycle's noise injected (exm_sample_perturbations), bit for bit."""
    wl = W.cfg2(K=512, T=16, N=2000)
    eng, _ = engine_and_oracle(wl)
    ref, _ = engine_and_oracle(wl)
    nom, up = wl.zero_state()
    nom_r, up_r = wl.zero_state()
    for cyc in [0, 1, 2, 3, 9, 10, 10, 11]:
        d = eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom, up, cyc)
        eps = ref.sample_perturbations(wl.params.seed, cyc)
        r = ref.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, nom_r, up_r, cyc, eps)
        assert np.array_equal(d.command, r.command), cyc
        assert np.array_equal(nom, nom_r), cyc
        assert d.argmin == r.argmin and d.best_cost == r.best_cost, cyc
        assert d.weight_entropy == r.weight_entropy, cyc


def _guidance_cases(q0, goal):
    x, y = float(q0[0]), float(q0[1])
    a, b = [x - 1.0, y + 0.3], [x + 4.0, y + 0.3]
    return {
        # segment 2 repeats segment 0 exactly: equal distances, the first segment's progress wins
        "repeated_segment": [a, b, a, b],
        "zero_length_segments": [a, a, [x + 1.0, y], [x + 1.0, y], b],
        "vertex_at_start_pose": [[x - 2.0, y], [x, y], [x + 2.0, y + 2.0]],
        "single_point": [[x + 3.0, y - 1.0]],
        "doubled_back": [a, b, a],
    }


@pytest.mark.parametrize("case", ["repeated_segment", "zero_length_segments",
                                  "vertex_at_start_pose", "single_point", "doubled_back"])
def test_task_cost_polyline_edge_cases(case):
    """Polyline projection (controller.cpp:50-66) in the rollout costs: zero-length segments,
    exact ties between segments (first segment kept), a single guide point."""
    wl = W.cfg1(K=256, T=16)
    path = _guidance_cases(wl.q0, wl.guidance.goal)[case]
    wl.guidance = Guidance(np.asarray(path, np.float64), wl.guidance.goal)
    eng, orc = engine_and_oracle(wl)
    D = wl.model.control_dim()
    eps = orc.sample_perturbations(3, 0)
    nom = 0.3 * np.ones(wl.params.horizon * D)
    up = np.zeros(3)
    got = eng.evaluate_rollouts(wl.q0, nom, eps, wl.obstacles(), wl.guidance, up)
    want = orc.evaluate_rollouts(wl.q0, nom, eps, wl.cloud, None, wl.guidance, up)
    ok = ~degenerate_rows(want["d_min"], wl.params.d_safe)
    rel = np.abs(got.costs - want["costs"]) / np.maximum(np.abs(want["costs"]), 1.0)
    assert ok.any() and np.max(rel[ok]) <= 1e-5
    g = eng.validate_nominal(nom, wl.q0, wl.obstacles(), wl.guidance, up)
    o = orc.validate_nominal(nom, wl.q0, wl.cloud, None, wl.guidance, up)
    assert g[0] == o[0] and abs(g[2] - o[2]) <= 1e-5 * max(1.0, abs(o[2]))


@pytest.mark.parametrize("n", [1, 2047, 65536 + 3, 300_001])
@pytest.mark.parametrize("threads", [1, 3, 8])
def test_batch_signed_distance_pipeline_chunks(n, threads):
    """exm_batch_signed_distance's pipeline (up to 8 chunks of >= 64k queries over three
    slot streams, host threads staging FP32 / widening FP64): every query, odd sizes and chunk
    boundaries, each host thread count, against the oracle (geometry.cpp:298-318)."""
    from paper_2605_29663_b200 import _abi
    wl = W.cfg1(K=4, T=2)
    wl.footprint = W.footprint("t_shape")
    eng, orc = engine_and_oracle(wl)
    eng.set_option(_abi.OPT_HOST_THREADS, threads)
    q = W.benchmark_queries(n, 12.0, 5 + n)
    got = eng.batch_signed_distance(q)
    want = orc.batch_signed_distance(q)
    assert got.shape == want.shape
    assert sd_close(got, want) <= SD_TOL and sign_mismatch(got, want) == 0
    again = eng.batch_signed_distance(q)  # buffers reused: identical
    assert np.array_equal(got, again)


def test_sdf_batch_recentres_on_device():
    """exm_sdf_stage: poses and points recentred at the poses' centroid on the device (no host
    loop); far-from-origin inputs keep the 1e-5 bound, the run/read split equals one-shot."""
    wl = W.cfg2(K=4, T=2, N=800)
    eng, orc = engine_and_oracle(wl)
    shift = np.array([1.5e3, -2.25e3])
    poses = W.cfg4_poses(64) * np.array([0.5, 0.5, 1.0]) + np.r_[shift, 0.0]
    pts = wl.cloud + shift
    mins = eng.sdf_batch(poses, pts)
    want = orc.sdf_batch(poses, pts)
    assert sd_close(mins, want) <= SD_TOL
    eng.sdf_stage(poses, pts)
    eng.sdf_run_resident(3, False)
    m2, _ = eng.sdf_read()
    assert np.array_equal(m2, mins)
    st = eng.step_stats()
    assert st["sdf_ms"] > 0 and st["launches_per_step"] == 3


def test_sdf_timing_ring_is_bounded():
    """Round 1 leaked two events per exm_sdf_batch call; the ring now folds at 512 entries and
    one-shot calls never use it: thousands of calls keep working and step_stats stays valid."""
    wl = W.cfg2(K=4, T=2, N=200)
    eng, _ = engine_and_oracle(wl)
    poses = W.cfg4_poses(8)
    for _ in range(1500):
        eng.sdf_batch(poses, wl.cloud)
    eng.sdf_stage(poses, wl.cloud)
    eng.sdf_run_resident(1200, False)  # more than one fold of the resident ring
    st = eng.step_stats()
    assert st["sdf_ms"] > 0.0


def test_option_and_argument_errors():
    from paper_2605_29663_b200 import _abi
    wl = W.cfg2(K=256, T=8, N=100)
    eng, _ = engine_and_oracle(wl)
    with pytest.raises(ValueError, match="unknown option"):
        eng.set_option(99, 1)
    with pytest.raises(ValueError, match="SDF mode"):
        eng.set_option(_abi.OPT_SDF_MODE, 42)
    with pytest.raises(ValueError, match="mapping"):
        eng.set_option(_abi.OPT_SDF_MAP, 7)
    nom, up = wl.zero_state()
    with pytest.raises(ValueError):  # nominal of the wrong length (checked before the ABI call)
        eng.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, np.zeros(5), up, 0)
    from paper_2605_29663_b200.api import ObstacleSet
    with pytest.raises(ValueError, match="mask length"):
        ObstacleSet(wl.cloud, np.ones(3, np.uint8))


def test_concurrent_calls_on_one_handle_serialise():
    """Every ABI call holds its handle's lock (ctypes releases the GIL, so the four threads below
    really call concurrently): each thread's sequence of control cycles on the shared handle
    equals the same sequence run alone."""
    import threading
    wl = W.cfg2(K=512, T=12, N=1500)
    shared, _ = engine_and_oracle(wl)
    alone, _ = engine_and_oracle(wl)
    qs = [wl.q0 + np.array([0.1 * t, -0.05 * t, 0.02 * t]) for t in range(4)]
    want = []
    for t in range(4):
        nom, up = wl.zero_state()
        want.append([alone.control_cycle_raw(qs[t], wl.obstacles(), wl.guidance, nom, up, 10 * t + c).command
                     for c in range(5)])
    got = [None] * 4
    obst = wl.obstacles()

    def run(t):
        nom, up = wl.zero_state()
        got[t] = [shared.control_cycle_raw(qs[t], obst, wl.guidance, nom, up, 10 * t + c).command
                  for c in range(5)]
    th = [threading.Thread(target=run, args=(t,)) for t in range(4)]
    for x in th:
        x.start()
    for x in th:
        x.join()
    for t in range(4):
        for c in range(5):
            assert np.array_equal(got[t][c], want[t][c]), (t, c)


def test_pinned_obstacle_set_same_decisions():
    """ObstacleSet.pinned (exm_host_alloc page-locked buffers, DMA uploads) gives the same
    decisions as pageable numpy buffers; its arrays outlive the ObstacleSet object."""
    from paper_2605_29663_b200.api import ObstacleSet
    wl = W.cfg2(K=1024, T=30, N=10_000)
    obst = wl.obstacles()
    pinned = ObstacleSet.pinned(obst.points, obst.mask)
    pts_view = pinned.points
    assert np.array_equal(pts_view, obst.points) and np.array_equal(pinned.mask, obst.mask)
    outs = []
    for o in (obst, pinned):
        eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)
        nom, up = wl.zero_state()
        outs.append([eng.control_cycle_raw(wl.q0, o, wl.guidance, nom, up, c) for c in range(3)])
        eng.close()
    for a, b in zip(*outs):
        assert np.array_equal(a.command, b.command) and a.argmin == b.argmin
        assert a.best_cost == b.best_cost
    del pinned
    import gc
    gc.collect()
    assert np.array_equal(pts_view, obst.points)  # the view keeps the allocation alive
