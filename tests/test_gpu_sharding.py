"""The library's own sharded path on one GPU (replaces the reference's fork-join
over rollouts, proj/src/controller.cpp:207-218).

* A 1-rank NCCL communicator (exm_attach_comm with an id at world 1) puts the in-place
  ncclAllGather of the softmax block partials into the step graph: dlopen of libnccl, graph
  capture of the collective and its execution all run, and the decisions must equal an
  unattached handle's bit for bit.
* G shard handles on one device (exm_set_shard + exm_sharded_cycle) run rank g's rollouts each
  (k_block_partials with block_offset != 0, k_update merging every rank's blocks) and exchange
  the block partials with one device-to-device copy per block where the ranks' all-gather runs:
  every shard's decision must equal the unsharded decision bit for bit, for G = 1, 2, 4, 8, at
  the full config-2 and config-5 sizes, over consecutive cycles with device-drawn noise.
"""
import numpy as np
import pytest

from paper_2605_29663_b200 import workloads as W
from paper_2605_29663_b200.api import Engine

pytestmark = pytest.mark.gpu


def _engine(wl):
    return Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=wl.n_points, guide_cap=8)


def _same(a, b):
    assert np.array_equal(a.command, b.command), (a.command, b.command)
    assert a.argmin == b.argmin and a.validated == b.validated
    assert a.best_cost == b.best_cost and a.weight_entropy == b.weight_entropy
    assert a.nominal_cost == b.nominal_cost
    assert np.array_equal(a.nominal_d_min, b.nominal_d_min)


def test_one_rank_nccl_allgather_in_graph():
    wl = W.cfg2(K=1024, T=20, N=3000)
    plain, comm = _engine(wl), _engine(wl)
    comm.attach_comm(0, 1, Engine.nccl_unique_id())
    n1, u1 = wl.zero_state()
    n2, u2 = wl.zero_state()
    for cyc in range(3):
        a = plain.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, n1, u1, cyc)
        b = comm.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, n2, u2, cyc)
        _same(a, b)
        assert np.array_equal(n1, n2) and np.array_equal(u1, u2)
    # resident stepping runs the same captured graph (collective included)
    comm.stage(wl.q0, wl.obstacles(), wl.guidance, *wl.zero_state(), 0)
    comm.run_resident(3)
    r = comm.read_resident()
    assert np.array_equal(r.command, a.command)
    comm.attach_comm(0, 1, None)  # detach: unsharded again
    n3, u3 = wl.zero_state()
    c = comm.control_cycle_raw(wl.q0, wl.obstacles(), wl.guidance, n3, u3, 0)
    assert np.array_equal(c.command, plain.control_cycle_raw(
        wl.q0, wl.obstacles(), wl.guidance, *wl.zero_state(), 0).command)


FULL = {"cfg2": lambda: W.cfg2(), "cfg5": lambda: W.cfg5()}


@pytest.mark.parametrize("cfg", list(FULL))
def test_sharded_decisions_bitwise_equal_for_every_G(cfg):
    wl = FULL[cfg]()
    D = wl.model.control_dim()
    TD = wl.params.horizon * D
    ref = _engine(wl)
    nom, up = wl.zero_state()
    want = []
    q = wl.q0.copy()
    qs = []
    for cyc in range(3):
        qs.append(q.copy())
        d = ref.control_cycle_raw(q, wl.obstacles(), wl.guidance, nom, up, cyc)
        want.append((d, nom.copy(), up.copy()))
        q = q + np.array([0.05, 0.01, 0.02])  # a new start pose each cycle
    ref.close()
    for G in (1, 2, 4, 8):
        shards = [_engine(wl) for _ in range(G)]
        for g, e in enumerate(shards):
            e.set_shard(g, G)
        noms = np.zeros((G, TD))
        ups = np.zeros((G, 3))
        for cyc in range(3):
            got = Engine.sharded_cycle(shards, qs[cyc], wl.obstacles(), wl.guidance, noms, ups, cyc)
            w, wn, wu = want[cyc]
            for g in range(G):
                _same(got[g], w)
                assert np.array_equal(noms[g], wn) and np.array_equal(ups[g], wu), (G, g, cyc)
        for e in shards:
            e.close()


def test_shard_argument_checks():
    wl = W.cfg2(K=1000, T=8, N=500)
    e = _engine(wl)
    with pytest.raises(ValueError):
        e.set_shard(0, 2)  # K not a multiple of 256 * G
    wl2 = W.cfg2(K=512, T=8, N=500)
    a, b = _engine(wl2), _engine(wl2)
    a.set_shard(0, 2)
    b.set_shard(1, 2)
    nom, up = wl2.zero_state()
    with pytest.raises(ValueError):  # a shard without a communicator cannot step alone
        a.control_cycle_raw(wl2.q0, wl2.obstacles(), wl2.guidance, nom, up, 0)
    with pytest.raises(ValueError):  # shard order must match ranks
        Engine.sharded_cycle([b, a], wl2.q0, wl2.obstacles(), wl2.guidance,
                             np.zeros((2, 16)), np.zeros((2, 3)), 0)
