"""world_size-2 gloo test of the rollout sharding + softmax-partial all-gather (the exchange
libexm_b200.so does with one NCCL all-gather), on CPU with oracle-evaluated rollouts."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from tests import sharding_model as S
from paper_2605_29663_b200 import workloads as W
from tests import oracle_bindings as ob

K, T = 1024, 10


def problem():
    wl = W.cfg2(K=K, T=T, N=1500)
    orc = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
    eps = orc.sample_perturbations(1, 0)
    nom, up = wl.zero_state()
    r = orc.evaluate_rollouts(wl.q0, nom, eps, wl.cloud, None, wl.guidance, up)
    aug = r["costs"] + wl.params.w_inf * r["unsafe"]
    return wl, eps.reshape(K, -1), aug


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    wl, eps, aug = problem()
    lo, hi = S.shard_range(K, rank, world)
    mine = torch.from_numpy(S.block_partials(aug[lo:hi], eps[lo:hi], lo, wl.params.lambda_))
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine)
    merged = S.merge_partials(torch.cat(parts).numpy(), wl.params.lambda_)
    q.put((rank, merged))
    dist.destroy_process_group()


def test_two_rank_allgather_is_bit_identical_to_one_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    wl, eps, aug = problem()
    single = S.merge_partials(S.block_partials(aug, eps, 0, wl.params.lambda_), wl.params.lambda_)
    for r in (0, 1):
        assert res[r]["argmin"] == single["argmin"]
        assert res[r]["beta"] == single["beta"]
        assert np.array_equal(res[r]["delta"], single["delta"])
        assert res[r]["entropy"] == single["entropy"]


def test_partials_merge_matches_reference_update():
    """Block-order merge == the reference's weights_from_costs + in-place weighted update
    (controller.cpp:314-328) to rounding, and the argmin/beta exactly."""
    wl, eps, aug = problem()
    merged = S.merge_partials(S.block_partials(aug, eps, 0, wl.params.lambda_), wl.params.lambda_)
    w = ob.oracle_weights(aug, wl.params.lambda_)
    assert merged["argmin"] == int(np.argmin(aug)) and merged["beta"] == aug.min()
    delta = w @ eps
    assert np.allclose(merged["delta"], delta, rtol=1e-12, atol=1e-15)
    H = -np.sum(w[w > 0] * np.log(w[w > 0]))
    assert abs(merged["entropy"] - H) <= 1e-9 * max(1.0, H)


def test_shard_ranges():
    assert S.shard_range(4096, 3, 8) == (1536, 2048)
    with pytest.raises(ValueError):
        S.shard_range(1000, 0, 2)
