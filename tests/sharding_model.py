"""TEST INFRASTRUCTURE: host-side restatement (numpy) of the rollout sharding and the
softmax-partial exchange that libexm_b200.so performs on the device (k_block_partials /
k_update, exm_attach_comm / exm_sharded_cycle). The world-size-2 gloo test
(tests/test_sharding_cpu.py) runs this model over a real process group on CPU; the library's own
sharded path is tested on the GPU (tests/test_gpu_sharding.py).

Rollouts are split into fixed blocks of BLOCK = 256 (independent of the GPU count); rank g of G
owns blocks [g*nb/G, (g+1)*nb/G). Each block b yields {beta_b, S_b, A_b, argmin_b, U_b}; the
ranks all-gather the partials and every rank merges them in block order, so the merged update
is bit-identical for every G. The reference equivalent is the weights_from_costs + weighted
update of MppiController::control_cycle (controller.cpp:310-328).
"""
from __future__ import annotations

import numpy as np

BLOCK = 256


def shard_range(K: int, rank: int, world: int) -> tuple[int, int]:
    if K % (BLOCK * world) and world > 1:
        raise ValueError("rollouts must be a multiple of 256 * world for sharding")
    k = K // world
    return rank * k, (rank + 1) * k


def block_partials(costs_aug: np.ndarray, eps: np.ndarray, r0: int, lam: float) -> np.ndarray:
    """Partials of consecutive blocks of one shard. costs_aug: (k,), eps: (k, T*D) for global
    rollouts r0..r0+k. Row layout: [beta, S, A, argmin, U...] (exm_common.cuh partial_stride)."""
    k = costs_aug.shape[0]
    TD = eps.shape[1]
    nb = (k + BLOCK - 1) // BLOCK
    out = np.zeros((nb, 4 + TD))
    for b in range(nb):
        J = costs_aug[b * BLOCK:(b + 1) * BLOCK]
        E = eps[b * BLOCK:(b + 1) * BLOCK]
        j = int(np.argmin(J))  # first index of the minimum
        beta = J[j]
        z = (J - beta) / lam
        e = np.exp(-z)
        out[b, 0], out[b, 1], out[b, 2], out[b, 3] = beta, e.sum(), (e * z).sum(), r0 + b * BLOCK + j
        out[b, 4:] = e @ E
    return out


def merge_partials(P: np.ndarray, lam: float):
    """Block-order merge: beta, argmin, entropy H = A/S + log S, weighted update U/S."""
    b = int(np.argmin(P[:, 0]))
    beta = P[b, 0]
    f = np.exp(-(P[:, 0] - beta) / lam)
    S = float((f * P[:, 1]).sum())
    A = float((f * (P[:, 2] + P[:, 1] * (P[:, 0] - beta) / lam)).sum())
    U = (f[:, None] * P[:, 4:]).sum(axis=0)
    return {"beta": float(beta), "argmin": int(P[b, 3]), "entropy": A / S + np.log(S),
            "delta": U / S}
