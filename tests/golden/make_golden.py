"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref/libexm_ref.so, built
from /root/reference/proj sources by oracle/Makefile). Run in the dev container:

    python tests/golden/make_golden.py

Inputs are the seeded synthetic workloads of paper_2605_29663_b200.workloads (Appendix A of
SURVEY.md), shrunk so the fixtures stay small.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from paper_2605_29663_b200 import workloads as W  # noqa: E402
from tests import oracle_bindings as ob  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

FOOTPRINTS = {**{n: (lambda n=n: W.footprint(n)) for n in W.GALLERY + list(W.RECT_FOOTPRINTS)},
              "l12": W.l12_footprint, "star64": W.star64_footprint,
              "forklift": W.forklift_footprint}

SMALL = {
    "cfg1": lambda: W.cfg1(K=48, T=12),
    "cfg2": lambda: W.cfg2(K=48, T=12, N=1500),
    "cfg3": lambda: W.cfg3(K=48, T=12, N=1500),
    "cfg5": lambda: W.cfg5(K=48, T=12, N=1500),
}


def main():
    base = W.cfg1(K=4, T=2)
    sd = {}
    q = W.benchmark_queries(512, 6.0, 99)
    sd["queries"] = q
    for name, mk in FOOTPRINTS.items():
        r = ob.Reference(mk(), base.model, base.limits, base.params)
        sd[name] = r.batch_signed_distance(q)
    np.savez_compressed(os.path.join(OUT, "sd_footprints.npz"), **sd)

    wl = W.cfg2(K=4, T=2, N=2000)
    r = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params)
    mask = (np.arange(wl.n_points) % 5 != 1).astype(np.uint8)
    poses = W.cfg4_poses(256) * np.array([1.2, 1.2, 1.0])
    r.set_cloud(wl.cloud, mask)
    np.savez_compressed(os.path.join(OUT, "min_sd_cfg2.npz"), cloud=wl.cloud, mask=mask,
                        poses=poses, d_min=r.min_sd_at(poses))

    for name, mk in SMALL.items():
        wl = mk()
        r = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params)
        D = wl.model.control_dim()
        eps = r.sample_perturbations(wl.params.seed, 0)
        nom = 0.15 * np.ones(wl.params.horizon * D)
        up = np.full(3, 0.05)
        out = r.evaluate_rollouts(wl.q0, nom, eps, wl.cloud, None, wl.guidance, up)
        np.savez_compressed(os.path.join(OUT, f"rollouts_{name}.npz"), eps=eps, nominal=nom,
                            u_prev=up, **out)

    for name in ("cfg1", "cfg2"):
        wl = SMALL[name]()
        r = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params)
        rows = {k: [] for k in ("q", "command", "validated", "best_cost", "weight_entropy",
                                "nominal_cost", "nominal_d_min", "nominal")}
        qq = wl.q0.copy()
        orc = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
        for _ in range(3):
            d = r.controller_cycle(qq, wl.cloud, None, wl.guidance)
            rows["q"].append(qq.copy())
            for k in ("command", "validated", "best_cost", "weight_entropy", "nominal_cost",
                      "nominal_d_min", "nominal"):
                rows[k].append(d[k])
            qq = orc.step(qq, d["command"][: wl.model.control_dim()])
        np.savez_compressed(os.path.join(OUT, f"cycles_{name}.npz"),
                            **{k: np.array(v) for k, v in rows.items()})
    print("golden fixtures written to", OUT)


if __name__ == "__main__":
    main()
