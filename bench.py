#!/usr/bin/env python
"""Benchmark of the B200 EXACT-MPPI hot path (BASELINE.json metric: MPPI control steps/sec and
point-footprint SDF evals/sec).

Workload (N=1 and every N): config 2 of BASELINE.json — 12-vertex L polygon, diff-drive,
K=4096, T=50, N=10k dense static clutter, synthetic, seeded.
A step is one full MPPI control cycle (noise, rollouts, exact SDF over K*T*N pairs, softmax
update, validation, shift). At N GPUs the K rollouts are sharded over the ranks (strong
scaling) with one NCCL all-gather of the softmax partials per step.

  value  device time per step (CUDA events on the library's stream) with inputs resident in
         HBM; L2 is flushed (256 MiB write) before every timed step, outside the events.
  e2e    the same step through the C ABI with host buffers (cloud, state in; decision,
         nominal out), host<->device copies inside the timed region (wall clock).
  roofline  the SDF kernel (k_sdf_grid) on EXECUTED FP32 work: its work counters
         (exm_sdf_work_stats) charged at each unit's FP32 op count, divided by the
         kernel's mean device time in the timed steps and by the measured FP32 peak. The
         unpruned algorithmic work (K*T*N pairs x F ops) over the executed work is reported as
         `culling_factor`.

`--impl reference` times the reference's own CPU implementation (MppiController::control_cycle
of the unmodified reference built into oracle/_ref) on this host's cores at the same config:
full K, a fresh controller per step, all host threads (plus a threads=1 sample and the
config-4 batch_signed_distance evals/s of the same build).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

F_POLY = lambda B: 12 + 19 * B  # noqa: E731  algorithmic ops per point-pose pair
F_RECT = lambda R: 9 + 16 * R   # noqa: E731


def ops_per_pair(fp) -> int:
    return F_POLY(fp.count()) if fp.is_polygon() else F_RECT(fp.count())


def cover_is_exact(fp) -> bool:
    """The polygon's cull cover tiles it exactly (rectilinear: the L), as exm_create decides."""
    if not fp.is_polygon():
        return False
    _, boxes = fp.cull_boxes()
    m = 1e-4 * (1.0 + fp.bounding_radius())  # slack added to the cull boxes (exm_abi.cu)
    area = float(np.sum((2 * (boxes[:, 2] - m)) * (2 * (boxes[:, 3] - m))))
    x, y = fp.a[:, 0], fp.a[:, 1]
    poly = 0.5 * abs(float(np.dot(x, np.roll(y, -1)) - np.dot(y, np.roll(x, -1))))
    return abs(area - poly) <= 1e-4 * poly


def executed_ops(counts: dict, fp) -> tuple[float, dict]:
    """FP32 ops executed by k_sdf_grid: each counted unit (exm_sdf_work_stats) at its op count,
    FMA = 2, as written in csrc/exm_kernels.cu (DESIGN.md §4 derives each figure):
      ring step 27 per lane (x32, counted per warp), cell bound 33, chunk bound 63, point circle
      test 6, body-frame transform 6, exact-cover tile test 44, tile value 7, cover/AABB bound
      8 (exact cover: interior AABB test) / 41 (polygon cover) / 15 (rect AABB), edge or box
      loop F - 8 (the reference-literal pair cost without its transform) + 2."""
    F = ops_per_pair(fp)
    bound = 8 if cover_is_exact(fp) else (41 if fp.is_polygon() else 15)
    per = {"ring_steps": 27 * 32, "cell_tests": 33, "chunk_tests": 63, "point_tests": 6,
           "point_iters_warp": 0, "transforms": 6, "tile_tests": 44, "tile_values": 7,
           "bound_tests": bound, "edge_loops": F - 8 + 2}
    parts = {k: counts[k] * per[k] for k in per}
    return float(sum(parts.values())), per


def bench_config(wl, world: int) -> dict:
    """The config dict both arms print (the driver compares them)."""
    fp = wl.footprint
    return {"workload": wl.name, "K": wl.params.rollouts, "T": wl.params.horizon,
            "N": wl.n_points,
            "footprint": f"{fp.name} ({'polygon B' if fp.is_polygon() else 'cover R'}={fp.count()})",
            "model": ["diff", "ackermann", "omni", "spin", "parallel"][wl.model.tag],
            "parallelism": f"K sharded over {world} GPU(s) (reference arm: host threads)",
            "l2": "GPU arm: flushed (256 MiB write) before every timed device step"}


def fp32_peak_tflops(sm_count: int = 148) -> tuple[float, str]:
    """FP32 SIMT peak. MEASURED_PEAKS.json holds only HBM and bf16 peaks, so the FP32 number is
    measured on this pool's B200 by tools/fp32_peak.cu (independent packed FFMA2 chains on all
    SMs; committed as profiles/r01_fp32_peak.json). Fallback: 2 flops/FMA x 128 lanes x SMs x
    sm_max_mhz of MEASURED_PEAKS.json."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_fp32_peak.json")))
    if files:
        try:
            d = json.load(open(files[-1]))
            return float(d["fp32_ffma2_tflops"]), (
                f"measured: {os.path.relpath(files[-1], ROOT)} (tools/fp32_peak.cu, FFMA2 chains, "
                f"{d['sms']} SMs; nominal {d['nominal_tflops_at_max_clock']} at {d['max_clock_mhz']} MHz)")
        except Exception:
            pass
    mhz = 1965.0
    src = "derived: 256 ops/SM/clk x %d SMs x sm_max_mhz" % sm_count
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            mhz = float(json.load(f).get("sm_max_mhz", mhz))
        src += " (MEASURED_PEAKS.json)"
    except Exception:
        src += " (fallback 1965 MHz)"
    return 256.0 * sm_count * mhz * 1e6 / 1e12, src


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.12)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [r for r in self.rows if len(r) == 6 and r[0].isdigit()]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(float(r[0]) for r in rows),
                "sm_max_mhz": max(float(r[1]) for r in rows), "reasons": reasons,
                "samples": len(rows)}


def ncu_profile(name: str) -> dict:
    """Per-launch DRAM traffic and executed pipe utilisation of a kernel from the newest
    committed `ncu --set full` summary (profiles/rNN_ncu_<name>.json, tools/ncu_summary.py)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_{name}.json")))
    if not files:
        return {}
    try:
        kern = next(iter(json.load(open(files[-1])).values()))[0]

        def num(key):
            v = kern.get(key, "")
            x, _, unit = v.partition(" ")
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(x.replace(",", "")) * scale
        return {"traffic": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
                "executed": {"source": os.path.relpath(files[-1], ROOT),
                             "fma_pipe_active_pct": num("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                             "alu_pipe_active_pct": num("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                             "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active")}}
    except Exception:
        return {}


def dist_setup():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        import torch
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def reference_steps(wl, threads: int, n_steps: int, warmup: int = 0, min_seconds: float = 0.0,
                    max_seconds: float = 1e9):
    """Wall times of MppiController::control_cycle of the unmodified reference (oracle/_ref) at
    the FULL workload (K, T, N as configured), a fresh controller (zero nominal, cycle 0) per
    step, built outside the timed call. Falls back to the C restatement when
    the reference build is absent (kind "port", one thread)."""
    from tests import oracle_bindings as ob
    if ob.reference_available():
        ref = ob.Reference(wl.footprint, wl.model, wl.limits, wl.params, threads=threads)
        ref.set_cloud(wl.cloud)
        kind = "reference"

        def step():
            ref.reset()  # fresh controller, untimed
            t0 = time.perf_counter()
            ref.controller_cycle(wl.q0, None, None, wl.guidance, use_stored_cloud=True)
            return time.perf_counter() - t0
    else:
        orc = ob.Oracle(wl.footprint, wl.model, wl.limits, wl.params)
        threads, kind = 1, "port"

        def step():
            nom, up = wl.zero_state()
            t0 = time.perf_counter()
            orc.control_cycle(wl.q0, wl.cloud, None, wl.guidance, nom, up, 0)
            return time.perf_counter() - t0
    for _ in range(warmup):
        step()
    times = []
    t_end = time.perf_counter() + min_seconds
    t_cap = time.perf_counter() + max_seconds
    while len(times) < n_steps or time.perf_counter() < t_end:
        times.append(step())
        if time.perf_counter() > t_cap and len(times) >= 1:
            break
    return times, threads, kind


def cpu_reference_sample(wl, seconds: float = 10.0):
    """cpu_baseline of the GPU arm: the reference's full-K control_cycle on all host threads for
    about `seconds` (at least 3 steps)."""
    threads = os.cpu_count() or 1
    times, threads, kind = reference_steps(wl, threads, 3, warmup=1, min_seconds=seconds)
    t = statistics.median(times)
    return {"value": 1.0 / t, "unit": "steps/s", "cores": threads, "kind": kind,
            "sample": (f"{len(times)} MppiController::control_cycle calls at the full workload "
                       f"(K={wl.params.rollouts}, T={wl.params.horizon}, N={wl.n_points}), fresh "
                       f"controller each, median {t * 1e3:.1f} ms, {threads} threads, "
                       f"CPU {cpu_model()}"),
            "sec_per_step": t}


def reference_sdf_evals(threads: int, trials: int = 5):
    """Config 4 on the reference's batch_signed_distance (the scaling_benchmark protocol,
    bench.cpp:67-113: 3 warm-ups, then timed trials): 64-vertex star, 10^6 body-frame queries
    (benchmark_queries, 50 m region, seed 1), evals/s."""
    from paper_2605_29663_b200 import workloads as W
    from tests import oracle_bindings as ob
    if not ob.reference_available():
        return None
    wl = W.cfg1(K=8, T=2)
    fp, _, pts = W.cfg4(P=1)
    ref = ob.Reference(fp, wl.model, wl.limits, wl.params, threads=threads)
    for _ in range(3):
        ref.batch_signed_distance(pts, threads)
    ts = []
    for _ in range(trials):
        t0 = time.perf_counter()
        ref.batch_signed_distance(pts, threads)
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return {"workload": "cfg4 star64, batch_signed_distance of 10^6 queries", "threads": threads,
            "median_ms": 1e3 * t, "evals_per_s": pts.shape[0] / t,
            "seconds_for_1e9_pairs": 1e9 / (pts.shape[0] / t)}


def run_reference(args, world, rank):
    """The reference arm: the reference's own CPU control_cycle at the GPU arm's config."""
    from paper_2605_29663_b200 import workloads as W
    if rank != 0:
        return
    wl = {"cfg1": W.cfg1, "cfg2": W.cfg2, "cfg3": W.cfg3, "cfg5": W.cfg5}[args.config]()
    nproc = os.cpu_count() or 1
    times, threads, kind = reference_steps(wl, nproc, args.steps, warmup=args.warmup)
    ms = 1e3 * statistics.mean(times)
    v = 1e3 / ms
    # threads = 1: >= 5 steps, or 1 when a step exceeds 10 s
    t1, _, _ = reference_steps(wl, 1, 1)
    if t1[0] < 10.0:
        more, _, _ = reference_steps(wl, 1, 4, max_seconds=60.0)
        t1 += more
    K, T, N = wl.params.rollouts, wl.params.horizon, wl.n_points
    line = {"metric": "MPPI control steps/sec", "value": v, "unit": "steps/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "ms_per_step_p50": 1e3 * statistics.median(times),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "impl": "reference",
            "config": bench_config(wl, world),
            "cpu_baseline": {"value": v, "unit": "steps/s", "cores": threads, "kind": kind,
                             "sample": (f"{len(times)} full-size MppiController::control_cycle "
                                        f"calls (K={K}, T={T}, N={N}), a fresh controller each, "
                                        f"{threads} threads, CPU {cpu_model()}")},
            "cpu_threads1": {"steps": len(t1), "ms_per_step_median": 1e3 * statistics.median(t1),
                             "steps_per_s": 1.0 / statistics.median(t1)},
            "cpu_model": cpu_model(), "nproc": nproc,
            "e2e": {"value": v, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "sdf_evals_per_s": K * T * N * v,
            "sdf_batch_cfg4": reference_sdf_evals(nproc)}
    print(json.dumps(line), flush=True)


def run_ours(args, world, rank, local):
    import torch
    from paper_2605_29663_b200 import workloads as W
    from paper_2605_29663_b200.api import Engine, ObstacleSet

    wl = {"cfg1": W.cfg1, "cfg2": W.cfg2, "cfg3": W.cfg3, "cfg5": W.cfg5}[args.config]()
    fp = wl.footprint
    K, T, N = wl.params.rollouts, wl.params.horizon, wl.n_points
    D = wl.model.control_dim()
    torch.cuda.set_device(local)
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=N, guide_cap=8, device=local)
    if world > 1:
        import torch.distributed as dist
        obj = [Engine.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        eng.attach_comm(rank, world, obj[0])
    ext = torch.cuda.ExternalStream(eng.stream_ptr())
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    obstacles = wl.obstacles()

    # ---- device-resident steps (value)
    nom, up = wl.zero_state()
    eng.stage(wl.q0, obstacles, wl.guidance, nom, up, 0)
    # at least the handle's lane-mapping tuning steps (6, outside the graph) before the timed region
    eng.run_resident(max(8, args.warmup))
    torch.cuda.synchronize()
    eng.step_stats()  # drop the warm-up launches from the SDF accumulation
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        for i in range(args.steps):
            with torch.cuda.stream(ext):
                flush.zero_()  # L2 flush (256 MiB > 126 MB L2), outside the timed events
                evs[i][0].record(ext)
            eng.run_resident(1)
            with torch.cuda.stream(ext):
                evs[i][1].record(ext)
            if (i + 1) % 16 == 0 or i + 1 == args.steps:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        step_ms = [a.elapsed_time(b) for a, b in evs]
    stats = eng.step_stats()  # SDF kernel mean over exactly the timed steps
    path, vpath = eng.last_sdf_path()
    counts = eng.sdf_work_stats()  # the last timed step's pose set, counters on
    ms_local = float(np.mean(step_ms))
    ms = allreduce_max(ms_local, world)
    value = 1e3 / ms
    dec = eng.read_resident()

    # ---- end to end through the C ABI with host buffers (e2e)
    nom, up = wl.zero_state()
    for c in range(max(3, args.warmup)):
        eng.control_cycle_raw(wl.q0, obstacles, wl.guidance, nom, up, c)
    if world > 1:
        torch.distributed.barrier()
    # config 5 has moving obstacles: the cloud is regenerated every cycle (quasi-static within
    # the horizon) — cycle through 8 pre-generated snapshots so every e2e step
    # uploads a different cloud.
    # input buffers in page-locked host memory (exm_host_alloc): the uploads are DMA from pinned
    # memory as the e2e protocol asks, without the driver's bounce-buffer copy
    clouds = [ObstacleSet.pinned(obstacles.points, obstacles.mask)]
    if args.config == "cfg5":
        clouds = [ObstacleSet.pinned(o.points, o.mask)
                  for o in (W.cfg5(cycle=10 * j).obstacles() for j in range(8))]
    e2e_ms = []
    t0 = time.perf_counter()
    for c in range(args.steps):
        t1 = time.perf_counter()
        eng.control_cycle_raw(wl.q0, clouds[c % len(clouds)], wl.guidance, nom, up, 1000 + c)
        e2e_ms.append(1e3 * (time.perf_counter() - t1))
    e2e_s = allreduce_max((time.perf_counter() - t0) / args.steps, world)
    h2d = 104 + 8 * T * D + 16 * wl.guidance.path.shape[0] + 16 * N + N
    d2h = 64 + 8 * (T + T * D + 3)

    F = ops_per_pair(fp)
    pairs = K // world * T * N
    peak, peak_src = fp32_peak_tflops(torch.cuda.get_device_properties(local).multi_processor_count)
    sdf_avg_ms = stats["sdf_ms"]
    ex_ops, per_unit = executed_ops(counts, fp)
    achieved = ex_ops / (sdf_avg_ms * 1e-3) / 1e12
    algorithmic = pairs * F
    prof = ncu_profile(f"sdf_grid_{args.config}")
    line = {
        "metric": "MPPI control steps/sec", "value": value, "unit": "steps/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "dtype_note": "SDF kernels FP32 on q0-recentred coordinates; dynamics, costs, softmax FP64",
        "ms_per_step_p50": float(np.percentile(step_ms, 50)),
        "ms_per_step_p99": float(np.percentile(step_ms, 99)),
        "data": "synthetic",
        "config": bench_config(wl, world),
        "sdf_evals_per_s": K * T * N / (ms * 1e-3),  # point-pose pairs per second of MPPI step
        "sdf_kernel_evals_per_s": pairs * world / (sdf_avg_ms * 1e-3),  # ... of the SDF kernel
        "e2e": {"value": 1.0 / e2e_s, "unit": "steps/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_p50": float(np.percentile(e2e_ms, 50)),
                "ms_p99": float(np.percentile(e2e_ms, 99)),
                "path": ("Engine.control_cycle_raw -> exm_control_cycle (C ABI): q0/goal/nominal/"
                         "u_prev/guidance via the handle's pinned mirror, the cloud and mask "
                         "DMA'd from the caller's page-locked buffers (ObstacleSet.pinned, "
                         "exm_host_alloc), one graph launch, one D2H of the decision + nominal")},
        "gpu_launches": stats["launches_per_step"] * args.steps,
        "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                     "frac": achieved / peak, "traffic": prof.get("traffic"),
                     "kernel": f"k_sdf_grid<{'POLYGON' if fp.is_polygon() else 'RECT'},{fp.count()}> (per-pose exact SDF min, exact culling)",
                     "sdf_kernel_ms": sdf_avg_ms,
                     "work": "EXECUTED FP32 ops: exm_sdf_work_stats counters x per-unit op counts (DESIGN.md §4)",
                     "executed_ops_per_launch": ex_ops,
                     "counters": counts, "ops_per_unit": per_unit,
                     "lane_efficiency_point_loop": (counts["point_tests"] / (32.0 * counts["point_iters_warp"])
                                                    if counts["point_iters_warp"] else None),
                     "algorithmic_ops_unpruned": algorithmic,
                     "culling_factor": algorithmic / ex_ops if ex_ops else None,
                     "ncu": prof.get("executed"),
                     "sdf_path": path,
                     "peak_source": peak_src},
        "clocks": clk.summary(),
        "decision": {"validated": dec.validated, "argmin": dec.argmin,
                     "best_cost": dec.best_cost},
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        base = cpu_reference_sample(wl, seconds=10.0)
        line["cpu_baseline"] = {k: base[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0 and not args.no_sdf_batch:
        line["sdf_batch"] = bench_sdf_batch(args, torch, peak, peak_src)
    if rank == 0 and not args.no_sdf_batch:
        line["hybrid"] = bench_hybrid(args, torch)
        line["hybrid_cfg5"] = bench_hybrid_cfg5(args, torch)
        line["sense"] = bench_sense(args, world == 1 and not args.no_cpu_baseline)
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_sdf_batch(args, torch, peak, peak_src):
    """Config 4: 64-vertex concave star vs 1,000 poses x 10^6 points (10^9 pairs), every pair
    evaluated (k_sdf_pairs, per-pose min), inputs resident; FP32 roofline of that kernel."""
    from paper_2605_29663_b200 import workloads as W
    from paper_2605_29663_b200.api import Engine
    fp, poses, pts = W.cfg4()
    wl = W.cfg1(K=8, T=2)
    eng = Engine(wl.model, wl.limits, fp, wl.params, n_cap=16, guide_cap=4)
    eng.sdf_stage(poses, pts)
    eng.sdf_run_resident(2, False)
    eng.step_stats()
    n = max(3, min(20, args.steps // 10))
    eng.sdf_run_resident(n, False)
    st = eng.step_stats()
    ms = st["sdf_ms"]
    pairs = poses.shape[0] * pts.shape[0]
    F = ops_per_pair(fp)
    achieved = pairs * F / (ms * 1e-3) / 1e12
    eng.sdf_run_resident(1, True)
    st2 = eng.step_stats()
    prof = ncu_profile("sdf_pairs_cfg4")
    return {"workload": "cfg4_star64_P1000_N1e6", "pairs": pairs, "kernel_ms_min_only": ms,
            "kernel_ms_with_pairs": st2["sdf_ms"], "sdf_evals_per_s": pairs / (ms * 1e-3),
            "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "kernel": "k_sdf_pairs<POLYGON,64>",
                         "traffic": prof.get("traffic"), "executed": prof.get("executed"),
                         "algorithmic": f"P*N pairs x {F} ops/pair (every pair evaluated)",
                         "peak_source": peak_src}}


def bench_hybrid(args, torch):
    """the three trap_hybrid mode families (Ackermann, parallel, spin; hybrid-box,
    K=384, T=25) stepped in one device call vs one exm_control_cycle per family (wall clock per
    hybrid step, host API both ways, selection on the host excluded)."""
    from paper_2605_29663_b200 import workloads as W
    from paper_2605_29663_b200.api import Engine, HybridController, ObstacleSet
    fp, modes, params, hp, q0, cloud, g = W.trap_hybrid()
    obst = ObstacleSet(cloud, np.ones(cloud.shape[0], np.uint8))
    hc = HybridController(modes, fp, params, hp, n_cap=cloud.shape[0], guide_cap=8)
    singles = []
    for m, mode in enumerate(modes):
        p = W.MppiParams(**{**params.__dict__})
        p.seed = params.seed ^ ((0x9E3779B97F4A7C15 * (m + 1)) & 0xFFFFFFFFFFFFFFFF)
        e = Engine(mode.model, mode.limits, fp, p, n_cap=cloud.shape[0], guide_cap=8)
        singles.append((e, np.zeros(params.horizon * mode.model.control_dim()), np.zeros(3)))
    n = max(20, args.steps // 2)
    for _ in range(5):
        hc.family_cycles(q0, obst, g)
    t0 = time.perf_counter()
    for _ in range(n):
        hc.family_cycles(q0, obst, g)
    batched = (time.perf_counter() - t0) / n
    for c in range(5):
        for e, nom, up in singles:
            e.control_cycle_raw(q0, obst, g, nom, up, c)
    t0 = time.perf_counter()
    for c in range(n):
        for e, nom, up in singles:
            e.control_cycle_raw(q0, obst, g, nom, up, c)
    seq = (time.perf_counter() - t0) / n
    return {"workload": "trap_hybrid 3 families (ackermann/parallel/spin), K=384, T=25, N=400",
            "batched_ms_per_step": 1e3 * batched, "per_family_calls_ms_per_step": 1e3 * seq,
            "speedup": seq / batched}


def bench_hybrid_cfg5(args, torch):
    """Config 5's hybrid variant: three mode families (Ackermann,
    parallel, spin) x K=65,536 rollouts x T=80 on config 5's 50k-point cloud. One hybrid step =
    all three families' MPPI steps: batched into one device call (exm_hybrid_cycle: one cloud
    preparation, one SDF launch over 3 x 5.24M poses) vs one exm_control_cycle per family;
    wall clock per hybrid step through the host API, selection on the host excluded."""
    from paper_2605_29663_b200 import workloads as W
    from paper_2605_29663_b200.api import Engine, HybridController, ObstacleSet
    fp, modes, params, hp, q0, cloud, g = W.cfg5_hybrid()
    obst = ObstacleSet(cloud, np.ones(cloud.shape[0], np.uint8))
    hc = HybridController(modes, fp, params, hp, n_cap=cloud.shape[0], guide_cap=8)
    singles = []
    for m, mode in enumerate(modes):
        p = W.MppiParams(**{**params.__dict__})
        p.seed = params.seed ^ ((0x9E3779B97F4A7C15 * (m + 1)) & 0xFFFFFFFFFFFFFFFF)
        e = Engine(mode.model, mode.limits, fp, p, n_cap=cloud.shape[0], guide_cap=8)
        singles.append((e, np.zeros(params.horizon * mode.model.control_dim()), np.zeros(3)))
    n = 10
    for _ in range(3):
        hc.family_cycles(q0, obst, g)
    t0 = time.perf_counter()
    for _ in range(n):
        hc.family_cycles(q0, obst, g)
    batched = (time.perf_counter() - t0) / n
    for c in range(3):
        for e, nom, up in singles:
            e.control_cycle_raw(q0, obst, g, nom, up, c)
    t0 = time.perf_counter()
    for c in range(n):
        for e, nom, up in singles:
            e.control_cycle_raw(q0, obst, g, nom, up, 3 + c)
    seq = (time.perf_counter() - t0) / n
    hc.close()
    for e, _, _ in singles:
        e.close()
    return {"workload": "cfg5 hybrid: 3 families (ackermann/parallel/spin) x K=65536, T=80, N=50k",
            "batched_ms_per_step": 1e3 * batched, "per_family_calls_ms_per_step": 1e3 * seq,
            "speedup": seq / batched, "hybrid_steps_per_s": 1.0 / batched}


def cfg5_world():
    """The config-5 world as the reference scenario holds it: the two omni_gap walls (static) and
    64 discs on 2-waypoint ping-pong trails (world.hpp TrailMotion)."""
    from paper_2605_29663_b200 import workloads as W
    from paper_2605_29663_b200.api import Trail, WorldObstacle
    obs = [WorldObstacle.polygon(p) for p in W.OMNI_WALLS]
    trails = [None] * len(obs)
    for k in range(64):
        ax, ay = W.uniform_range(9, k, 0, -8.0, 8.0), W.uniform_range(9, k, 1, -8.0, 8.0)
        bx, by = W.uniform_range(9, k, 2, -8.0, 8.0), W.uniform_range(9, k, 3, -8.0, 8.0)
        obs.append(WorldObstacle.disc((ax, ay), W.uniform_range(9, k, 4, 0.2, 0.5)))
        trails.append(Trail([[ax, ay], [bx, by]], W.uniform_range(9, k, 5, 0.0, 0.2)))
    return obs, trails


def bench_sense(args, with_cpu):
    """one world cycle of the config-5 scene — step_world (world.cpp:127-157, the
    64 discs' trails) then sense() (:182-243) from q0, range 10 m, budget 720 — with the world kept
    on the device (exm_world_step + exm_world_sense: host ObstacleSet out) vs the reference's own
    step_world + sense from oracle/_ref on one host core (the reference is single-threaded here).
    Also the one-shot exm_sense (obstacle geometry and offsets from the host each call)."""
    from paper_2605_29663_b200 import workloads as W
    from paper_2605_29663_b200.api import Engine, WorldObstacle
    obs, trails = cfg5_world()
    wl = W.cfg1(K=32, T=4)
    eng = Engine(wl.model, wl.limits, wl.footprint, wl.params, n_cap=16, guide_cap=4)
    robot = np.array([-4.0, 0.0, 0.0])
    world = eng.world(obs, trails, 10.0, 720, 7)
    for c in range(3):
        world.step(0.1)
        cloud = world.sense(robot, c)
    n = max(20, args.steps // 4)
    t0 = time.perf_counter()
    for c in range(n):
        world.step(0.1)
        cloud = world.sense(robot, c)
    gpu = (time.perf_counter() - t0) / n
    arc, _, off = world.state()
    moved = [WorldObstacle(o.vertices, o.center, o.radius, tuple(off[i])) for i, o in enumerate(obs)]
    for _ in range(3):
        eng.sense(moved, robot, 10.0, 720, 7, 0)
    t0 = time.perf_counter()
    for c in range(n):
        eng.sense(moved, robot, 10.0, 720, 7, c)
    one_shot = (time.perf_counter() - t0) / n
    world.close()
    out = {"workload": "cfg5 world: 2 walls + 64 discs on trails, step 0.1 s + sense, range 10 m, budget 720",
           "visible_points": int(cloud.mask.sum()), "exm_world_step_sense_ms": 1e3 * gpu,
           "exm_sense_one_shot_ms": 1e3 * one_shot}
    if with_cpu:
        from tests.oracle_bindings import ReferenceWorld, reference_available
        if reference_available():
            ref = ReferenceWorld(obs, trails, 10.0, 720, 7)
            for c in range(3):
                ref.step(0.1)
                ref.sense(robot, c)
            t0 = time.perf_counter()
            for c in range(n):
                ref.step(0.1)
                ref.sense(robot, c)
            cpu = (time.perf_counter() - t0) / n
            out.update({"reference_step_sense_ms": 1e3 * cpu, "cores": 1, "speedup": cpu / gpu})
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-sdf-batch", action="store_true")
    ap.add_argument("--config", default="cfg2", choices=["cfg1", "cfg2", "cfg3", "cfg5"],
                    help="workload (the headline is cfg2; the others are reported separately)")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    world, rank, local = dist_setup()
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        run_ours(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist
        if args.impl != "reference":  # the reference arm runs on rank 0 alone: no rendezvous
            dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
