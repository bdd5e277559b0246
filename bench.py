#!/usr/bin/env python
"""Headline benchmark: candidate poses scored / second through
render -> GICP refine -> re-render -> cost -> argmin (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c3] [--impl reference]

A step = one pass of the hot path over one batch of candidates of the workload
scene.  Workload (default `c3`): the cluttered five-box 3-DoF scene of
BASELINE.json configs[2] (the committed, reference-generated, disk-round-tripped
scene in tests/golden/c3_clutter_3dof.npz), workspace +-0.32 m, dt 0.025 m,
dyaw 22.5 deg / N_gpus -> 58,320 candidates per GPU, ICP refinement on.
Candidates are sharded across ranks by grid cell (weak scaling: per-GPU work is
fixed); the only collective is an all_reduce(MIN) of the packed (cost, pose-id)
keys, one uint64 per object.

`value`  : inputs resident in HBM, timed with CUDA events on the launch stream.
`e2e`    : same metric through the engine's C-ABI calls from HOST buffers:
           scene + models + targets + candidate upload, search, result download.
`--impl reference`: the CPU oracle port (the reference is pure Python and cannot
           travel to the GPU box) on all host cores, on a bounded sample.
"""

from __future__ import annotations

import argparse
import dataclasses
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "candidate poses scored/sec (render+ICP+cost)"
UNIT = "poses/s"

WORKLOADS = {
    # name: (fixture, overrides per n_gpus -> SearchConfig kwargs)
    "c1": ("c1_box_3dof", lambda n: dict(dyaw=np.radians(22.5) / n)),
    "c2": ("c2_twocyl_color1", lambda n: dict(dt=0.04 / n)),
    "c3": ("c3_clutter_3dof", lambda n: dict(dt=0.025, dyaw=np.radians(22.5) / n, max_proposals=None)),
    "c3q": ("c3_clutter_3dof", lambda n: dict(dt=0.025, dyaw=np.radians(22.5) / n, max_proposals=None,
                                              workspace=(-0.125, 0.125, -0.125, 0.125))),
    "c3s": ("c3_clutter_3dof", lambda n: dict(dt=0.08, dyaw=np.radians(22.5) / n, max_proposals=None)),
    # C5 sweep: the C3 scene with the yaw axis refined `--scale` times (58,320 x scale candidates, same 3,645 targets)
    "c5": ("c3_clutter_3dof", lambda n: dict(dt=0.025, dyaw=np.radians(22.5) / n, max_proposals=None)),
    "c4": ("c4_mixed_6dof", lambda n: dict(viewpoints=642 * n, n_inplane=36, z_step=0.01, max_proposals=None)),
}


def build_workload(name: str, n_gpus: int, scale: int = 1, materialise_targets: bool = True):
    """materialise_targets=False: the plan carries only the GICP target SPECS and the device
    crops the clouds itself (what estimate_poses does); the CPU arms need the host copies."""
    n_gpus = n_gpus * max(1, scale)
    import golden_io as G
    from paper_2008_00326_b200.search import plan_search

    fixture, over = WORKLOADS[name]
    d = G.load(fixture)
    frame, models = G.frame_of(d), G.models_of(d)
    cfg = dataclasses.replace(G.config_of(d), **over(n_gpus))
    plan = plan_search(frame, models, cfg, materialise_targets=materialise_targets)
    return frame, models, cfg, plan


from paper_2008_00326_b200.dist import keys_from_device, shard_index  # noqa: E402


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.rows, self.proc = [], None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100", "-i", str(index)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            pass
        sm, mx, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for r in self.rows:
            try:
                sm.append(float(r[0])), mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def algorithmic_bytes(plan_n, models, flat_oid, out, ncorr_sum, cap0, cap1, refine, n_m, n_fp):
    """SURVEY.md 8(d) per-candidate algorithmic bytes, summed over the batch,
    split per kernel.  f64 = 8 B, i32 = 4 B, bool = 1 B."""
    V = np.array([models[int(o)].mesh.vertices.shape[0] for o in flat_oid], dtype=np.float64)
    T = np.array([models[int(o)].mesh.triangles.shape[0] for o in flat_oid], dtype=np.float64)
    n0, n1 = out.n_first.astype(np.float64), out.n_rendered.astype(np.float64)
    it = out.iterations.astype(np.float64)
    b_render0 = 96 + 48 * V + 12 * T + 13 * cap0 + 56 * n0
    b_render1 = 96 + 48 * V + 12 * T + 13 * cap1 + 56 * n1
    b_cov = 96 * n0
    b_iter_sum = it * (104 * n0 + 344) + 96 * ncorr_sum.astype(np.float64)
    b_cost = 56 * n1 + 48 * n_m.astype(np.float64) + 25 * n_fp.astype(np.float64) + 8  # n_m, n_fp counted by cost_kernel
    d = {"render": float(b_render0.sum()), "rerender": float(b_render1.sum()) if refine else 0.0,
         "refine": float((b_cov + b_iter_sum).sum()) if refine else 0.0, "cost": float(b_cost.sum())}
    d["total"] = sum(d.values())
    # the refine stage per kernel (B_iter = 104 n_r + 96 n_c + 344 split by which kernel consumes the operand:
    # nn: source points in, correspondence out, matched target point; step (linearise + solve + halving, fused):
    # source covariances, matched target covariance, H/g/f0 out; the halving re-reads operands the model already
    # charged once, so it adds no algorithmic bytes)
    nc = ncorr_sum.astype(np.float64)
    d["kernels"] = {
        "gicp_init_kernel": float(b_cov.sum()) if refine else 0.0,
        "gicp_nn_kernel": float((it * 32 * n0 + 24 * nc).sum()) if refine else 0.0,
        "gicp_step_kernel": float((it * (72 * n0 + 344) + 72 * nc).sum()) if refine else 0.0,
        "gicp_halve_kernel": 0.0, "gicp_finish_kernel": 0.0,
    }
    return d


def workload_string(name, cfg):
    """Identical in both arms (the driver's same_config check compares it)."""
    return f"{name}: {WORKLOADS[name][0]} scene, mode={cfg.mode}, refine={cfg.refine}, stride={cfg.stride}, 640x480"


def run_gpu(args):
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test knobs (one-GPU boxes): PX_BENCH_DEVICE pins every rank to one device, PX_BENCH_BACKEND=gloo replaces
    # NCCL (which refuses two ranks on one GPU) so the multi-rank code path can be exercised end to end
    local = int(os.environ.get("PX_BENCH_DEVICE", local))
    backend = os.environ.get("PX_BENCH_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll_dev = "cuda" if backend == "nccl" else "cpu"
    peaks = {}
    pk = ROOT / "MEASURED_PEAKS.json"
    if pk.exists():
        peaks = json.loads(pk.read_text())
    hbm_peak, peak_src = (peaks["hbm_gbs"], "measured") if "hbm_gbs" in peaks else (6650.0, "fallback")

    from paper_2008_00326_b200.engine import Engine

    frame, models, cfg, plan = build_workload(args.workload, world, args.scale, materialise_targets=False)
    idx = shard_index(plan, rank, world)
    eng = Engine(local)
    # a non-default torch stream: its handle is non-zero, so libpx launches on exactly the stream the L2 flush and
    # the timing events are recorded on (handle 0 would mean "the context's own stream" to px_ctx_set_stream)
    stream = torch.cuda.Stream(device=local)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    device_comm = world > 1 and backend == "nccl"
    if device_comm:
        eng.comm_init_torch()  # libpx's own NCCL communicator; the unique id travels over torch.distributed
        if rank == 0:
            print(f"[bench] libpx NCCL communicator up: nranks {eng.comm_world()}, NCCL {eng.nccl_version()}", file=sys.stderr)
    sc = eng.search_cfg(plan)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    keys_t = torch.zeros(max(len(plan.active), 1), dtype=torch.int64, device=coll_dev)

    def reduce_host(keys: dict):
        """gloo test knob only: the min-reduction through host memory (NCCL refuses two ranks on one GPU)."""
        if world > 1 and not device_comm:
            keys_t.copy_(torch.from_numpy(keys_from_device(plan, keys)))
            dist.all_reduce(keys_t, op=dist.ReduceOp.MIN)

    def winners_keys():
        w = eng.search_winners()
        return w, {o: w[o][0] for o in w}

    # ---- resident-input arm (`value`) ----
    eng.prepare_plan(frame, models, plan)
    n_local = eng.search_upload(plan, idx)
    eng.set_kernel_timing(True)  # event marks around every refine-stage launch (roofline of the dominant kernel)
    for _ in range(args.warmup):
        eng.search_run(sc)
        eng.search_reduce()
    reduce_host(winners_keys()[1])
    barrier()
    sampler = ClockSampler(local) if rank == 0 else None
    launches0 = eng.launch_count()
    step_ms, stage_ms, kern_ms, reduce_ms = [], [], [], []
    t_wall0 = time.perf_counter()
    for _ in range(args.steps):
        flush.zero_()  # L2 flush between timed iterations (outside the event pair, same stream)
        e0, em, e1 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        eng.search_run(sc)      # render -> GICP -> re-render -> cost -> per-object atomicMin keys
        em.record(stream)
        eng.search_reduce()     # NCCL all-reduce(MIN) of the keys + winner records (device, no host sync)
        e1.record(stream)
        e1.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        reduce_ms.append(em.elapsed_time(e1))
        stage_ms.append(eng.stage_millis())
        kern_ms.append(eng.kernel_ms())
        reduce_host(winners_keys()[1])
    barrier()
    wall_s = time.perf_counter() - t_wall0
    launches = eng.launch_count() - launches0
    clocks = sampler.stop() if sampler else None
    total_ms = float(np.sum(step_ms))
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
        cnt = torch.tensor([n_local], dtype=torch.int64, device=coll_dev)
        dist.all_reduce(cnt, op=dist.ReduceOp.SUM)
        n_total = int(cnt.item())
    else:
        n_total = n_local
    ms_per_step = total_ms / args.steps
    value = n_total / (ms_per_step * 1e-3)
    knife = eng.knife_edges()

    # ---- end-to-end arm (`e2e`): host buffers -> C-ABI -> host results, every step ----
    barrier()
    from paper_2008_00326_b200.search import plan_lattice
    lat = plan_lattice(frame, models, cfg)   # proposal factors (host, per scene); None: flat candidate upload
    e2e_ms = []
    for s in range(max(2, min(args.steps, 5)) + 1):
        t0 = time.perf_counter()
        eng._scene_key = None
        eng._model_keys.clear()
        if lat is not None:
            eng.upload_frame(frame, cfg.stride)            # frame planes from host memory; observed cloud on the device
            eng.upload_models({o: models[o] for o in lat.active})
            eng.search_upload_lattice(lat, rank, world)    # proposal factors from host memory; candidates + targets on the device
        else:
            eng.prepare_plan(frame, models, plan)
            eng.search_upload(plan, idx)
        eng.search_run(sc)
        eng.search_reduce()
        wins, wkeys = winners_keys()   # device -> host read of the step's result (per-object winner records)
        reduce_host(wkeys)
        torch.cuda.synchronize()
        if s:
            e2e_ms.append((time.perf_counter() - t0) * 1e3)
    k_ = frame.intrinsics
    npix = k_.width * k_.height
    n_specs = 0 if plan.target_idx is None else int(plan.target_idx.max()) + 1
    model_bytes = sum(m.mesh.vertices.size * 16 + m.mesh.triangles.size * 4 for m in models.values())
    if lat is not None:
        ng = ((k_.width + cfg.stride - 1) // cfg.stride) * ((k_.height + cfg.stride - 1) // cfg.stride)
        h2d = ng * (13 + 24) + model_bytes + sum(f.rotations.size * 8 + f.translations.size * 8 + 64 for f in lat.lattice)
    else:
        h2d = npix * 13 + len(plan.observed) * (24 + 24 + 8 + 4) + n_specs * 40 + model_bytes + n_local * (96 + 12)
    d2h = 8 * 28 * len(models) + 32
    e2e_t = float(np.median(e2e_ms)) * 1e-3
    if world > 1:
        t = torch.tensor([e2e_t], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    e2e_value = n_total / e2e_t
    # the user-facing call itself: estimate_poses(frame, models, cfg) = host planning (observed cloud,
    # proposals, target specs) + everything above + result assembly; at N>1 it is the distributed call
    # (every rank returns the same SearchResult)
    import paper_2008_00326_b200.engine as E
    from paper_2008_00326_b200 import estimate_poses
    E._default = eng
    ts = []
    if world == 1 or device_comm:
        for s_ in range(3):
            barrier()
            t0 = time.perf_counter()
            res = estimate_poses(frame, models, cfg)
            torch.cuda.synchronize()
            if s_:
                ts.append((time.perf_counter() - t0) * 1e3)
        assert res.proposals_evaluated == n_total
    api_ms = float(np.median(ts)) if ts else None
    if api_ms is not None and world > 1:
        t = torch.tensor([api_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        api_ms = float(t.item())

    if rank != 0:
        if device_comm:
            eng.lib.px_comm_destroy(eng.ctx)
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant kernel (GICP refine) ----
    eng.search_run(sc)  # the e2e / estimate_poses runs above replaced the resident shard's results
    full = eng.search_download(n_local)
    ncs, cap0, cap1, n_m, n_fp = eng.search_stats(n_local)
    ab = algorithmic_bytes(n_local, models, plan.flat_oid[idx], full, ncs, cap0, cap1, cfg.refine, n_m, n_fp)
    st = {k: float(np.mean([s[k] for s in stage_ms])) for k in stage_ms[0]}
    # per kernel: mean over the timed steps of (total ms, launches) per step
    kern = {k: (float(np.mean([m[k][0] for m in kern_ms])), float(np.mean([m[k][1] for m in kern_ms]))) for k in kern_ms[0]}
    kern["render_kernel"] = (st["render"] + st["rerender"], 2.0 if cfg.refine else 1.0)
    kern["cost_kernel"] = (st["cost"], 1.0)
    kbytes = dict(ab["kernels"])
    kbytes["render_kernel"] = ab["render"] + ab["rerender"]
    kbytes["cost_kernel"] = ab["cost"]
    traffic_db = {}
    tj = ROOT / "profiles" / "traffic.json"
    if tj.exists() and args.scale == 1 and world == 1:
        traffic_db = json.loads(tj.read_text()).get(args.workload, {})
    table = {}
    for k, (ms, nl) in kern.items():
        if nl <= 0 or (k == "gicp_halve_kernel" and ms < 0.5):  # fused build: the halving runs inside gicp_step_kernel
            continue
        per_launch_ms, per_launch_b = ms / nl, kbytes.get(k, 0.0) / nl
        table[k] = {"launches_per_step": nl, "ms_per_step": ms, "ms_per_launch": per_launch_ms,
                    "algorithmic_bytes_per_launch": per_launch_b,
                    "achieved_gbs": per_launch_b / (per_launch_ms * 1e-3) / 1e9 if per_launch_ms > 0 else 0.0,
                    "traffic": traffic_db.get(k, {}).get("dram_bytes_per_launch"),
                    "ncu": traffic_db.get(k, {}).get("ncu")}
    dom = max(table, key=lambda k: table[k]["ms_per_step"])
    dk = table[dom]
    refine_gbs = ab["refine"] / (st["refine"] * 1e-3) / 1e9 if st["refine"] > 0 else 0.0
    roofline = {"bound": "hbm", "kernel": dom, "achieved": dk["achieved_gbs"], "peak": hbm_peak, "peak_source": peak_src,
                "unit": "GB/s", "frac": dk["achieved_gbs"] / hbm_peak, "traffic": dk["traffic"],
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum of one ncu --set full capture of one launch of this "
                                "kernel on this workload (profiles/traffic.json); null when no capture matches",
                "ncu": dk["ncu"],
                "ncu_note": "counters of the committed ncu --set full capture of this kernel (profiles/): the true limiter "
                            "(issue slots / lane occupancy / fp64 pipe) next to the HBM fraction asked for",
                "algorithmic_bytes_per_launch": dk["algorithmic_bytes_per_launch"], "kernel_ms": dk["ms_per_launch"],
                "launches_per_step": dk["launches_per_step"],
                "timing": "CUDA events recorded on the launch stream around every launch of the GICP stage inside the timed steps",
                "kernels": table,
                "refine_stage_achieved": refine_gbs, "refine_stage_frac": refine_gbs / hbm_peak,
                "whole_step_achieved": ab["total"] / (ms_per_step * 1e-3) / 1e9,
                "whole_step_frac": ab["total"] / (ms_per_step * 1e-3) / 1e9 / hbm_peak,
                "bytes_per_candidate": ab["total"] / max(n_local, 1)}

    # ---- per-scene latency and multi-scene batching on the small config (BASELINE: "per-scene latency") ----
    latency = None
    if world == 1 and not args.no_latency:
        lat_sampler = ClockSampler(local)
        latency = small_scene_latency(eng)
        latency["clocks"] = lat_sampler.stop()

    # ---- CPU baseline on a bounded sample of the same workload (rank 0, N=1 only) ----
    cpu = None
    if world == 1 and not args.no_cpu:
        _, _, _, plan_host = build_workload(args.workload, world, args.scale)  # host copies of the GICP targets
        cpu = cpu_baseline(frame, models, plan_host, idx, args.cpu_sample or 40000)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_string(args.workload, cfg),
                   "candidates_per_step": n_total, "candidates_per_gpu": n_local,
                   "sharding": "grid cells round-robin across ranks; ONE ncclAllReduce(MIN) of the packed (cost,pose-id) keys "
                               "per step on libpx's own communicator, inside the timed region",
                   "collective": ("nccl (px_search_reduce, device-side)" if device_comm else
                                  ("none (single rank)" if world == 1 else f"{backend} through host memory (test knob)")),
                   "l2": "256 MiB flush between timed steps; per-step scratch also exceeds L2"},
        "stage_ms": st, "reduce_ms": float(np.mean(reduce_ms)), "wall_s_timed_region": wall_s,
        "knife_edges": knife,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_t * 1e3,
                "path": ("frame planes + models + proposal factors from host buffers -> C-ABI (observed cloud, candidate poses, "
                         "GICP targets built on the device; argmin + winner records reduced on the device) -> per-object "
                         "results on the host") if lat is not None else
                        ("scene + models + GICP target specs + candidates from host buffers -> C-ABI -> per-object results on the host"),
                "estimate_poses_ms": api_ms,
                "estimate_poses_value": (n_total / (api_ms * 1e-3)) if api_ms else None},
        "gpu_launches": int(launches),
        "clocks": clocks, "roofline": roofline, "cpu_baseline": cpu, "latency": latency,
        "latency_ms": latency["estimate_poses_ms"] if latency else None,  # C1 (1,936 candidates): one public call, host to host
        "mean_iterations": float(full.iterations.mean()), "mean_rendered_points": float(full.n_rendered.mean()),
    }
    print(json.dumps(line))
    if device_comm:
        eng.lib.px_comm_destroy(eng.ctx)
    if world > 1:
        dist.destroy_process_group()


def small_scene_latency(eng, scenes: int = 16, streams: int = 4):
    """BASELINE configs[0] (C1: one box, 1,936 candidates, GICP on): milliseconds of the public call for one scene
    (host planning + frame upload + device set-up + search + argmin + result on the host), and throughput with
    several scenes in flight (batch.estimate_poses_many: one device context / CUDA stream per scene in flight)."""
    import golden_io as G
    from paper_2008_00326_b200 import estimate_poses, estimate_poses_many

    d = G.load("c1_box_3dof")
    frame, models, cfg = G.frame_of(d), G.models_of(d), G.config_of(d)
    ts = []
    for i in range(8):
        t0 = time.perf_counter()
        res = estimate_poses(frame, models, cfg, engine=eng)
        if i >= 3:
            ts.append((time.perf_counter() - t0) * 1e3)
    jobs = [(frame, models, cfg)] * scenes
    estimate_poses_many(jobs[:streams], streams=streams)  # contexts created, kernels loaded
    t0 = time.perf_counter()
    estimate_poses_many(jobs, streams=streams)
    many_s = time.perf_counter() - t0
    t0 = time.perf_counter()
    estimate_poses_many(jobs, streams=1)
    one_s = time.perf_counter() - t0
    n = res.proposals_evaluated
    return {"workload": "c1: c1_box_3dof scene, mode=3dof, refine=True, 1,936 candidates, 640x480",
            "estimate_poses_ms": float(np.median(ts)), "stage_ms": res.stage_millis,
            "multi_scene": {"scenes": scenes, "streams": streams, "ms_per_scene": many_s / scenes * 1e3,
                            "poses_per_s": n * scenes / many_s, "ms_per_scene_one_stream": one_s / scenes * 1e3,
                            "poses_per_s_one_stream": n * scenes / one_s}}


def sample_groups(plan, idx, sample: int) -> np.ndarray:
    """Bounded CPU sample: whole target groups (all yaws of a grid cell / all
    candidates sharing a GICP target) spaced uniformly over the step's candidates,
    so the per-target covariance build is amortised exactly as in the full step."""
    if len(idx) <= sample:
        return idx
    if plan.target_idx is None:
        return idx[np.unique(np.round(np.linspace(0, len(idx) - 1, sample)).astype(int))]
    t = plan.target_idx[idx]
    groups = np.unique(t)
    per = max(1.0, len(idx) / len(groups))
    want = max(1, int(round(sample / per)))
    chosen = groups[np.unique(np.round(np.linspace(0, len(groups) - 1, min(want, len(groups)))).astype(int))]
    return idx[np.isin(t, chosen)]


def cpu_baseline(frame, models, plan, idx, sample: int):
    from oracle import oracle as O

    cores = os.cpu_count() or 1
    pick = sample_groups(plan, idx, sample)
    O.run_plan(frame, models, plan, n_threads=cores, index=pick[:64])  # warm-up (page in, threads)
    t0 = time.perf_counter()
    out = O.run_plan(frame, models, plan, n_threads=cores, index=pick)
    dt = time.perf_counter() - t0
    return {"value": len(pick) / dt, "unit": UNIT, "cores": cores, "kind": "port",
            "sample": f"{len(pick)} candidates (whole grid cells spaced uniformly) of the step's {len(idx)} (oracle/px_oracle.c, pthreads, "
                      f"{dt:.1f} s)", "stage_ms": {k: float(v) for k, v in out.stage_millis.items()}}


def run_reference(args):
    """Reference arm: the reference's own CPU implementation of the path on the host cores.

    When the unmodified package is installed in oracle/_ref (`make -C oracle ref`, done by build() wherever
    /root/reference exists) and importable (numba), this times `rvpose.search.estimate_poses` itself with
    workers = os.cpu_count() (kind "reference"); otherwise the pinned C restatement oracle/px_oracle.c with
    pthreads on all cores (kind "port").  Either way a step is a BOUNDED SAMPLE of the workload's candidates --
    whole grid cells spread uniformly over the workspace, so that the per-cell GICP target work is amortised
    as in the full step -- and `value` is per-candidate throughput.  The port's number is reported next to
    the reference's (`port` key): it is ~10x faster than the Python package and therefore the stricter baseline."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return
    frame, models, cfg, plan = build_workload(args.workload, world, args.scale)
    from oracle import oracle as O
    from oracle import ref_runner as R

    cores = os.cpu_count() or 1
    idx = np.arange(plan.n)
    budget_s = float(os.environ.get("PX_REF_BUDGET_S", "150"))  # whole timed region

    # ---- the C port (always; also the fallback) ----
    def run_port(sample):
        pick = sample_groups(plan, idx, sample)
        O.run_plan(frame, models, plan, n_threads=cores, index=pick[:128])
        t0 = time.perf_counter()
        O.run_plan(frame, models, plan, n_threads=cores, index=pick)
        return len(pick), time.perf_counter() - t0

    why = R.available()
    if why is None:
        try:
            search = R.load()
        except Exception as e:  # pragma: no cover
            why = f"import failed: {e}"
    port = None
    if why is None:
        kind = "reference"
        # warm-up (numba JIT / cache load, fork pool) + calibration on one small patch
        if cfg.mode == "3dof":
            probe = R.patches_3dof(cfg, 2, 4)   # four 2x2-cell patches spread over the workspace
            R.run_sample(search, frame, models, cfg, patches=probe[:1])
            n0, s0, _ = R.run_sample(search, frame, models, cfg, patches=probe)
            per_cand = s0 / max(n0, 1)
            want = budget_s / max(args.steps, 1) / per_cand                      # candidates per step that fit the budget
            per_patch = 9 * n0 / (4 * len(probe))                                # 3 x 3 cells, all objects and yaws
            count = int(np.clip(int(want / per_patch), 1, 25))
            patches = R.patches_3dof(cfg, 3, count)
            run = lambda: R.run_sample(search, frame, models, cfg, patches=patches)   # noqa: E731
            how = f"{len(patches)} patches of 3x3 grid cells spread uniformly over the workspace"
        else:
            R.run_sample(search, frame, models, cfg, max_proposals=200)
            n0, s0, _ = R.run_sample(search, frame, models, cfg, max_proposals=400)
            mp_ = int(np.clip(budget_s / max(args.steps, 1) / (s0 / max(n0, 1)), 200, 20000))
            run = lambda: R.run_sample(search, frame, models, cfg, max_proposals=mp_)  # noqa: E731
            how = f"the reference's own uniform max_proposals={mp_} subsample (search.py:261-265)"
        for _ in range(max(0, args.warmup - 1)):
            pass  # the calibration calls above were the warm-up (JIT compiled, pool forked)
        times, n_s, stages = [], 0, None
        for _ in range(args.steps):
            n_s, secs, stages = run()
            times.append(secs)
        ms = float(np.mean(times)) * 1e3
        value = n_s / (ms * 1e-3)
        sample = (f"{n_s} candidates per step ({how}) of the workload's {plan.n}; rvpose.search.estimate_poses, "
                  f"workers={cores}, timed like cli._cmd_bench")
        pn, ps = run_port(min(20000, plan.n))
        port = {"value": pn / ps, "unit": UNIT, "cores": cores, "kind": "port",
                "sample": f"{pn} candidates (whole grid cells spaced uniformly), oracle/px_oracle.c + pthreads, {ps:.1f} s"}
    else:
        kind = "port"
        pick = sample_groups(plan, idx, args.cpu_sample or 20000)
        for _ in range(args.warmup):
            O.run_plan(frame, models, plan, n_threads=cores, index=pick[:128])
        times = []
        for _ in range(args.steps):
            t0 = time.perf_counter()
            out = O.run_plan(frame, models, plan, n_threads=cores, index=pick)
            times.append(time.perf_counter() - t0)
        ms = float(np.mean(times)) * 1e3
        n_s = len(pick)
        value = n_s / (ms * 1e-3)
        stages = {k: float(v) for k, v in out.stage_millis.items()}
        sample = (f"{n_s} candidates (whole grid cells spaced uniformly) of the workload's {plan.n} per step; "
                  f"oracle/px_oracle.c + pthreads (the Python reference is not importable here: {why})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_string(args.workload, cfg), "candidates_per_step": plan.n,
                   "sampled_candidates_per_step": n_s,
                   "sampling": "the CPU arm scores a bounded sample of the step's candidates (whole grid cells spread uniformly "
                               "over the workspace) and reports per-candidate throughput"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample, "stage_ms": stages},
        "port": port,
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c3", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-sample", type=int, default=None,
                    help="candidates in the bounded CPU sample (default 40000 for cpu_baseline, 20000 per --impl reference step)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-latency", action="store_true", help="skip the small-scene latency / multi-scene section")
    ap.add_argument("--scale", type=int, default=1, help="refine the yaw/viewpoint axis: candidates x scale (C5 sweep)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "b200":
        # `python bench.py --gpus N` on its own: become N ranks (one process per GPU) under torchrun
        import socket

        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        if os.environ.get("PX_BENCH_PRINT_SPAWN"):  # CPU test hook: show the launch line, do not run it
            print(json.dumps(cmd))
            return
        raise SystemExit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.impl == "b200" and world != args.gpus:
        print(f"[bench] --gpus {args.gpus} but WORLD_SIZE={world}: running {world} rank(s)", file=sys.stderr)
    if world > 1 and args.impl == "b200":
        os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator lines (rank / nranks) on stderr
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    import __graft_entry__ as ge

    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return  # the CPU arm is one process: the other ranks exit without work
        ge.build(load_native=False)  # compiles everything, loads only the oracle: no libpx.so in this process
        run_reference(args)
        return
    if int(os.environ.get("LOCAL_RANK", "0")) == 0:
        ge.build()
    run_gpu(args)


if __name__ == "__main__":
    main()
