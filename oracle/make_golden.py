"""Generate tests/golden/*.npz by running the REFERENCE itself.

Run in the build container only (needs /root/reference; the GPU box never runs
this):

    NUMBA_CACHE_DIR=/tmp/nb python oracle/make_golden.py

Every array written here is an output of the unmodified reference package
`rvpose` imported from /root/reference/pkg/src (or an input handed to it).  The
fixtures pin oracle/px_oracle.c (tests/test_oracle_golden.py) and, through it and
directly, the CUDA path (tests/test_gpu_*.py).  Scenes go through the
reference's own save_scene -> load_scene round trip.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nb")

import rvpose  # noqa: E402
import rvpose.scenegen as sg  # noqa: E402
import rvpose.search as rs  # noqa: E402
from rvpose import raster as rr, registration as rg, cost as rc, neighbors as rn  # noqa: E402
from rvpose import colorspace as rcol, reference as rref, selftest_data  # noqa: E402
from rvpose.geometry import CameraIntrinsics, Pose3Dof, RigidTransform, lift_pose3dof  # noqa: E402
from rvpose.registration import project_to_3dof  # noqa: E402

OUT = Path(__file__).resolve().parent.parent / "tests" / "golden"
WORKERS = int(os.environ.get("GOLDEN_WORKERS", "8"))


def sha(a: np.ndarray) -> bytes:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


def cloud_digest(c) -> np.ndarray:
    """sha256 over points bytes + source_pixel bytes (bit-exact part of a cloud)."""
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(c.points).tobytes())
    h.update(np.ascontiguousarray(c.source_pixel).tobytes())
    return np.frombuffer(h.digest(), dtype=np.uint8)


def pack_models(models: dict) -> dict:
    d = {"model_ids": np.array(sorted(models), dtype=np.int32)}
    for oid in sorted(models):
        m = models[oid]
        d[f"m{oid}_verts"] = m.mesh.vertices
        d[f"m{oid}_colors"] = m.mesh.vertex_colors
        d[f"m{oid}_tris"] = m.mesh.triangles
        d[f"m{oid}_cyl"] = np.array([m.inscribed_cylinder.radius, m.inscribed_cylinder.z_min,
                                     m.inscribed_cylinder.z_max])
        d[f"m{oid}_sym"] = np.array(int(m.yaw_symmetric))
    return d


def pack_frame(frame) -> dict:
    k = frame.intrinsics
    col8 = np.clip(np.rint(frame.color * 255.0), 0, 255).astype(np.uint8)
    mm = np.clip(np.where(frame.depth.valid, np.rint(frame.depth.values * 1000.0), 0.0), 0, 65535).astype(np.uint16)
    return {
        "col8": col8, "depth_mm": mm, "lab8": frame.labels.astype(np.uint8),
        "intr": np.array([k.fx, k.fy, k.cx, k.cy, k.width, k.height], dtype=np.float64),
        "cam_rot": np.ascontiguousarray(k.camera_pose.rotation), "cam_rot_c_contig": np.array(int(k.camera_pose.rotation.flags.c_contiguous)),
        "cam_t": k.camera_pose.translation,
        "det_ids": np.array([d.object_id for d in frame.detections], dtype=np.int32),
        "det_bbox": np.array([d.full_bbox for d in frame.detections], dtype=np.float64).reshape(-1, 4),
        "gt_ids": np.array([s.object_id for s in (frame.ground_truth or [])], dtype=np.int32),
        "gt_pose": np.array([s.pose.matrix3x4() for s in (frame.ground_truth or [])]).reshape(-1, 3, 4),
    }


def disk_roundtrip(frame):
    d = tempfile.mkdtemp(prefix="golden_scene_")
    sg.save_scene(d, frame)
    return sg.load_scene(d)


def staged_search(frame, models, cfg):
    """The reference's estimate_poses, stage by stage with its own functions
    (search.py:217-336), keeping every per-candidate intermediate."""
    k = frame.intrinsics
    world_to_cam, cam_to_world = k.world_to_camera(), k.camera_pose
    object_ids = [d.object_id for d in frame.detections] if frame.detections else sorted(models)
    observed = rr.frame_to_cloud(frame, cfg.stride)
    obs_labels = rr.cloud_labels(observed, frame.labels)
    obs_world = cam_to_world.apply(observed.points) if cfg.mode == "3dof" else None
    psets, cams = {}, {}
    for oid in object_ids:
        ps = rs._build_proposals(oid, frame, models[oid], cfg)
        psets[oid] = ps
        cams[oid] = ([world_to_cam.compose(ps.pose(i)) for i in range(len(ps))]
                     if cfg.mode == "3dof" else ps.transforms())
    active = list(object_ids)
    flat = [(oid, i) for oid in active for i in range(len(psets[oid]))]
    if cfg.max_proposals is not None and len(flat) > cfg.max_proposals:
        pick = np.unique(np.round(np.linspace(0, len(flat) - 1, cfg.max_proposals)).astype(int))
        flat = [flat[i] for i in pick]
        active = [oid for oid in active if any(f[0] == oid for f in flat)]
    grouped = {oid: [] for oid in active}
    for oid, i in flat:
        grouped[oid].append(cams[oid][i])
    clouds0 = rr.render_batch(models, [(oid, grouped[oid]) for oid in active], frame, k, cfg.stride,
                              cfg.occluder_marking, cfg.delta, cfg.workers, cfg.chunk_size)
    refined = [cams[oid][i] for oid, i in flat]
    regs = None
    clouds1 = clouds0
    targets = target_idx = None
    if cfg.refine:
        targets, target_idx = rs._build_targets(active, psets, flat, observed, obs_labels, obs_world, models, cfg)
        regs = rg.m2m_gicp(clouds0, targets, [RigidTransform.identity()] * len(flat), cfg.gicp,
                           target_indices=target_idx, workers=cfg.workers, chunksize=cfg.chunk_size)
        for j, reg in enumerate(regs):
            if reg.failure == "too_few_points" and reg.iterations == 0:
                continue
            cam_pose = reg.transform.compose(refined[j])
            if cfg.mode == "3dof":
                world = cam_to_world.compose(cam_pose)
                cam_pose = world_to_cam.compose(lift_pose3dof(project_to_3dof(world, cfg.fixed_z), cfg.fixed_z))
            refined[j] = cam_pose
        regrouped = {oid: [] for oid in active}
        for (oid, _), pose in zip(flat, refined):
            regrouped[oid].append(pose)
        clouds1 = rr.render_batch(models, [(oid, regrouped[oid]) for oid in active], frame, k, cfg.stride,
                                  cfg.occluder_marking, cfg.delta, cfg.workers, cfg.chunk_size)
    return dict(observed=observed, obs_labels=obs_labels, flat=flat, cams=cams, clouds0=clouds0, regs=regs,
                refined=refined, clouds1=clouds1, targets=targets, target_idx=target_idx)


def search_fixture(name, frame, models, cfg, keep_every=97):
    """Scene + config + the reference's per-candidate outputs."""
    print(f"[{name}] staged reference run ...", flush=True)
    st = staged_search(frame, models, cfg)
    flat = st["flat"]
    n = len(flat)
    trace = tempfile.mktemp(suffix=".jsonl")
    import dataclasses
    res = rs.estimate_poses(frame, models, dataclasses.replace(cfg, trace_path=trace))
    rows = [json.loads(line) for line in open(trace)]
    assert len(rows) == n
    d = {}
    d.update(pack_frame(frame))
    d.update(pack_models(models))
    d["cfg_json"] = np.array(json.dumps({**cfg.to_dict(), "max_proposals": cfg.max_proposals}))
    d["flat_oid"] = np.array([f[0] for f in flat], dtype=np.int32)
    d["flat_local"] = np.array([f[1] for f in flat], dtype=np.int32)
    d["cam_poses"] = np.array([st["cams"][oid][i].matrix3x4() for oid, i in flat])
    d["n_obs"] = np.array(len(st["observed"]))
    d["obs_digest"] = cloud_digest(st["observed"])
    d["obs_lab_sample"] = st["observed"].lab_colors[::257].copy()
    d["n0"] = np.array([len(c) for c in st["clouds0"]], dtype=np.int32)
    d["dig0"] = np.stack([cloud_digest(c) for c in st["clouds0"]])
    d["n1"] = np.array([len(c) for c in st["clouds1"]], dtype=np.int32)
    d["dig1"] = np.stack([cloud_digest(c) for c in st["clouds1"]])
    keep = list(range(0, n, keep_every))
    d["keep"] = np.array(keep, dtype=np.int32)
    for j in keep:
        c = st["clouds0"][j]
        d[f"c0_{j}_pts"], d[f"c0_{j}_lab"], d[f"c0_{j}_src"] = c.points, c.lab_colors, c.source_pixel
    if st["regs"] is not None:
        regs = st["regs"]
        d["reg_T"] = np.array([r.transform.matrix3x4() for r in regs])
        d["reg_iters"] = np.array([r.iterations for r in regs], dtype=np.int32)
        fails = [None, "too_few_points", "degenerate_correspondences", "singular_normal_equations", "no_decrease"]
        d["reg_fail"] = np.array([fails.index(r.failure) for r in regs], dtype=np.int32)
        d["reg_conv"] = np.array([int(r.converged) for r in regs], dtype=np.int32)
        d["reg_f_first"] = np.array([r.objective_trace[0][0] if r.objective_trace else np.nan for r in regs])
        d["reg_f_last"] = np.array([r.objective_trace[-1][1] if r.objective_trace else np.nan for r in regs])
        d["target_idx"] = np.array(st["target_idx"], dtype=np.int32)
        d["target_sizes"] = np.array([len(t) for t in st["targets"]], dtype=np.int32)
        d["target_digest"] = np.stack([np.frombuffer(sha(t.points), dtype=np.uint8) for t in st["targets"]])
    d["refined"] = np.array([p.matrix3x4() for p in st["refined"]])
    d["j_o"] = np.array([r["j_o"] for r in rows], dtype=np.int32)
    d["j_r"] = np.array([r["j_r"] for r in rows], dtype=np.int32)
    d["result_json"] = np.array(rs.result_to_json(res))
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"[{name}] n={n} best={[(e.object_id, e.proposal_index, e.cost.j_o, e.cost.j_r) for e in res.estimates if not e.failed]}"
          f" -> {(OUT / (name + '.npz')).stat().st_size / 1024:.0f} KiB", flush=True)


def scene_c1():
    k = sg.make_camera(640, 480)
    models = {1: sg.mixed_object_suite()[1]}
    spec = sg.SceneSpec(((1, lift_pose3dof(Pose3Dof(0.07, -0.05, 0.7), 0.0)),), (0.42, 0.42), k)
    return disk_roundtrip(sg.generate_scene(spec, models)), models


def scene_c2():
    """Two cylinders identical but for colour (tests/test_search.py:29-43 recipe)."""
    k = sg.make_camera(640, 480)
    models = {
        1: sg.build_model(1, sg.PrimitiveSpec("cylinder", (0.033, 0.12), ((0.0, 1.0, (0.82, 0.06, 0.09)),)), (24, 4)),
        2: sg.build_model(2, sg.PrimitiveSpec("cylinder", (0.033, 0.12), ((0.0, 1.0, (0.05, 0.55, 0.12)),)), (24, 4)),
    }
    spec = sg.SceneSpec(((1, lift_pose3dof(Pose3Dof(-0.1, -0.05, 0.0), 0.0)),
                         (2, lift_pose3dof(Pose3Dof(0.1, 0.05, 0.0), 0.0))), (0.42, 0.42), k)
    return disk_roundtrip(sg.generate_scene(spec, models)), models


def scene_c3():
    """Five distinct boxes, random placement with mutual occlusion."""
    k = sg.make_camera(640, 480)
    dims = [(0.046, 0.036, 0.09), (0.06, 0.04, 0.12), (0.05, 0.05, 0.07), (0.08, 0.03, 0.10), (0.04, 0.03, 0.15)]
    cols = [((0.75, 0.65, 0.1), (0.2, 0.2, 0.55)), ((0.8, 0.1, 0.1), (0.9, 0.8, 0.7)), ((0.1, 0.6, 0.2), (0.1, 0.2, 0.1)),
            ((0.1, 0.3, 0.8), (0.8, 0.8, 0.2)), ((0.6, 0.2, 0.7), (0.2, 0.7, 0.7))]
    models = {i + 1: sg.build_model(i + 1, sg.PrimitiveSpec("box", dims[i], ((0.0, 0.5, cols[i][0]), (0.5, 1.0, cols[i][1]))))
              for i in range(5)}
    spec = sg.random_scene_spec(models, seed=11, placement_extent=(0.2, 0.2), intrinsics=k)
    return disk_roundtrip(sg.generate_scene(spec, models)), models


def scene_c3_noisy():
    """C3's scene with the sensor noise model of SURVEY.md 8(d): depth sigma 2 mm, 2 % dropout, colour
    jitter 0.02 (scenegen.apply_noise, default_rng(seed)) -- holes in the organised clouds, jittered colours."""
    k = sg.make_camera(640, 480)
    dims = [(0.046, 0.036, 0.09), (0.06, 0.04, 0.12), (0.05, 0.05, 0.07), (0.08, 0.03, 0.10), (0.04, 0.03, 0.15)]
    cols = [((0.75, 0.65, 0.1), (0.2, 0.2, 0.55)), ((0.8, 0.1, 0.1), (0.9, 0.8, 0.7)), ((0.1, 0.6, 0.2), (0.1, 0.2, 0.1)),
            ((0.1, 0.3, 0.8), (0.8, 0.8, 0.2)), ((0.6, 0.2, 0.7), (0.2, 0.7, 0.7))]
    models = {i + 1: sg.build_model(i + 1, sg.PrimitiveSpec("box", dims[i], ((0.0, 0.5, cols[i][0]), (0.5, 1.0, cols[i][1]))))
              for i in range(5)}
    spec = sg.random_scene_spec(models, seed=11, placement_extent=(0.2, 0.2), intrinsics=k)
    frame = sg.apply_noise(sg.generate_scene(spec, models), sg.NoiseModel(0.002, 0.02, 0.02), seed=7)
    return disk_roundtrip(frame), models


def scene_c4():
    k = sg.make_camera(640, 480)
    models = sg.mixed_object_suite()
    spec = sg.random_scene_spec(models, seed=5, intrinsics=k)
    return disk_roundtrip(sg.generate_scene(spec, models)), models


def unit_fixtures():
    rng = np.random.default_rng(20260)
    d = {}
    # ---- colour: the reference's own golden vectors (selftest_data.py:8-46) ----
    pairs = np.array(selftest_data.CIEDE2000_VECTORS, dtype=np.float64)  # (34, 7)
    d["srgb_lab_vector"] = np.array([*selftest_data.SRGB_LAB_VECTOR[0], *selftest_data.SRGB_LAB_VECTOR[1]])
    d["ciede_pairs"] = pairs
    rgb = rng.uniform(0, 1, (200, 3))
    d["lab_rgb"], d["lab_out"] = rgb, rcol.srgb_to_lab(rgb)
    la, lb = rng.uniform([0, -80, -80], [100, 80, 80], (300, 3)), rng.uniform([0, -80, -80], [100, 80, 80], (300, 3))
    la[:10, 1:] = 0.0  # zero-chroma branches
    lb[5:15, 1:] = 0.0
    d["de_a"], d["de_b"], d["de_out"] = la, lb, rcol.ciede2000(la, lb)
    # ---- raster: _raster_kernel on random triangle soups (64x64, tests/test_raster.py:68-80 style) ----
    k = CameraIntrinsics(500.0, 500.0, 32.0, 32.0, 64, 64, RigidTransform.identity())
    for t in range(6):
        nv, nt = 30, 40
        verts = np.column_stack([rng.uniform(-0.08, 0.08, nv), rng.uniform(-0.08, 0.08, nv), rng.uniform(0.8, 1.4, nv)])
        if t == 4:   # lattice-aligned vertices: pixel centres on edges, exact depth ties
            verts = np.column_stack([(rng.integers(0, 64, nv) + 0.5 - 32.0) / 500.0, (rng.integers(0, 64, nv) + 0.5 - 32.0) / 500.0,
                                     np.ones(nv)])
        if t == 5:   # some vertices behind the near plane
            verts[::7, 2] = -0.5
        tris = rng.integers(0, nv, (nt, 3)).astype(np.int32)
        cols = rng.uniform(0, 1, (nv, 3))
        z = np.full((64, 64), np.inf)
        c = np.zeros((64, 64, 3))
        v = np.zeros((64, 64), dtype=np.bool_)
        rr._raster_kernel(np.ascontiguousarray(verts), tris, np.ascontiguousarray(cols), 500.0, 500.0, 32.0, 32.0, 64, 64, z, c, v)
        d[f"ras{t}_verts"], d[f"ras{t}_tris"], d[f"ras{t}_cols"] = verts, tris, cols
        d[f"ras{t}_z"], d[f"ras{t}_c"], d[f"ras{t}_valid"] = z, c, v
    # ---- kNN (neighbors.py) incl. integer-lattice ties ----
    for t in range(4):
        q = rng.normal(size=(40, 3)) if t < 2 else rng.integers(0, 3, (40, 3)).astype(float)
        tg = rng.normal(size=(70, 3)) if t < 2 else rng.integers(0, 3, (70, 3)).astype(float)
        kk = (1, 5, 1, 20)[t]
        nn = rn.knn_streamed(q, tg, kk)
        nf = rn.knn_full(q, tg, kk)
        assert np.array_equal(nn.indices, nf.indices)
        d[f"knn{t}_q"], d[f"knn{t}_t"], d[f"knn{t}_k"] = q, tg, np.array(kk)
        d[f"knn{t}_idx"], d[f"knn{t}_d2"] = nn.indices, nn.sq_dists
    # ---- cost: tests/test_cost.py:102-125 recipe against reference.ref_costs ----
    from rvpose.model import LabeledCloud
    cost_cases = []
    for trial in range(60):
        nr, no = int(rng.integers(0, 60)), int(rng.integers(0, 80))
        scale = 0.03 if trial % 2 else 0.2
        rp, op = rng.normal(scale=scale, size=(nr, 3)), rng.normal(scale=scale, size=(no, 3))
        rl = np.column_stack([rng.uniform(0, 100, nr), rng.uniform(-60, 60, (nr, 2))])
        ol = np.column_stack([rng.uniform(0, 100, no), rng.uniform(-60, 60, (no, 2))])
        delta, tau, uc = float(rng.uniform(0.005, 0.1)), float(rng.uniform(3, 40)), bool(trial % 3)
        sel = rng.random(no) < 0.6
        ren = LabeledCloud(rp, rl, np.zeros((nr, 2), dtype=np.int32))
        obs = LabeledCloud(op, ol, np.zeros((no, 2), dtype=np.int32))
        j_r, explained = rc.rendered_cost(ren, obs, rc.CostParams(delta, tau, uc))
        j_o = int(np.count_nonzero(sel & ~explained))
        assert (j_o, j_r) == rref.ref_costs(rp, rl, op, ol, sel, delta, tau, uc)
        cost_cases.append((rp, rl, op, ol, sel, np.array([delta, tau, float(uc)]), np.array([j_o, j_r]), explained))
    for i, cse in enumerate(cost_cases):
        for nm, arr in zip(("rp", "rl", "op", "ol", "sel", "par", "out", "expl"), cse):
            d[f"cost{i}_{nm}"] = arr
    d["cost_n"] = np.array(len(cost_cases))
    # ---- covariances + GICP on box-surface clouds (tests/test_registration.py style) ----
    def box_cloud(n, half=0.1):
        pts = rng.uniform(-half, half, (n, 3))
        face = rng.integers(0, 3, n)
        for i in range(n):
            pts[i, face[i]] = half * (np.sign(pts[i, face[i]]) or 1.0)
        return pts
    cfg = rg.GicpConfig()
    for t in range(4):
        tgt = box_cloud(400)
        ang, shift = math.radians((3, 10, 6, 1)[t]), (0.01, 0.05, 0.03, 0.002)[t]
        axis = rng.normal(size=3)
        from rvpose.geometry import rotation_about_axis
        T = RigidTransform(rotation_about_axis(axis, ang), rng.normal(size=3) / 3 ** 0.5 * shift)
        src = T.inverse().apply(tgt[rng.permutation(400)[:250]])
        ca, cb = rg.estimate_covariances(src), rg.estimate_covariances(tgt)
        h, g = np.zeros((6, 6)), np.zeros(6)
        corr, wb = np.empty(250, dtype=np.int64), np.zeros((250, 3, 3))
        f0, ncorr = rg._gicp_linearize(src, tgt, ca, cb, np.eye(3), np.zeros(3), cfg.max_correspondence_distance ** 2,
                                       h, g, corr, wb)
        reg = rg.gicp_align(src, tgt, ca, cb, RigidTransform.identity(), cfg)
        d[f"gicp{t}_src"], d[f"gicp{t}_tgt"], d[f"gicp{t}_ca"], d[f"gicp{t}_cb"] = src, tgt, ca, cb
        d[f"gicp{t}_h"], d[f"gicp{t}_g"], d[f"gicp{t}_f0"], d[f"gicp{t}_ncorr"] = h, g, np.array(f0), np.array(ncorr)
        d[f"gicp{t}_corr"], d[f"gicp{t}_w"] = corr, wb
        d[f"gicp{t}_T"] = reg.transform.matrix3x4()
        d[f"gicp{t}_iters"], d[f"gicp{t}_conv"] = np.array(reg.iterations), np.array(int(reg.converged))
        d[f"gicp{t}_resid"] = np.array(reg.final_residual)
        d[f"gicp{t}_trace"] = np.array(reg.objective_trace).reshape(-1, 2)
    np.savez_compressed(OUT / "units.npz", **d)
    print(f"[units] -> {(OUT / 'units.npz').stat().st_size / 1024:.0f} KiB", flush=True)


def tiny_dataset():
    """A small scene + models directory WRITTEN BY THE REFERENCE (save_scene / save_models,
    scenegen.py:542-625) and its `estimate` result JSON: pins paper_2008_00326_b200.io and
    the CLI (tests/test_host_api.py, tests/test_gpu_parity.py)."""
    import shutil
    k = sg.make_camera(96, 72)
    models = {1: sg.mixed_object_suite()[1], 2: sg.mixed_object_suite()[2]}
    spec = sg.SceneSpec(((1, lift_pose3dof(Pose3Dof(0.05, -0.04, 0.6), 0.0)),
                         (2, lift_pose3dof(Pose3Dof(-0.08, 0.06, 0.0), 0.0))), (0.42, 0.42), k)
    frame = disk_roundtrip(sg.generate_scene(spec, models))
    d = OUT / "dataset_tiny"
    shutil.rmtree(d, ignore_errors=True)
    sg.save_scene(d / "scene_0000", frame)
    sg.save_models(d / "models", models)
    cfg = rs.SearchConfig(mode="3dof", workspace=(-0.16, 0.16, -0.16, 0.16), stride=1, workers=WORKERS)
    res = rs.estimate_poses(sg.load_scene(d / "scene_0000"), sg.load_models(d / "models"), cfg)
    (d / "config.json").write_text(json.dumps({k_: v for k_, v in cfg.to_dict().items() if k_ != "workers"}, indent=2, sort_keys=True))
    (d / "results_reference.json").write_text(rs.result_to_json(res))
    print("[dataset_tiny]", sum(f.stat().st_size for f in d.rglob("*") if f.is_file()) // 1024, "KiB", flush=True)


def dense_fixture(name, frame, models, cfg):
    """Per-candidate outputs of the reference at the BENCHMARK's own grid density (dt 0.025, no subsampling) on a
    sub-workspace of the C3 scene: integer costs, refined poses, GICP iteration counts,
    final-render point counts and the result JSON.  The scene itself is the one stored in c3_clutter_3dof.npz (its
    depth digest is kept here to prove it)."""
    import dataclasses
    print(f"[{name}] staged reference run ...", flush=True)
    st = staged_search(frame, models, cfg)
    trace = tempfile.mktemp(suffix=".jsonl")
    res = rs.estimate_poses(frame, models, dataclasses.replace(cfg, trace_path=trace))
    rows = [json.loads(line) for line in open(trace)]
    assert len(rows) == len(st["flat"])
    d = {"cfg_json": np.array(json.dumps({**cfg.to_dict(), "max_proposals": cfg.max_proposals})),
         "scene_digest": np.frombuffer(sha(pack_frame(frame)["depth_mm"]), dtype=np.uint8),
         "flat_oid": np.array([f[0] for f in st["flat"]], dtype=np.int32),
         "flat_local": np.array([f[1] for f in st["flat"]], dtype=np.int32),
         "refined": np.array([p.matrix3x4() for p in st["refined"]]),
         "reg_iters": np.array([r.iterations for r in st["regs"]], dtype=np.int8),
         "n0": np.array([len(c) for c in st["clouds0"]], dtype=np.int16),
         "n1": np.array([len(c) for c in st["clouds1"]], dtype=np.int16),
         "j_o": np.array([r["j_o"] for r in rows], dtype=np.int16),
         "j_r": np.array([r["j_r"] for r in rows], dtype=np.int16),
         "result_json": np.array(rs.result_to_json(res))}
    assert max(r["j_o"] for r in rows) < 32767 and max(r["j_r"] for r in rows) < 32767
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"[{name}] n={len(rows)} -> {(OUT / (name + '.npz')).stat().st_size / 1024:.0f} KiB", flush=True)


def full_fixture(name, frame, models, cfg):
    """Per-candidate outputs of the reference on the WHOLE benchmark step (BASELINE configs[2] as bench.py measures it:
    58,320 candidates of the C3 scene, dt 0.025): integer costs, GICP iteration counts, first / final render point counts,
    the result JSON, and every refined pose as its world-frame (x, y, yaw) -- a 3-DoF refined pose is re-lifted onto
    the table (search.py:291-301), so these three numbers are the whole pose (kept in float64, 1.4 MB)."""
    import dataclasses
    print(f"[{name}] staged reference run ...", flush=True)
    st = staged_search(frame, models, cfg)
    c2w = frame.intrinsics.camera_pose
    xyyaw = np.empty((len(st["flat"]), 3))
    for j, p in enumerate(st["refined"]):
        w = c2w.compose(p)
        xyyaw[j] = (w.translation[0], w.translation[1], np.arctan2(w.rotation[1, 0], w.rotation[0, 0]))
    d = {"cfg_json": np.array(json.dumps({**cfg.to_dict(), "max_proposals": cfg.max_proposals})),
         "scene_digest": np.frombuffer(sha(pack_frame(frame)["depth_mm"]), dtype=np.uint8),
         "xyyaw": xyyaw,
         "reg_iters": np.array([r.iterations for r in st["regs"]], dtype=np.int8),
         "n0": np.array([len(c) for c in st["clouds0"]], dtype=np.int16),
         "n1": np.array([len(c) for c in st["clouds1"]], dtype=np.int16)}
    n = len(st["flat"])
    del st
    print(f"[{name}] full reference run with trace ...", flush=True)
    trace = tempfile.mktemp(suffix=".jsonl")
    res = rs.estimate_poses(frame, models, dataclasses.replace(cfg, trace_path=trace))
    rows = [json.loads(line) for line in open(trace)]
    assert len(rows) == n
    assert max(r["j_o"] for r in rows) < 32767 and max(r["j_r"] for r in rows) < 32767
    d["j_o"] = np.array([r["j_o"] for r in rows], dtype=np.int16)
    d["j_r"] = np.array([r["j_r"] for r in rows], dtype=np.int16)
    d["result_json"] = np.array(rs.result_to_json(res))
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"[{name}] n={n} -> {(OUT / (name + '.npz')).stat().st_size / 1024:.0f} KiB", flush=True)


def full_fixture_6dof(name, frame, models, cfg, pose_every=8):
    """Same for the 6-DoF workload bench.py --workload c4 measures (BASELINE configs[3], 249,738 mask-constrained
    candidates): integer costs, GICP iteration counts and first / final render point counts of EVERY candidate (the final
    count is a function of the refined pose), the refined pose itself (translation + unit quaternion, float32) of every
    `pose_every`-th, and the result JSON."""
    import dataclasses
    print(f"[{name}] staged reference run ...", flush=True)
    st = staged_search(frame, models, cfg)
    n = len(st["flat"])
    sel = np.arange(0, n, pose_every)
    tv = np.empty((sel.size, 7), dtype=np.float32)  # translation, unit quaternion (w, x, y, z)
    for q, j in enumerate(sel):
        p = st["refined"][j]
        r = p.rotation
        # Shepperd's method: the largest of (trace, r00, r11, r22) picks a well-conditioned branch at every angle
        c = [r[0, 0] + r[1, 1] + r[2, 2], r[0, 0], r[1, 1], r[2, 2]]
        b = int(np.argmax(c))
        if b == 0:
            qq = [1.0 + c[0], r[2, 1] - r[1, 2], r[0, 2] - r[2, 0], r[1, 0] - r[0, 1]]
        elif b == 1:
            qq = [r[2, 1] - r[1, 2], 1.0 + 2 * r[0, 0] - c[0], r[0, 1] + r[1, 0], r[0, 2] + r[2, 0]]
        elif b == 2:
            qq = [r[0, 2] - r[2, 0], r[0, 1] + r[1, 0], 1.0 + 2 * r[1, 1] - c[0], r[1, 2] + r[2, 1]]
        else:
            qq = [r[1, 0] - r[0, 1], r[0, 2] + r[2, 0], r[1, 2] + r[2, 1], 1.0 + 2 * r[2, 2] - c[0]]
        qq = np.array(qq) / np.linalg.norm(qq)
        tv[q] = (*p.translation, *qq)
    d = {"cfg_json": np.array(json.dumps({**cfg.to_dict(), "max_proposals": cfg.max_proposals})),
         "scene_digest": np.frombuffer(sha(pack_frame(frame)["depth_mm"]), dtype=np.uint8),
         "pose_every": np.array(pose_every), "pose_tv": tv,
         "reg_iters": np.array([r.iterations for r in st["regs"]], dtype=np.int8),
         "n0": np.array([len(c) for c in st["clouds0"]], dtype=np.int16),
         "n1": np.array([len(c) for c in st["clouds1"]], dtype=np.int16)}
    del st
    print(f"[{name}] full reference run with trace ...", flush=True)
    trace = tempfile.mktemp(suffix=".jsonl")
    res = rs.estimate_poses(frame, models, dataclasses.replace(cfg, trace_path=trace))
    rows = [json.loads(line) for line in open(trace)]
    assert len(rows) == n
    assert max(r["j_o"] for r in rows) < 32767 and max(r["j_r"] for r in rows) < 32767
    d["j_o"] = np.array([r["j_o"] for r in rows], dtype=np.int16)
    d["j_r"] = np.array([r["j_r"] for r in rows], dtype=np.int16)
    d["result_json"] = np.array(rs.result_to_json(res))
    np.savez_compressed(OUT / f"{name}.npz", **d)
    print(f"[{name}] n={n} -> {(OUT / (name + '.npz')).stat().st_size / 1024:.0f} KiB", flush=True)


def main():
    OUT.mkdir(parents=True, exist_ok=True)
    which = set(sys.argv[1:]) or {"units", "c1", "c2", "c3", "c3n", "c4", "tiny", "c3d"}
    if "c4f" in which:  # ~45 minutes on 8 cores: only on request
        frame, models = scene_c4()
        full_fixture_6dof("c4f_full_reference", frame, models,
                          rs.SearchConfig(mode="6dof", viewpoints=642, n_inplane=36, z_step=0.01, max_proposals=None,
                                          workers=WORKERS))
    if "c3f" in which:  # ~5 minutes on 8 cores: only on request
        frame, models = scene_c3()
        full_fixture("c3f_full_reference", frame, models,
                     rs.SearchConfig(mode="3dof", workspace=(-0.32, 0.32, -0.32, 0.32), dt=0.025, workers=WORKERS))
    if "c3d" in which:
        frame, models = scene_c3()
        dense_fixture("c3d_dense_reference", frame, models,
                      rs.SearchConfig(mode="3dof", workspace=(-0.125, 0.125, -0.125, 0.125), dt=0.025, workers=WORKERS))
    if "tiny" in which:
        tiny_dataset()
    if "units" in which:
        unit_fixtures()
    if "c1" in which:
        frame, models = scene_c1()
        search_fixture("c1_box_3dof", frame, models,
                       rs.SearchConfig(mode="3dof", workspace=(-0.4, 0.4, -0.4, 0.4), workers=WORKERS))
    if "c2" in which:
        frame, models = scene_c2()
        for uc in (True, False):
            search_fixture(f"c2_twocyl_color{int(uc)}", frame, models,
                           rs.SearchConfig(mode="3dof", workspace=(-0.32, 0.32, -0.32, 0.32), dt=0.04,
                                           use_color=uc, workers=WORKERS), keep_every=41)
    if "c3" in which:
        frame, models = scene_c3()
        search_fixture("c3_clutter_3dof", frame, models,
                       rs.SearchConfig(mode="3dof", workspace=(-0.32, 0.32, -0.32, 0.32), dt=0.02,
                                       max_proposals=1500, workers=WORKERS), keep_every=211)
    if "c3n" in which:
        frame, models = scene_c3_noisy()
        search_fixture("c3n_clutter_noisy", frame, models,
                       rs.SearchConfig(mode="3dof", workspace=(-0.32, 0.32, -0.32, 0.32), dt=0.02,
                                       max_proposals=700, workers=WORKERS), keep_every=233)
    if "c4" in which:
        frame, models = scene_c4()
        search_fixture("c4_mixed_6dof", frame, models,
                       rs.SearchConfig(mode="6dof", max_proposals=1000, workers=WORKERS), keep_every=173)


if __name__ == "__main__":
    main()
