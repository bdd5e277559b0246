"""CPU tests of the host-side mirror of the reference interface and of the C-ABI
surface (no compute calls: those need a GPU)."""

import ctypes
import json
import math
import re
from pathlib import Path

import numpy as np
import pytest

import golden_io as G
import paper_2008_00326_b200 as px
from paper_2008_00326_b200 import _native
from paper_2008_00326_b200.errors import ConfigError, DeviceError, EmptyBatch
from paper_2008_00326_b200.proposals import _inclusive_range, compose_many
from paper_2008_00326_b200.search import assemble_result, plan_search, StageOutputs

ROOT = Path(__file__).resolve().parent.parent


def test_cabi_exports_every_declared_symbol():
    """libpx.so loads without a GPU and exports exactly what include/px.h declares."""
    header = (ROOT / "include" / "px.h").read_text()
    declared = set(re.findall(r"\b(px_[a-z_0-9]+)\s*\(", header))
    lib = ctypes.CDLL(str(_native.lib_path()))
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert declared == set(_native.EXPORTS), declared ^ set(_native.EXPORTS)


def test_no_cpu_fallback_without_device():
    """Without a CUDA device the product fails loudly (never a silent CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(DeviceError, match="no CUDA device|CUDA"):
        px.engine.Engine(0) if hasattr(px, "engine") else __import__("paper_2008_00326_b200.engine", fromlist=["Engine"]).Engine(0)
    d, frame, models, cfg, plan = G.scene("c1_box_3dof")
    with pytest.raises(DeviceError):
        px.estimate_poses(frame, models, cfg)
    with pytest.raises(DeviceError):
        px.rendered_cost(plan.observed.subset(np.arange(5)), plan.observed, px.CostParams())


def test_product_never_imports_oracle():
    for f in (ROOT / "paper_2008_00326_b200").rglob("*.py"):
        assert "oracle" not in f.read_text(), f
    for f in (ROOT / "paper_2008_00326_b200" / "csrc").iterdir():
        if f.is_file():
            txt = f.read_text()
            assert "px_oracle" not in txt and "liborc" not in txt, f


def test_search_config_validation_and_roundtrip():
    # reference search.py:63-81, 91-144
    with pytest.raises(ConfigError):
        px.SearchConfig(mode="9dof")
    with pytest.raises(ConfigError):
        px.SearchConfig(mode="3dof")  # workspace required
    with pytest.raises(ConfigError):
        px.SearchConfig(mode="3dof", workspace=(1, 0, 0, 1))
    with pytest.raises(ConfigError):
        px.SearchConfig(stride=0)
    with pytest.raises(ConfigError):
        px.SearchConfig(delta=0.0)
    with pytest.raises(ConfigError):
        px.SearchConfig.from_dict({"bogus": 1})
    with pytest.raises(ConfigError):
        px.SearchConfig.from_dict({"gicp": {"k_covariance": 2}})
    c = px.SearchConfig(mode="3dof", workspace=(-0.4, 0.4, -0.4, 0.4), dyaw=math.radians(10.0), workers=3)
    c2 = px.SearchConfig.from_dict(c.to_dict())
    assert c2.workspace == c.workspace and abs(c2.dyaw - c.dyaw) < 1e-15 and c2.gicp == c.gicp
    assert c.cost_params == px.CostParams(c.delta, c.tau_c, c.use_color) and c.knn_config.k == 1


def test_select_best_and_types():
    from paper_2008_00326_b200 import CostBreakdown
    costs = [CostBreakdown(3, 4), CostBreakdown(1, 2), CostBreakdown(2, 1), CostBreakdown(9, 9)]
    assert px.select_best(costs) == 1          # ties -> lowest index (search.py:178-183)
    with pytest.raises(EmptyBatch):
        px.select_best([])
    with pytest.raises(ValueError):
        CostBreakdown(-1, 0)
    with pytest.raises(ValueError):
        px.GicpConfig(k_covariance=3)
    with pytest.raises(ValueError):
        px.RigidTransform(np.eye(3) * 2.0, np.zeros(3))
    cyl = px.InscribedCylinder(0.05, 0.0, 0.1)
    assert cyl.contains(np.array([[0.05, 0.0, 0.05], [0.050001, 0.0, 0.05]])).tolist() == [True, False]


def test_inclusive_range_reference_behaviour():
    # proposals.py:97-105 always appends `hi` when the last step falls short
    assert np.allclose(_inclusive_range(0.0, 0.05, 0.08), [0.0, 0.05])
    assert len(_inclusive_range(-0.4, 0.4, 0.08)) == 11
    g = px.grid_proposals_3dof((-0.4, 0.4, -0.4, 0.4), 0.08, math.radians(22.5), 0.0)
    assert len(g) == 11 * 11 * 16 and g.provenance[-1].tolist() == [120, 15]
    s = px.grid_proposals_3dof((-0.4, 0.4, -0.4, 0.4), 0.08, math.radians(22.5), 0.0, yaw_symmetric=True)
    assert len(s) == 121


def test_compose_many_matches_per_item_bits():
    rng = np.random.default_rng(0)
    from paper_2008_00326_b200.geometry import rotation_about_axis
    a = px.RigidTransform(rotation_about_axis(rng.normal(size=3), 0.7), rng.normal(size=3))
    rots = np.stack([rotation_about_axis(rng.normal(size=3), rng.uniform(-3, 3)) for _ in range(40)])
    trs = rng.normal(size=(40, 3))
    for t in (a, a.inverse()):  # C-contiguous rotation and transposed view
        r, tr = compose_many(t, rots, trs)
        for i in range(40):
            ref = t.compose(px.RigidTransform(rots[i], trs[i]))
            assert np.array_equal(r[i], ref.rotation) and np.array_equal(tr[i], ref.translation)


def test_quantize_frame_is_disk_roundtrip_equivalent():
    d, frame, models, cfg, plan = G.scene("c2_twocyl_color1")
    q = px.quantize_frame(frame)  # fixture frames already went through the reference's save/load
    assert np.array_equal(q.color, frame.color) and np.array_equal(q.depth.values, frame.depth.values)
    assert np.array_equal(q.labels, frame.labels) and np.array_equal(q.depth.valid, frame.depth.valid)


def test_assemble_result_and_json():
    d, frame, models, cfg, plan = G.scene("c4_mixed_6dof")
    out = StageOutputs(plan.cam_poses.copy(), np.tile(np.hstack([np.eye(3), np.zeros((3, 1))]), (plan.n, 1, 1)),
                       d["j_o"].copy(), d["j_r"].copy(), n_rendered=d["n1"])
    res = assemble_result(plan, out, 0.0)
    js = json.loads(px.result_to_json(res))
    ref = json.loads(str(d["result_json"]))
    assert set(res.stage_millis) == {"render", "refine", "rerender", "cost"}
    for a, b in zip(js["objects"], ref["objects"]):
        assert (a["object_id"], a["proposal_index"], a["j_o"], a["j_r"], a["provenance"]) == \
               (b["object_id"], b["proposal_index"], b["j_o"], b["j_r"], b["provenance"])
    assert "stage_millis" in json.loads(px.timings_to_json(res))


def test_plan_failures_are_data():
    # search.py:237-251: unknown objects are per-object failures, not exceptions
    d, frame, models, cfg, plan = G.scene("c4_mixed_6dof")
    fewer = {k: v for k, v in models.items() if k != 2}
    p = plan_search(frame, fewer, cfg, build_targets=False)
    assert p.failures == {2: "unknown_object"} and 2 not in p.active
    out = StageOutputs(p.cam_poses, p.cam_poses, np.zeros(p.n, np.int32), np.zeros(p.n, np.int32))
    est = assemble_result(p, out, 0.0).estimate_for(2)
    assert est.failed and est.failure == "unknown_object"
    with pytest.raises(ConfigError):
        plan_search(dataclass_replace(frame, detections=[]), models, cfg)


def dataclass_replace(obj, **kw):
    import dataclasses
    return dataclasses.replace(obj, **kw)


# ---- dataset I/O and CLI plumbing (reference: scenegen.py:542-625, model.py:223-350, cli.py:40-215) ----

DATASET = Path(__file__).resolve().parent / "golden" / "dataset_tiny"


def test_io_roundtrip_is_byte_identical_to_reference_files(tmp_path):
    """tests/golden/dataset_tiny was written by the reference's save_scene / save_models
    (oracle/make_golden.py tiny): reading it with this package and writing it back
    must reproduce every file byte for byte."""
    import filecmp
    from paper_2008_00326_b200 import load_models, load_scene, save_models, save_scene
    frame, models = load_scene(DATASET / "scene_0000"), load_models(DATASET / "models")
    assert frame.depth.values.shape == (72, 96) and frame.labels.dtype == np.int32
    assert sorted(models) == [1, 2] and models[2].yaw_symmetric and not models[1].yaw_symmetric
    assert [d.object_id for d in frame.detections] == [1, 2] and frame.ground_truth is not None
    assert frame.detections[0].mask.sum() == (frame.labels == 1).sum()
    save_scene(tmp_path / "s", frame)
    save_models(tmp_path / "m", models)
    for f in ("scene.json", "color.ppm", "depth.pgm", "labels.pgm"):
        assert filecmp.cmp(tmp_path / "s" / f, DATASET / "scene_0000" / f, shallow=False), f
    for f in ("models.json", "object_001.ply", "object_002.ply"):
        assert filecmp.cmp(tmp_path / "m" / f, DATASET / "models" / f, shallow=False), f


def test_io_errors(tmp_path):
    from paper_2008_00326_b200 import load_models, load_scene
    from paper_2008_00326_b200.errors import DatasetError
    from paper_2008_00326_b200.io import load_depth_pgm, load_ply
    with pytest.raises(DatasetError):
        load_scene(tmp_path / "nope")
    with pytest.raises(DatasetError):
        load_models(tmp_path)
    (tmp_path / "x.ply").write_text("ply\nformat ascii 1.0\nelement vertex 3\nelement face 1\nend_header\n0 0 0 1 1 1\n")
    with pytest.raises(DatasetError):
        load_ply(tmp_path / "x.ply")
    (tmp_path / "d.pgm").write_bytes(b"P5\n# comment\n2 2\n255\n\x00\x00\x00\x00")
    with pytest.raises(DatasetError):
        load_depth_pgm(tmp_path / "d.pgm")  # 8-bit file where 16-bit depth is expected


def test_cli_exit_codes_without_device(tmp_path, capsys):
    """cli.py:40-59: config errors -> 2, dataset errors -> 3 (both raised before any device work)."""
    from paper_2008_00326_b200.cli import main
    bad = tmp_path / "cfg.json"
    bad.write_text('{"no_such_key": 1}')
    assert main(["estimate", "--scene", str(DATASET / "scene_0000"), "--models", str(DATASET / "models"),
                 "--out", str(tmp_path / "o"), "--config", str(bad)]) == 2
    assert main(["estimate", "--scene", str(tmp_path / "missing"), "--models", str(DATASET / "models"),
                 "--out", str(tmp_path / "o"), "--mode", "3dof"]) == 3
    assert main(["bench", "--scene", str(DATASET / "scene_0000"), "--models", str(DATASET / "models"),
                 "--workers", "0"]) == 2
    capsys.readouterr()


def test_blas_order_probe_passes_here_and_fails_loudly(monkeypatch):
    """the start-up probe accepts this host's numpy/BLAS and raises when the
    fused orders differ from what csrc/px_common.cuh bakes in."""
    from paper_2008_00326_b200 import blas_probe as B
    bad = B.check_blas_orders(force=True)
    assert not any(bad.values())
    # a host whose (3,3)@(3,) product used the k = 0,1,2 order instead of 1,0,2
    monkeypatch.setattr(B, "dot_f102", B.dot_f012)
    with pytest.raises(B.BlasOrderError, match="rounds small matrix products"):
        B.check_blas_orders(force=True)
    monkeypatch.undo()
    B.check_blas_orders(force=True)


def test_bench_gpus_flag_spawns_one_rank_per_gpu(monkeypatch):
    """`python bench.py --gpus N` without torchrun re-executes itself under torch.distributed.run
    with N ranks on 127.0.0.1 (the flag used to be parsed and ignored)."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, PX_BENCH_PRINT_SPAWN="1")
    env.pop("WORLD_SIZE", None)
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--steps", "2"], env=env,
                         capture_output=True, text=True, check=True).stdout
    cmd = json.loads(out.strip().splitlines()[-1])
    assert "torch.distributed.run" in cmd and "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]


@pytest.mark.parametrize("name,over", [("c1_box_3dof", {}), ("c2_twocyl_color1", {}),
                                       ("c4_mixed_6dof", dict(viewpoints=8, n_inplane=3, max_proposals=None))])
def test_lattice_plan_factors_reproduce_the_flat_plan(name, over):
    """plan_lattice hands the device each object's proposal set as outer x inner FACTORS (px_search_upload_lattice);
    expanding them on the host with the reference's own composition gives exactly plan_search's flat candidate
    list (object ids, poses, counts, provenance) -- the GPU test checks the device expansion against the same arrays."""
    import dataclasses
    from paper_2008_00326_b200.geometry import RigidTransform
    from paper_2008_00326_b200.search import plan_lattice
    d, frame, models, cfg, _ = G.scene(name)
    cfg = dataclasses.replace(cfg, **over)
    flat = plan_search(frame, models, cfg, build_targets=False)
    lat = plan_lattice(frame, models, cfg)
    assert lat.n == flat.n and lat.active == flat.active and lat.object_ids == flat.object_ids
    w2c = RigidTransform.from_matrix3x4(flat.w2c) if flat.w2c_vec_order == 0 else flat.cam_to_world.inverse()
    row = 0
    for f in lat.lattice:
        assert lat.count_of(f.object_id) == flat.count_of(f.object_id) == f.n_outer * f.n_inner
        for outer in range(f.n_outer):
            for inner in range(0, f.n_inner, max(1, f.n_inner // 3)):
                j = row + outer * f.n_inner + inner
                if cfg.mode == "3dof":
                    pose = w2c.compose(RigidTransform(f.rotations[inner].copy(), f.translations[outer].copy()))
                    want = np.concatenate([pose.rotation, pose.translation[:, None]], axis=1)
                else:
                    want = np.concatenate([f.rotations[outer], f.translations[inner][:, None]], axis=1)
                assert np.array_equal(flat.cam_poses[j], want)
                assert lat.provenance_of(f.object_id, outer * f.n_inner + inner) == flat.provenance_of(f.object_id, outer * f.n_inner + inner)
        row += f.n_outer * f.n_inner
    assert plan_lattice(frame, models, dataclasses.replace(cfg, max_proposals=10)) is None  # subsampling needs the flat plan
