"""GPU parity tests: the CUDA path (through the C-ABI) against the reference's
golden outputs and against the CPU oracle on the same inputs.

Bit-exact: z-buffer depth/colour/validity/owner, cloud points and source pixels,
kNN, covariances, the first GICP linearisation objective, integer costs, argmin.
Tolerance (stated per test): Lab (libdevice pow/cbrt vs numpy), refined poses
(libdevice sin/cos/atan2 vs libm inside a chaotic iteration).
"""

import dataclasses
import json

import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O
from paper_2008_00326_b200 import (CameraIntrinsics, CostParams, GicpConfig, LabeledCloud, RigidTransform,
                                   TriangleMesh, cost, registration)
from paper_2008_00326_b200.search import assemble_result, result_to_json

pytestmark = pytest.mark.gpu
U = G.load("units")
I34 = np.hstack([np.eye(3), np.zeros((3, 1))])
K64 = CameraIntrinsics(500.0, 500.0, 32.0, 32.0, 64, 64, RigidTransform.identity())


class _LinMesh:
    """Mesh whose colours are already linear light (fixture colours)."""
    def __init__(self, v, c, t):
        self.vertices, self.triangles = v, t
        # invert srgb_decode so that the engine's host decode reproduces c: not exact in general,
        # therefore the dense test patches colours through an sRGB round trip only for validity/depth/owner
        self.vertex_colors = c
        self.num_triangles = t.shape[0]


@pytest.mark.parametrize("t", range(6))
def test_rasterize_dense_bit_exact(engine, t):
    """z-buffer visibility and per-pixel ownership vs the reference kernel
    (depth, validity) and the oracle (owner, colour) -- tests/test_raster.py:68-97."""
    v, c, tr = U[f"ras{t}_verts"], U[f"ras{t}_cols"], U[f"ras{t}_tris"]
    mesh = TriangleMesh(v, c, tr)
    z, cb, valid, owner = engine.rasterize_mesh(mesh, RigidTransform.identity(), K64)
    assert np.array_equal(valid, U[f"ras{t}_valid"])
    assert np.array_equal(z, U[f"ras{t}_z"])
    om = O.OracleModel(1, mesh)  # same host srgb_decode of the colours as the engine
    oz, oc, ov, oo = O.rasterize(om, I34, K64)
    assert np.array_equal(owner, oo)
    assert np.array_equal(cb[valid], oc[ov])


def test_rasterize_large_mesh_atomic_path(engine):
    """> PX_TRI_SMEM triangles and several z tiles: the two-pass atomic path."""
    d = G.load("c4_mixed_6dof")
    models = G.models_of(d)
    frame = G.frame_of(d)
    k = frame.intrinsics
    for oid in (2, 4):
        mesh = models[oid].mesh
        assert mesh.num_triangles > 64
        pose = d["cam_poses"][np.nonzero(d["flat_oid"] == oid)[0][3]]
        T = RigidTransform.from_matrix3x4(pose)
        z, cb, valid, owner = engine.rasterize_mesh(mesh, T, k)
        oz, oc, ov, oo = O.rasterize(O.OracleModel(oid, mesh), pose, k)
        assert valid.sum() > 100
        assert np.array_equal(valid, ov) and np.array_equal(z, oz) and np.array_equal(owner, oo)
        assert np.array_equal(cb[valid], oc[ov])


@pytest.mark.parametrize("t", range(4))
def test_knn_exact(engine, t):
    idx, d2 = engine.knn(U[f"knn{t}_q"], U[f"knn{t}_t"], int(U[f"knn{t}_k"]))
    assert np.array_equal(idx, U[f"knn{t}_idx"]) and np.array_equal(d2, U[f"knn{t}_d2"])


def test_knn_empty(engine):
    idx, d2 = engine.knn(np.zeros((3, 3)), np.zeros((0, 3)), 2)
    assert (idx == -1).all() and np.isinf(d2).all()


def test_rendered_cost_generic_exact(engine):
    """tests/test_cost.py:102-125: (j_o, j_r) and the explained set, exact."""
    z2 = lambda n: np.zeros((n, 2), dtype=np.int32)
    for i in range(int(U["cost_n"])):
        delta, tau, uc = U[f"cost{i}_par"]
        ren = LabeledCloud(U[f"cost{i}_rp"], U[f"cost{i}_rl"], z2(len(U[f"cost{i}_rp"])))
        obs = LabeledCloud(U[f"cost{i}_op"], U[f"cost{i}_ol"], z2(len(U[f"cost{i}_op"])))
        jr, ex = cost.rendered_cost(ren, obs, CostParams(float(delta), float(tau), bool(uc)))
        jo = int(np.count_nonzero(U[f"cost{i}_sel"] & ~ex))
        assert (jo, jr) == tuple(U[f"cost{i}_out"]), i
        assert np.array_equal(ex, U[f"cost{i}_expl"])


@pytest.mark.parametrize("t", range(4))
def test_covariances_bit_exact(engine, t):
    assert np.array_equal(registration.estimate_covariances(U[f"gicp{t}_src"]), U[f"gicp{t}_ca"])
    assert np.array_equal(registration.estimate_covariances(U[f"gicp{t}_tgt"]), U[f"gicp{t}_cb"])


@pytest.mark.parametrize("t", range(4))
def test_m2m_gicp_matches_reference(engine, t):
    cfg = GicpConfig()
    res = registration.m2m_gicp([U[f"gicp{t}_src"]], [U[f"gicp{t}_tgt"]], [RigidTransform.identity()], cfg)[0]
    ref_tr = U[f"gicp{t}_trace"]
    # lock-step: the first linearisation objective is a fixed-order sum -> bit-exact
    assert res.objective_trace[0][0] == ref_tr[0, 0]
    assert res.iterations == int(U[f"gicp{t}_iters"]) and res.converged == bool(U[f"gicp{t}_conv"])
    assert res.failure is None
    dt, dr = G.pose_delta(res.transform.matrix3x4(), U[f"gicp{t}_T"])
    assert dt < 1e-9 and dr < 1e-7
    assert np.allclose(np.array(res.objective_trace), ref_tr, rtol=1e-6, atol=1e-12)
    assert abs(res.final_residual - float(U[f"gicp{t}_resid"])) < 1e-9


def test_m2m_gicp_failure_slots(engine):
    """registration.py:504-510 / tests/test_registration.py:219-226: per-slot
    failures never abort the batch."""
    rng = np.random.default_rng(0)
    big, small = rng.normal(size=(200, 3)) * 0.05, rng.normal(size=(10, 3)) * 0.05
    far = big + 10.0
    cfg = GicpConfig()
    ident = RigidTransform.identity()
    out = registration.m2m_gicp([big, small, far], [big, big, big], [ident] * 3, cfg, [0, 1, 2])
    assert out[0].failure is None and out[0].iterations >= 1
    assert out[1].failure == "too_few_points" and out[1].iterations == 0 and out[1].transform is ident
    assert out[2].failure == "degenerate_correspondences" and out[2].iterations == 1


# candidates whose GICP iteration is chaotic under last-bit differences of the linear solve / libm
# (reference 16 iterations, restated arithmetic 30): 1 of 1,500 in C3, none elsewhere
KNOWN_CHAOTIC = {"c3_clutter_3dof": {1131}}

SEARCH = ["c1_box_3dof", "c2_twocyl_color1", "c2_twocyl_color0", "c3_clutter_3dof", "c3n_clutter_noisy", "c4_mixed_6dof"]


@pytest.mark.parametrize("name", SEARCH)
def test_render_batch_bit_exact(engine, name):
    """Every candidate's first render: count, points and source pixels equal the
    reference's bit for bit (digest), kept clouds element-wise, Lab to 1e-9."""
    d, frame, models, cfg, plan = G.scene(name)
    engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
    engine.upload_models(models)
    h = engine.render_clouds_handle(plan.flat_oid, plan.cam_poses, cfg.occluder_marking, cfg.delta)
    try:
        clouds = engine._download_clouds(h)
    finally:
        engine.lib.px_clouds_free(engine.ctx, h)
    assert np.array_equal(np.array([len(c) for c in clouds]), d["n0"])
    bad = [j for j, c in enumerate(clouds) if not np.array_equal(G.cloud_digest(c.points, c.source_pixel), d["dig0"][j])]
    assert not bad, f"{len(bad)} of {len(clouds)} clouds differ, first {bad[:5]}"
    for j in d["keep"]:
        j = int(j)
        if len(clouds[j]):
            assert np.abs(clouds[j].lab_colors - d[f"c0_{j}_lab"]).max() < 1e-9


def test_render_batch_public_api_and_flags(engine):
    """raster.render_batch signature: grouped proposals in, flat clouds out;
    occluder flag off == plain render (tests/test_raster.py:164-191)."""
    from paper_2008_00326_b200 import render_batch
    d, frame, models, cfg, plan = G.scene("c3_clutter_3dof")
    sel = np.arange(0, plan.n, 37)
    groups = {}
    for j in sel:
        groups.setdefault(int(plan.flat_oid[j]), []).append(RigidTransform.from_matrix3x4(plan.cam_poses[j]))
    props = [(oid, groups[oid]) for oid in plan.active if oid in groups]
    on = render_batch(models, props, frame, frame.intrinsics, cfg.stride, True, cfg.delta)
    off = render_batch(models, props, frame, frame.intrinsics, cfg.stride, False, cfg.delta)
    assert len(on) == len(off) == len(sel)
    order = [j for oid in plan.active for j in sel if plan.flat_oid[j] == oid]
    for c, j in zip(on, order):
        assert np.array_equal(G.cloud_digest(c.points, c.source_pixel), d["dig0"][j])
    assert any(len(a) < len(b) for a, b in zip(on, off))       # something is occluded in the clutter scene
    assert all(len(a) <= len(b) for a, b in zip(on, off))      # marking is monotone
    sc = O.OracleScene(frame, cfg.stride, plan.observed, plan.obs_labels)
    for c, j in list(zip(off, order))[::5]:
        oid = int(plan.flat_oid[j])
        pts, lab, src = O.render_one(sc, O.OracleModel(oid, models[oid].mesh), plan.cam_poses[j], False, cfg.delta)
        assert np.array_equal(c.points, pts) and np.array_equal(c.source_pixel, src)


@pytest.fixture(scope="module")
def runs(engine):
    cache = {}

    def run(name):
        if name not in cache:
            d, frame, models, cfg, plan = G.scene(name)
            cache[name] = (engine.run_plan(frame, models, plan), O.run_plan(frame, models, plan))
        return cache[name]
    return run


@pytest.mark.parametrize("name", SEARCH)
def test_target_covariances_bit_exact(engine, name):
    d, frame, models, cfg, plan = G.scene(name)
    if not cfg.refine:
        pytest.skip("no refine")
    engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
    engine.upload_targets(plan.target_offsets, plan.target_points, cfg.gicp, plan.target_obs_index)
    cov = engine.target_covariances(int(plan.target_offsets[-1]))
    for t in range(0, len(plan.target_offsets) - 1, max(1, (len(plan.target_offsets) - 1) // 12)):
        a, b = int(plan.target_offsets[t]), int(plan.target_offsets[t + 1])
        if b - a > cfg.gicp.k_covariance:
            assert np.array_equal(cov[a:b], O.covariances(plan.target_points[a:b]))


@pytest.mark.parametrize("name", SEARCH)
def test_search_matches_oracle_and_reference(engine, runs, name):
    """Whole path.  vs oracle on identical inputs: first/final render counts,
    GICP iteration counts and refined poses (tolerance 1e-4 m / 1e-4 rad, fraction
    reported), integer costs exact wherever the refined pose agrees, argmin exact.
    vs reference golden: per-object winner index, integer costs, winner pose."""
    d, frame, models, cfg, plan = G.scene(name)
    dev, cpu = runs(name)
    assert np.array_equal(dev.n_first, cpu.n_first) and np.array_equal(dev.n_first, d["n0"])
    dt, dr = G.pose_delta(dev.refined_cam, cpu.refined_cam)
    close = (dt <= 1e-4) & (dr <= 1e-4)
    same = (dev.j_o == cpu.j_o) & (dev.j_r == cpu.j_r)
    same_ref = (dev.j_o == d["j_o"]) & (dev.j_r == d["j_r"])
    it_eq = dev.iterations == cpu.iterations
    rt, rr = G.pose_delta(dev.refined_cam, d["refined"])
    close_ref = (rt <= 1e-4) & (rr <= 1e-4)
    print(f"{name}: n={plan.n} pose-agree(oracle)={close.mean():.4f} pose-agree(reference)={close_ref.mean():.4f} "
          f"iters-equal={it_eq.mean():.4f} costs-equal(oracle)={same.mean():.4f} costs-equal(reference)={same_ref.mean():.4f} "
          f"max dt={dt.max():.3e}; divergent vs oracle {np.nonzero(~close)[0].tolist()}, vs reference {np.nonzero(~close_ref)[0].tolist()}")
    # Pinned to what is measured: every candidate of every fixture agrees with the oracle AND the
    # reference in pose (1e-4 m / 1e-4 rad) and in both integer costs, except the ONE chaotic candidate of C3 named in
    # KNOWN_CHAOTIC, on which the reference (LAPACK dgesv / libm) and the restated arithmetic part ways.
    known = KNOWN_CHAOTIC.get(name, set())
    assert set(np.nonzero(~close)[0].tolist()) <= known and set(np.nonzero(~close_ref)[0].tolist()) <= known
    assert set(np.nonzero(~same)[0].tolist()) <= known and set(np.nonzero(~same_ref)[0].tolist()) <= known
    assert set(np.nonzero(~it_eq)[0].tolist()) <= known
    a = json.loads(result_to_json(assemble_result(plan, dev, 0.0)))
    b = json.loads(result_to_json(assemble_result(plan, cpu, 0.0)))
    ref = json.loads(str(d["result_json"]))
    for x, y, r in zip(a["objects"], b["objects"], ref["objects"]):
        for other in (y, r):
            assert x["failed"] == other["failed"]
            if x["failed"]:
                continue
            assert (x["proposal_index"], x["j_o"], x["j_r"], x["provenance"]) == \
                   (other["proposal_index"], other["j_o"], other["j_r"], other["provenance"])
            wt, wr = G.pose_delta(np.array(x["pose"]).reshape(3, 4), np.array(other["pose"]).reshape(3, 4))
            assert wt <= 1e-4 and wr <= 1e-4
    # fused device argmin key == host argmin
    for e in assemble_result(plan, dev, 0.0).estimates:
        if not e.failed:
            key = dev.best_keys[e.object_id]
            assert (key >> 32, key & 0xffffffff) == (e.cost.total, e.proposal_index)


@pytest.mark.parametrize("name", ["c1_box_3dof", "c4_mixed_6dof"])
def test_search_refine_off_exact(engine, name):
    """Without GICP nothing on the path is tolerance-based: every candidate's
    (j_o, j_r) equals the oracle's, and the result JSON is byte-identical."""
    d, frame, models, cfg, plan = G.scene(name)
    from paper_2008_00326_b200.search import plan_search
    cfg0 = dataclasses.replace(cfg, refine=False)
    plan0 = plan_search(frame, models, cfg0)
    dev, cpu = engine.run_plan(frame, models, plan0), O.run_plan(frame, models, plan0)
    assert np.array_equal(dev.j_o, cpu.j_o) and np.array_equal(dev.j_r, cpu.j_r)
    assert np.array_equal(dev.refined_cam, plan0.cam_poses)
    assert result_to_json(assemble_result(plan0, dev, 0.0)) == result_to_json(assemble_result(plan0, cpu, 0.0))


def test_cost_batch_stage_isolated(engine):
    """Stage-isolated cost: identical clouds and poses in, integers out (cylinder
    and label association), vs oracle rendered_cost / observed_cost."""
    for name in ("c1_box_3dof", "c4_mixed_6dof"):
        d, frame, models, cfg, plan = G.scene(name)
        engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
        engine.upload_models(models)
        sel = np.arange(0, plan.n, 13)
        h = engine.render_clouds_handle(plan.flat_oid[sel], plan.cam_poses[sel], cfg.occluder_marking, cfg.delta)
        try:
            clouds = engine._download_clouds(h)
            cyl = plan.cam_poses[sel] if cfg.mode == "3dof" else None
            jo, jr = engine.cost_handle(h, plan.flat_oid[sel], cyl, cfg.delta, cfg.tau_c, cfg.use_color)
        finally:
            engine.lib.px_clouds_free(engine.ctx, h)
        obs = plan.observed
        for q, j in enumerate(sel):
            c, oid = clouds[q], int(plan.flat_oid[j])
            ejr, ex = O.rendered_cost(c.points, c.lab_colors, obs.points, obs.lab_colors, cfg.delta, cfg.tau_c, cfg.use_color)
            if cfg.mode == "3dof":
                cy = models[oid].inscribed_cylinder
                ejo, _ = O.observed_cost_cyl(obs.points, plan.cam_poses[j], cy.radius ** 2, cy.z_min, cy.z_max, ex)
            else:
                ejo = int(np.count_nonzero((plan.obs_labels == oid) & ~ex))
            assert (int(jo[q]), int(jr[q])) == (ejo, ejr), (name, int(j))


def test_unknown_object_and_missing_state(engine):
    from paper_2008_00326_b200.errors import DeviceError, UnknownObjectId
    d, frame, models, cfg, plan = G.scene("c1_box_3dof")
    engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
    with pytest.raises(UnknownObjectId):
        engine.render_clouds_handle(np.array([12345]), plan.cam_poses[:1], True, 0.0075)


def test_estimate_poses_public_entry(engine):
    """The drop-in call: estimate_poses(frame, models, cfg) -> SearchResult."""
    from paper_2008_00326_b200 import estimate_poses
    d, frame, models, cfg, plan = G.scene("c2_twocyl_color1")
    res = estimate_poses(frame, models, cfg)
    ref = json.loads(str(d["result_json"]))
    assert set(res.stage_millis) == {"render", "refine", "rerender", "cost"}
    assert res.proposals_evaluated == ref["proposals_evaluated"] and res.observed_points == int(d["n_obs"])
    for e, r in zip(res.estimates, ref["objects"]):
        assert (e.object_id, e.proposal_index, e.cost.j_o, e.cost.j_r) == (r["object_id"], r["proposal_index"], r["j_o"], r["j_r"])


def test_organised_targets_equal_generic(engine):
    """The organised (pixel-ring) neighbour searches are exact: refining the same
    rendered clouds against targets uploaded with and without their
    observed-cloud indices gives bit-identical transforms, and so do the
    covariances."""
    d, frame, models, cfg, plan = G.scene("c3_clutter_3dof")
    engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
    engine.upload_models(models)
    sel = np.arange(0, plan.n, 7)
    h = engine.render_clouds_handle(plan.flat_oid[sel], plan.cam_poses[sel], cfg.occluder_marking, cfg.delta)
    try:
        clouds = engine._download_clouds(h)
        engine.upload_targets(plan.target_offsets, plan.target_points, cfg.gicp, plan.target_obs_index)
        cov_o = engine.target_covariances(int(plan.target_offsets[-1]))
        To, ito, flo, *_ = engine.refine_handle(h, plan.target_idx[sel], cfg.gicp)
        engine.upload_targets(plan.target_offsets, plan.target_points, cfg.gicp, None)
        cov_g = engine.target_covariances(int(plan.target_offsets[-1]))
        Tg, itg, flg, *_ = engine.refine_handle(h, plan.target_idx[sel], cfg.gicp)
    finally:
        engine.lib.px_clouds_free(engine.ctx, h)
    sizes = np.diff(plan.target_offsets)
    big = np.repeat(sizes > cfg.gicp.k_covariance, sizes)
    assert np.array_equal(cov_o[big], cov_g[big])
    assert np.array_equal(ito, itg) and np.array_equal(flo, flg)
    assert np.array_equal(To, Tg)
    # and uploaded (generic) source clouds behave like device-rendered ones
    hu = engine._upload_clouds([c.points for c in clouds])
    try:
        Tu, itu, flu, *_ = engine.refine_handle(hu, plan.target_idx[sel], cfg.gicp)
    finally:
        engine.lib.px_clouds_free(engine.ctx, hu)
    assert np.array_equal(Tu, Tg) and np.array_equal(itu, itg)


@pytest.mark.parametrize("name", ["c1_box_3dof", "c3_clutter_3dof", "c4_mixed_6dof"])
def test_device_built_targets_equal_host_plan(engine, name):
    """search._build_targets on the device (capsule crops in 3-DoF, label sub-clouds in
    6-DoF): offsets, observed indices, points and covariances are bit-identical to the
    host plan (which tests/test_oracle_golden.py pins to the reference), and a search
    that starts from the target SPECS gives the same outputs as one from uploaded clouds."""
    from paper_2008_00326_b200.search import plan_search
    d, frame, models, cfg, plan = G.scene(name)
    spec = plan_search(frame, models, cfg, materialise_targets=False)
    assert spec.target_points is None and np.array_equal(spec.target_idx, plan.target_idx)
    engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
    engine.build_targets(spec)
    off, pts, oi = engine.download_targets()
    assert np.array_equal(off, plan.target_offsets)
    assert np.array_equal(oi.astype(np.int64), plan.target_obs_index)
    assert np.array_equal(pts, plan.target_points)
    cov_dev = engine.target_covariances(int(off[-1]))
    engine.upload_targets(plan.target_offsets, plan.target_points, cfg.gicp, plan.target_obs_index)
    cov_host = engine.target_covariances(int(off[-1]))
    sizes = np.diff(off)
    big = np.repeat(sizes > cfg.gicp.k_covariance, sizes)
    assert np.array_equal(cov_dev[big], cov_host[big])
    sel = np.arange(0, plan.n, max(1, plan.n // 400))
    a = engine.run_plan(frame, models, spec, sel)
    b = engine.run_plan(frame, models, plan, sel)
    assert np.array_equal(a.refined_cam, b.refined_cam) and np.array_equal(a.iterations, b.iterations)
    assert np.array_equal(a.j_o, b.j_o) and np.array_equal(a.j_r, b.j_r)


def test_device_targets_empty_and_tiny(engine):
    """Capsules that catch no point, or fewer than k_covariance points, are legal targets
    (registration.py:504-510: too_few_points keeps the candidate's pose)."""
    d, frame, models, cfg, plan = G.scene("c1_box_3dof")
    engine.upload_scene(frame, cfg.stride, plan.observed, plan.obs_labels)
    caps = np.array([[5.0, 5.0, 0.0, 0.1, 0.05],                  # far outside the scene
                     list(plan.target_capsules[0][:4]) + [0.004]])  # a few points at most
    spec = dataclasses.replace(plan, target_capsules=caps, target_points=None, target_offsets=None,
                               target_obs_index=None)
    engine.build_targets(spec)
    off, pts, oi = engine.download_targets()
    assert off[0] == 0 and off[1] == 0 and off[2] - off[1] <= cfg.gicp.k_covariance


def test_cli_estimate_bench_selftest(engine, tmp_path, capsys):
    """`estimate` on a dataset written by the reference (tests/golden/dataset_tiny) reproduces the
    reference's results.json (winner index, integer costs, provenance; pose <= 1e-4), `bench` emits
    the reference's figure keys, `selftest` passes (cli.py:192-265, 268-335)."""
    from pathlib import Path
    from paper_2008_00326_b200.cli import main
    ds = Path(__file__).resolve().parent / "golden" / "dataset_tiny"
    out = tmp_path / "out"
    rc = main(["estimate", "--scene", str(ds / "scene_0000"), "--models", str(ds / "models"), "--out", str(out),
               "--config", str(ds / "config.json"), "--trace"])
    assert rc == 0
    got = json.loads((out / "results.json").read_text())
    ref = json.loads((ds / "results_reference.json").read_text())
    assert got["proposals_evaluated"] == ref["proposals_evaluated"]
    for x, r in zip(got["objects"], ref["objects"]):
        assert (x["object_id"], x["proposal_index"], x["j_o"], x["j_r"], x["provenance"]) == \
               (r["object_id"], r["proposal_index"], r["j_o"], r["j_r"], r["provenance"])
        wt, wr = G.pose_delta(np.array(x["pose"]).reshape(3, 4), np.array(r["pose"]).reshape(3, 4))
        assert wt <= 1e-4 and wr <= 1e-4
    assert set(json.loads((out / "timings.json").read_text())) == {"total_millis", "stage_millis", "per_object_millis"}
    assert len((out / "trace.jsonl").read_text().splitlines()) == ref["proposals_evaluated"]
    fig = tmp_path / "fig.json"
    assert main(["bench", "--scene", str(ds / "scene_0000"), "--models", str(ds / "models"), "--config",
                 str(ds / "config.json"), "--repeat", "2", "--json-out", str(fig)]) == 0
    f = json.loads(fig.read_text())
    assert {"proposals", "proposals_per_sec", "total_seconds", "stage_millis", "workers", "rendered_points_max",
            "observed_points", "knn_full_relation_bytes", "knn_streamed_relation_bytes",
            "knn_last_relation_bytes"} == set(f) and f["proposals"] == ref["proposals_evaluated"]
    assert main(["selftest"]) == 0
    capsys.readouterr()


def _full_c3():
    """BASELINE configs[2] at the size bench.py measures: 58,320 candidates, GICP on."""
    import bench
    return bench.build_workload("c3", 1, 1, materialise_targets=False)


def test_full_size_determinism_chunking_and_sharding(engine):
    """Size-independent properties at the benchmark's full size (no oracle run needed):
    * re-running the same search gives bit-identical outputs (no atomics-order or timing dependence),
    * forcing the scratch chunking (px_ctx_set_scratch_budget) changes nothing -- candidates are independent,
    * the per-object argmin of the union of 4 rank shards (dist.shard_index + packed-key MIN, the
      multi-GPU path) equals the unsharded one, and every shard's per-candidate outputs equal the
      unsharded rows -- the device analogue of the reference's worker-count determinism test
      (tests/test_search.py:100-106)."""
    from paper_2008_00326_b200 import dist as pxd
    frame, models, cfg, plan = _full_c3()
    assert plan.n == 58320
    engine.prepare_plan(frame, models, plan)
    sc = engine.search_cfg(plan)
    n = engine.search_upload(plan)
    engine.search_run(sc)
    a = engine.search_download(n)
    engine.search_run(sc)
    b = engine.search_download(n)
    for f in ("refined_cam", "reg_T", "j_o", "j_r", "iterations", "flags", "n_rendered"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert a.best_keys == b.best_keys
    # chunked: 1 GiB of scratch forces several chunks at this size
    N_ = engine.lib
    assert N_.px_ctx_set_scratch_budget(engine.ctx, 1 << 30) == 0
    try:
        engine.search_run(sc)
        c = engine.search_download(n)
    finally:
        N_.px_ctx_set_scratch_budget(engine.ctx, 8 << 30)
    for f in ("refined_cam", "j_o", "j_r", "iterations", "flags"):
        assert np.array_equal(getattr(a, f), getattr(c, f)), f
    assert a.best_keys == c.best_keys
    # sharded: 4 ranks' worth of work on this one GPU
    world = 4
    keys = []
    for r in range(world):
        idx = pxd.shard_index(plan, r, world)
        m = engine.search_upload(plan, idx)
        engine.search_run(sc)
        s = engine.search_download(m)
        assert np.array_equal(s.refined_cam, a.refined_cam[idx]) and np.array_equal(s.j_o, a.j_o[idx]) \
            and np.array_equal(s.j_r, a.j_r[idx])
        keys.append(pxd.keys_from_device(plan, s.best_keys))
    merged = np.minimum.reduce(keys)
    assert np.array_equal(merged, pxd.keys_from_device(plan, a.best_keys))
    # and the winner decoded from the merged keys is the host argmin over all candidates
    res = assemble_result(plan, a, 0.0)
    for slot, oid in enumerate(plan.active):
        e = res.estimate_for(oid)
        assert (int(merged[slot]) >> 32, int(merged[slot]) & 0xffffffff) == (e.cost.total, e.proposal_index)


def _adds(mesh_pts, pose_a, pose_b):
    """ADD-S: mean distance from every model point under pose_a to the closest model point under pose_b."""
    a = mesh_pts @ pose_a.rotation.T + pose_a.translation
    b = mesh_pts @ pose_b.rotation.T + pose_b.translation
    d = ((a[:, None, :] - b[None, :, :]) ** 2).sum(-1)
    return float(np.sqrt(d.min(axis=1)).mean())


def test_reference_search_tests_through_public_api(engine):
    """The reference's own search-level tests (pkg/tests/test_search.py:151-245) replayed on the
    committed two-cylinder scene through estimate_poses: recovery within 1 cm with colour on,
    refinement never worse than no refinement, small 6-DoF search with the in-plane axis collapsed
    for symmetric models, failures reported per object, uniform subsampling by max_proposals, and
    timing kept out of the result JSON."""
    from paper_2008_00326_b200 import SearchConfig, estimate_poses, timings_to_json
    d, frame, models, cfg, plan = G.scene("c2_twocyl_color1")
    gt = {s.object_id: s.pose for s in frame.ground_truth}
    ws = (-0.32, 0.32, -0.32, 0.32)
    # :151-161 colour on separates the same-shape objects
    res = estimate_poses(frame, models, SearchConfig(mode="3dof", workspace=ws, dt=0.1))
    for e in res.estimates:
        assert not e.failed and _adds(models[e.object_id].mesh.vertices, gt[e.object_id], e.pose) < 0.01
    # :183-192 refinement never increases the winning cost
    off = estimate_poses(frame, models, SearchConfig(mode="3dof", workspace=ws, dt=0.1, refine=False))
    for on_e, off_e in zip(res.estimates, off.estimates):
        assert on_e.cost.total <= off_e.cost.total
    # :195-209 6-DoF, yaw-symmetric models collapse n_inplane
    r1 = estimate_poses(frame, models, SearchConfig(mode="6dof", viewpoints=16, n_inplane=1))
    r16 = estimate_poses(frame, models, SearchConfig(mode="6dof", viewpoints=16, n_inplane=16))
    assert r16.proposals_evaluated == r1.proposals_evaluated
    for e in r1.estimates:
        assert not e.failed and _adds(models[e.object_id].mesh.vertices, gt[e.object_id], e.pose) < 0.02
    # :212-220 failures are per object
    one = estimate_poses(frame, {1: models[1]}, SearchConfig(mode="3dof", workspace=ws, dt=0.1))
    by_id = {e.object_id: e for e in one.estimates}
    assert by_id[2].failed and by_id[2].failure == "unknown_object" and not by_id[1].failed
    # :223-233 timing stays out of the result JSON
    assert "millis" not in result_to_json(res)
    t = json.loads(timings_to_json(res))
    assert t["total_millis"] > 0 and set(t["stage_millis"]) == {"render", "refine", "rerender", "cost"}
    # :236-242 uniform subsample
    sub = estimate_poses(frame, models, SearchConfig(mode="3dof", workspace=ws, dt=0.05, max_proposals=20))
    assert sub.proposals_evaluated == 20


def test_randomised_units_against_oracle(engine):
    """Seeded random sweeps, device vs the pinned oracle, everything bit-exact: kNN (random and
    integer-lattice clouds with many exact ties, k up to 8), rendered cost (colour on/off, clouds
    from 1 to 200 points), covariances (flat, noisy and duplicate-heavy clouds) and single-view
    z-buffers of random meshes -- the randomised halves of the reference's unit tests
    (tests/test_neighbors.py:54-84, test_cost.py:102-125, test_registration.py:59-78,
    test_raster.py:68-80)."""
    rng = np.random.default_rng(20260117)
    for trial in range(40):
        nq, nt, k = int(rng.integers(1, 70)), int(rng.integers(1, 90)), int(rng.integers(1, 9))
        if trial % 2:
            q, t = rng.integers(-3, 4, (nq, 3)).astype(float), rng.integers(-3, 4, (nt, 3)).astype(float)
        else:
            q, t = rng.normal(size=(nq, 3)), rng.normal(size=(nt, 3))
        gi, gd = engine.knn(q, t, k)
        oi, od = O.knn(q, t, k)
        assert np.array_equal(gi, oi) and np.array_equal(gd, od), trial
    for trial in range(40):
        nr, no = int(rng.integers(1, 200)), int(rng.integers(1, 200))
        rp, op = rng.normal(scale=0.03, size=(nr, 3)), rng.normal(scale=0.03, size=(no, 3))
        rl, ol = rng.uniform(0, 100, (nr, 3)) * [1, 0.6, 0.6], rng.uniform(0, 100, (no, 3)) * [1, 0.6, 0.6]
        delta, tau, uc = float(rng.uniform(0.005, 0.03)), float(rng.uniform(5, 40)), bool(trial % 2)
        z2 = lambda n: np.zeros((n, 2), dtype=np.int32)
        jr, ex = cost.rendered_cost(LabeledCloud(rp, rl, z2(nr)), LabeledCloud(op, ol, z2(no)), CostParams(delta, tau, uc))
        ojr, oex = O.rendered_cost(rp, rl, op, ol, delta, tau, uc)
        assert jr == ojr and np.array_equal(ex, oex.astype(bool)), trial
    for trial in range(12):
        n = int(rng.integers(25, 400))
        pts = rng.normal(size=(n, 3)) * [0.1, 0.1, 0.002 if trial % 3 == 0 else 0.05]
        if trial % 4 == 3:
            pts[n // 2:] = pts[: n - n // 2]  # exact duplicates: zero distances and ties
        assert np.array_equal(engine.covariances(pts, 20, 1e-3), O.covariances(pts)), trial
    for trial in range(6):
        nv = int(rng.integers(4, 40))
        v = rng.uniform(-0.06, 0.06, (nv, 3))
        tris = rng.integers(0, nv, (int(rng.integers(1, 120)), 3)).astype(np.int32)  # may contain degenerate faces
        mesh = TriangleMesh(v, rng.uniform(0, 1, (nv, 3)), tris)
        pose = np.hstack([np.eye(3), [[0.0], [0.0], [0.35]]])
        z, cb, valid, owner = engine.rasterize_mesh(mesh, RigidTransform.from_matrix3x4(pose), K64)
        oz, oc, ov, oo = O.rasterize(O.OracleModel(1, mesh), pose, K64)
        assert np.array_equal(valid, ov) and np.array_equal(z, oz) and np.array_equal(owner, oo), trial
        assert np.array_equal(cb[valid], oc[ov])


def test_full_size_sample_against_oracle(engine):
    """At the benchmark's own density (dt 0.025, 58,320 candidates): ~3,000 candidates in whole grid
    cells spread over the workspace, device (targets cropped on the device) vs the pinned oracle
    (host-built targets).  Poses within 1e-4 m / 1e-4 rad and equal iteration counts for >= 99 %,
    integer costs equal wherever the poses agree, first-render point counts equal everywhere."""
    import bench
    frame, models, cfg, spec = _full_c3()
    _, _, _, host = bench.build_workload("c3", 1, 1, materialise_targets=True)
    pick = bench.sample_groups(host, np.arange(host.n), 3000)
    dev = engine.run_plan(frame, models, spec, pick)
    cpu = O.run_plan(frame, models, host, index=pick)
    assert np.array_equal(dev.n_first, cpu.n_first)
    dt, dr = G.pose_delta(dev.refined_cam, cpu.refined_cam)
    close = (dt <= 1e-4) & (dr <= 1e-4)
    same = (dev.j_o == cpu.j_o) & (dev.j_r == cpu.j_r)
    print(f"full-size sample: n={pick.size} pose-agree={close.mean():.4f} iters-equal={(dev.iterations == cpu.iterations).mean():.4f} "
          f"costs-equal={same.mean():.4f}")
    # pinned to the measured value: all 3,008 sampled candidates agree (poses, iteration counts, integer costs)
    assert close.all() and (dev.iterations == cpu.iterations).all() and same.all()


def test_full_size_6dof_sample_against_oracle(engine):
    """BASELINE configs[3] at the size bench.py --workload c4 measures (249,738 mask-constrained 6-DoF
    candidates): every 83rd candidate, device (label targets built on the device) vs the pinned oracle."""
    import bench
    frame, models, cfg, spec = bench.build_workload("c4", 1, 1, materialise_targets=False)
    _, _, _, host = bench.build_workload("c4", 1, 1, materialise_targets=True)
    assert spec.n == 249738
    pick = np.arange(0, spec.n, 83)
    dev = engine.run_plan(frame, models, spec, pick)
    cpu = O.run_plan(frame, models, host, index=pick)
    assert np.array_equal(dev.n_first, cpu.n_first)
    dt, dr = G.pose_delta(dev.refined_cam, cpu.refined_cam)
    close = (dt <= 1e-4) & (dr <= 1e-4)
    same = (dev.j_o == cpu.j_o) & (dev.j_r == cpu.j_r)
    print(f"full-size 6-DoF sample: n={pick.size} pose-agree={close.mean():.4f} "
          f"iters-equal={(dev.iterations == cpu.iterations).mean():.4f} costs-equal={same.mean():.4f}")
    assert close.all() and (dev.iterations == cpu.iterations).all() and same.all()  # measured: 3,009 of 3,009
