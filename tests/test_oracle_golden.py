"""Pin the CPU oracle (oracle/px_oracle.c) and the host-side planning code to
outputs of the reference itself (tests/golden/, made by oracle/make_golden.py).

CPU only.  Bit-exact for everything the reference computes in plain float64
without LAPACK / SIMD libm (visibility, clouds, kNN, covariances, the GICP
normal equations, integer costs, argmin); stated tolerances elsewhere.
"""

import json

import numpy as np
import pytest

import golden_io as G
from oracle import oracle as O
from paper_2008_00326_b200 import GicpConfig, colorspace
from paper_2008_00326_b200.search import assemble_result, result_to_json

U = G.load("units")


# ---- colour -------------------------------------------------------------------

def test_ciede2000_published_pairs():
    # reference tests/test_colorspace.py:39-44 -- 34 published pairs to 1e-4
    worst = 0.0
    for row in U["ciede_pairs"]:
        worst = max(worst, abs(O.ciede2000(row[0:3], row[3:6]) - row[6]))
        assert abs(colorspace.ciede2000(row[0:3], row[3:6]) - row[6]) < 1e-4
    assert worst < 1e-4


def test_srgb_lab_spot_vector():
    v = U["srgb_lab_vector"]
    assert np.abs(O.srgb_to_lab(v[:3])[0] - v[3:]).max() < 0.01
    assert np.abs(colorspace.srgb_to_lab(v[:3]) - v[3:]).max() < 0.01


def test_lab_and_de_match_reference_outputs():
    assert np.abs(O.srgb_to_lab(U["lab_rgb"]) - U["lab_out"]).max() < 1e-9
    assert np.array_equal(colorspace.srgb_to_lab(U["lab_rgb"]), U["lab_out"])  # same numpy path, same bits
    de = np.array([O.ciede2000(a, b) for a, b in zip(U["de_a"], U["de_b"])])
    assert np.abs(de - U["de_out"]).max() < 1e-9
    assert np.abs(colorspace.ciede2000(U["de_a"], U["de_b"]) - U["de_out"]).max() == 0.0


# ---- raster ---------------------------------------------------------------------

class _Mesh:
    def __init__(self, v, c, t):
        self.vertices, self.vertex_colors, self.triangles = v, c, t


@pytest.mark.parametrize("t", range(6))
def test_raster_kernel_bit_exact(t):
    from paper_2008_00326_b200 import CameraIntrinsics, RigidTransform
    k = CameraIntrinsics(500.0, 500.0, 32.0, 32.0, 64, 64, RigidTransform.identity())
    m = O.OracleModel(1, _Mesh(U[f"ras{t}_verts"], U[f"ras{t}_cols"], U[f"ras{t}_tris"]))
    m.col[:] = U[f"ras{t}_cols"]  # the fixture colours are already linear
    z, c, v, owner = O.rasterize(m, np.hstack([np.eye(3), np.zeros((3, 1))]), k)
    assert np.array_equal(v, U[f"ras{t}_valid"])
    assert np.array_equal(z, U[f"ras{t}_z"])
    assert np.array_equal(c[v], U[f"ras{t}_c"][v])
    assert (owner[v] >= 0).all() and (owner[~v] == -1).all()


# ---- kNN / cost -------------------------------------------------------------------

@pytest.mark.parametrize("t", range(4))
def test_knn_exact(t):
    idx, d2 = O.knn(U[f"knn{t}_q"], U[f"knn{t}_t"], int(U[f"knn{t}_k"]))
    assert np.array_equal(idx, U[f"knn{t}_idx"])
    assert np.array_equal(d2, U[f"knn{t}_d2"])


def test_cost_counts_exact():
    for i in range(int(U["cost_n"])):
        delta, tau, uc = U[f"cost{i}_par"]
        jr, ex = O.rendered_cost(U[f"cost{i}_rp"], U[f"cost{i}_rl"], U[f"cost{i}_op"], U[f"cost{i}_ol"],
                                 delta, tau, bool(uc))
        jo = int(np.count_nonzero(U[f"cost{i}_sel"] & ~ex))
        assert (jo, jr) == tuple(U[f"cost{i}_out"]), i
        assert np.array_equal(ex, U[f"cost{i}_expl"])


# ---- registration -------------------------------------------------------------------

@pytest.mark.parametrize("t", range(4))
def test_covariances_bit_exact(t):
    assert np.array_equal(O.covariances(U[f"gicp{t}_src"]), U[f"gicp{t}_ca"])
    assert np.array_equal(O.covariances(U[f"gicp{t}_tgt"]), U[f"gicp{t}_cb"])


@pytest.mark.parametrize("t", range(4))
def test_gicp_linearize_bit_exact(t):
    gate2 = GicpConfig().max_correspondence_distance ** 2
    f0, nc, h, g, corr, w = O.gicp_linearize(U[f"gicp{t}_src"], U[f"gicp{t}_tgt"], U[f"gicp{t}_ca"],
                                             U[f"gicp{t}_cb"], np.eye(3), np.zeros(3), gate2)
    assert nc == int(U[f"gicp{t}_ncorr"]) and f0 == float(U[f"gicp{t}_f0"])
    assert np.array_equal(corr, U[f"gicp{t}_corr"])
    assert np.array_equal(h, U[f"gicp{t}_h"]) and np.array_equal(g, U[f"gicp{t}_g"])
    on = corr >= 0
    assert np.array_equal(w[on], U[f"gicp{t}_w"][on])


@pytest.mark.parametrize("t", range(4))
def test_gicp_align_matches_reference(t):
    cfg = GicpConfig()
    T, iters, conv, fail, trace, _ = O.gicp_align(U[f"gicp{t}_src"], U[f"gicp{t}_tgt"], U[f"gicp{t}_ca"],
                                                  U[f"gicp{t}_cb"], np.hstack([np.eye(3), np.zeros((3, 1))]), cfg)
    # well-conditioned recovery problems: LAPACK-vs-LU solve differences stay at rounding level
    assert iters == int(U[f"gicp{t}_iters"]) and conv == bool(U[f"gicp{t}_conv"]) and fail is None
    dt, dr = G.pose_delta(T, U[f"gicp{t}_T"])
    assert dt < 1e-9 and dr < 1e-7
    ref_tr = U[f"gicp{t}_trace"]
    assert trace.shape == ref_tr.shape and trace[0, 0] == ref_tr[0, 0]
    assert np.allclose(trace, ref_tr, rtol=1e-6, atol=1e-12)
    resid = O.rms_residual(U[f"gicp{t}_src"], U[f"gicp{t}_tgt"], T, cfg.max_correspondence_distance)
    assert abs(resid - float(U[f"gicp{t}_resid"])) < 1e-9


# ---- whole-path fixtures ---------------------------------------------------------------

SEARCH = ["c1_box_3dof", "c2_twocyl_color1", "c2_twocyl_color0", "c3_clutter_3dof", "c3n_clutter_noisy", "c4_mixed_6dof"]


@pytest.mark.parametrize("name", SEARCH)
def test_plan_matches_reference(name):
    """Host planning: candidate poses, observed cloud and GICP targets carry the
    reference's bits (search.py:232-265, 393-426)."""
    d, frame, models, cfg, plan = G.scene(name)
    assert np.array_equal(plan.flat_oid, d["flat_oid"]) and np.array_equal(plan.flat_local, d["flat_local"])
    assert np.array_equal(plan.cam_poses, d["cam_poses"])
    assert len(plan.observed) == int(d["n_obs"])
    assert np.array_equal(G.cloud_digest(plan.observed.points, plan.observed.source_pixel), d["obs_digest"])
    assert np.array_equal(plan.observed.lab_colors[::257], d["obs_lab_sample"])
    if cfg.refine:
        assert np.array_equal(plan.target_idx, d["target_idx"])
        sizes = np.diff(plan.target_offsets)
        assert np.array_equal(sizes, d["target_sizes"])
        import hashlib
        for t in range(len(sizes)):
            seg = plan.target_points[plan.target_offsets[t]:plan.target_offsets[t + 1]]
            dig = np.frombuffer(hashlib.sha256(np.ascontiguousarray(seg).tobytes()).digest(), dtype=np.uint8)
            assert np.array_equal(dig, d["target_digest"][t])


@pytest.fixture(scope="module")
def oracle_runs():
    cache = {}

    def run(name):
        if name not in cache:
            d, frame, models, cfg, plan = G.scene(name)
            cache[name] = O.run_plan(frame, models, plan)
        return cache[name]
    return run


@pytest.mark.parametrize("name", SEARCH)
def test_oracle_first_render_bit_exact(name):
    """Visibility / ownership / cloud order: digest of (points, source_pixel) of
    every candidate's first render equals the reference's; kept clouds equal
    element-wise, Lab to 1e-9."""
    d, frame, models, cfg, plan = G.scene(name)
    sc = O.OracleScene(frame, cfg.stride, plan.observed, plan.obs_labels)
    om = {oid: O.OracleModel(oid, models[oid].mesh, models[oid].inscribed_cylinder) for oid in plan.active}
    step = max(1, plan.n // 400)
    for j in sorted(set(range(0, plan.n, step)) | set(int(x) for x in d["keep"])):
        pts, lab, src = O.render_one(sc, om[int(plan.flat_oid[j])], plan.cam_poses[j], cfg.occluder_marking, cfg.delta)
        assert pts.shape[0] == d["n0"][j]
        assert np.array_equal(G.cloud_digest(pts, src), d["dig0"][j]), j
        if f"c0_{j}_pts" in d:
            assert np.array_equal(pts, d[f"c0_{j}_pts"]) and np.array_equal(src, d[f"c0_{j}_src"])
            if pts.shape[0]:
                assert np.abs(lab - d[f"c0_{j}_lab"]).max() < 1e-9


@pytest.mark.parametrize("name", SEARCH)
def test_oracle_search_matches_reference(name, oracle_runs):
    """End to end (SURVEY.md 7.3 H4 contract): integer costs of every candidate,
    per-object argmin and winner pose; refined-pose agreement is reported as a
    fraction because GICP is chaotic for a minority of candidates under
    LAPACK-level rounding differences."""
    d, frame, models, cfg, plan = G.scene(name)
    out = oracle_runs(name)
    assert np.array_equal(out.n_first, d["n0"])
    dt, dr = G.pose_delta(out.refined_cam, d["refined"])
    close = (dt <= 1e-4) & (dr <= 1e-4)
    same_cost = (out.j_o == d["j_o"]) & (out.j_r == d["j_r"])
    print(f"{name}: poses within 1e-4 m/rad {close.mean():.4f}; integer costs equal {same_cost.mean():.4f}")
    if cfg.refine:
        assert np.array_equal(out.iterations == 0, d["reg_iters"] == 0)
        # pinned to what is measured: every candidate except the one chaotic C3 candidate (index 1131: the reference
        # stops after 16 iterations, the restated LU / libm arithmetic runs 30); the reference's own self-agreement
        # under 4-ulp input noise is only ~0.81, so this is as tight as the domain allows
        known = {"c3_clutter_3dof": {1131}}.get(name, set())
        assert set(np.nonzero(~close)[0].tolist()) <= known
        assert set(np.nonzero(~same_cost)[0].tolist()) <= known
    else:
        assert close.all() and same_cost.all()
    ref = json.loads(str(d["result_json"]))
    mine = json.loads(result_to_json(assemble_result(plan, out, 0.0)))
    assert mine["proposals_evaluated"] == ref["proposals_evaluated"]
    for a, b in zip(ref["objects"], mine["objects"]):
        assert a["object_id"] == b["object_id"] and a["failed"] == b["failed"]
        if a["failed"]:
            continue
        assert (a["proposal_index"], a["j_o"], a["j_r"], a["provenance"]) == \
               (b["proposal_index"], b["j_o"], b["j_r"], b["provenance"])
        pa, pb = np.array(a["pose"]).reshape(3, 4), np.array(b["pose"]).reshape(3, 4)
        wt, wr = G.pose_delta(pa, pb)
        assert wt <= 1e-4 and wr <= 1e-4


def test_gicp_weights_are_not_bit_symmetric_at_a_general_pose():
    """VERDICT r1 #4 asked whether W = (Cb + R Ca R^T)^-1 could be stored as six entries.  It cannot: the reference
    forms (R Ca) R^T with left-to-right sums (registration.py:262-283), which associates differently across the
    diagonal, so W[i][j] != W[j][i] in the last bits for most matches once R is not the identity -- and the objective
    (registration.py:387-407) reads all nine.  At R = I the matrices are bit-symmetric, which is why the golden
    vectors alone would suggest otherwise."""
    rng = np.random.default_rng(1)
    src, tgt, ca, cb = (U[f"gicp1_{k}"] for k in ("src", "tgt", "ca", "cb"))
    w0 = U["gicp1_w"][U["gicp1_corr"] >= 0]
    assert np.array_equal(w0, np.transpose(w0, (0, 2, 1)))
    ax = rng.normal(size=3)
    ax /= np.linalg.norm(ax)
    K = np.array([[0, -ax[2], ax[1]], [ax[2], 0, -ax[0]], [-ax[1], ax[0], 0]])
    R = np.eye(3) + np.sin(0.2) * K + (1 - np.cos(0.2)) * K @ K
    f0, nc, h, g, corr, w = O.gicp_linearize(src, tgt, ca, cb, R, np.array([0.003, -0.002, 0.001]), 0.05 ** 2)
    w = w[corr >= 0]
    asym = (w != np.transpose(w, (0, 2, 1))).any(axis=(1, 2))
    assert nc > 50 and asym.mean() > 0.5
    assert np.abs(w - np.transpose(w, (0, 2, 1))).max() < 1e-9 * np.abs(w).max()  # symmetric as a matrix, not as bits


def test_oracle_at_benchmark_density_against_the_reference():
    """9,680 candidates of the C3 scene at the benchmark's own grid density (dt 0.025, no subsampling), the reference's
    per-candidate outputs (tests/golden/c3d_dense_reference.npz): first / final render counts and GICP iteration
    counts; integer costs and refined poses (1e-4 m / 1e-4 rad) for every candidate
    but the chaotic few named below; per-object winners."""
    dd, frame, models, cfg, plan = G.dense_scene()
    out = O.run_plan(frame, models, plan, n_threads=8)
    assert np.array_equal(out.n_first, dd["n0"])
    dt, dr = G.pose_delta(out.refined_cam, dd["refined"])
    close = (dt <= 1e-4) & (dr <= 1e-4)
    same = (out.j_o == dd["j_o"]) & (out.j_r == dd["j_r"])
    bad = sorted(set(np.nonzero(~close)[0].tolist()) | set(np.nonzero(~same)[0].tolist()))
    print(f"dense: n={plan.n} poses within tol {close.mean():.5f}, costs equal {same.mean():.5f}, divergent {bad}")
    assert set(bad) <= DENSE_CHAOTIC_ORACLE
    ok = np.ones(plan.n, bool)
    ok[sorted(DENSE_CHAOTIC_ORACLE)] = False
    assert np.array_equal(out.iterations[ok], dd["reg_iters"][ok]) and np.array_equal(out.n_rendered[ok], dd["n1"][ok])
    ref = json.loads(str(dd["result_json"]))
    mine = json.loads(result_to_json(assemble_result(plan, out, 0.0)))
    for a, b in zip(ref["objects"], mine["objects"]):
        assert (a["proposal_index"], a["j_o"], a["j_r"], a["provenance"]) == (b["proposal_index"], b["j_o"], b["j_r"], b["provenance"])


# candidates on which the reference (LAPACK / libm) and the restated arithmetic part ways: 5 of 9,680
DENSE_CHAOTIC_ORACLE = {1813, 1821, 9555, 9563, 9566}


def test_oracle_on_the_benchmark_step_against_the_reference():
    """The C port against the reference's outputs on the WHOLE benchmark step (58,320 candidates, tests/golden/
    c3f_full_reference.npz), here on every sixth grid cell (9,720 candidates; the GPU test covers all of them and finds the
    same divergent set): poses, costs and render counts agree except on the named chaotic candidates."""
    import bench
    dd, frame, models, cfg = G.full_scene()
    _, _, _, plan = bench.build_workload("c3", 1, 1, materialise_targets=True)
    assert plan.n == 58320
    per_cell = 16                                                   # yaws per grid cell
    cells = np.arange(plan.n // per_cell).reshape(-1)
    pick = (cells[::6, None] * per_cell + np.arange(per_cell)[None, :]).reshape(-1)
    out = O.run_plan(frame, models, plan, index=pick, n_threads=8)
    bad, iters = G.compare_with_full_reference(frame, dd, out, pick)
    print(f"benchmark step, every sixth cell: n={pick.size} divergent {sorted(bad)}")
    assert bad == G.FULL_CHAOTIC & set(pick.tolist())
    assert iters <= G.FULL_CHAOTIC | G.FULL_ITERS_ONLY


def test_oracle_on_the_6dof_workload_against_the_reference():
    """The C port against the reference's outputs on the whole 6-DoF workload (249,738 candidates, tests/golden/
    c4f_full_reference.npz), here on every 21st candidate (11,893; the GPU test covers all of them)."""
    import bench
    dd = G.load("c4f_full_reference")
    frame, models, cfg, plan = bench.build_workload("c4", 1, 1, materialise_targets=True)
    pick = np.arange(0, plan.n, 21)
    out = O.run_plan(frame, models, plan, index=pick, n_threads=8)
    bad, badpose, iters = G.compare_with_full_reference_6dof(dd, out, pick)
    here = set(pick.tolist())
    assert bad == G.FULL6_CHAOTIC & here and badpose <= G.FULL6_POSE and iters == G.FULL6_ITERS & here
