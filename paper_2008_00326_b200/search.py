"""Flat parallel pose search: the drop-in `estimate_poses` entry point.

Reference: pkg/src/rvpose/search.py:217-377.  The orchestration is split in
two so the per-candidate stages can run as batched device launches:

* `plan_search`  -- host, per scene: observed cloud, proposals, candidate
  camera poses (array-valued, reference bits), GICP targets.  No per-candidate
  Python objects.
* `Engine.run`   -- device (paper_2008_00326_b200.engine): render -> GICP ->
  re-render -> cost -> per-object argmin over the flat candidate list.

`estimate_poses` glues them and builds the reference's result types.  There
is no CPU implementation of the stages in this package: without the CUDA
library the call raises `DeviceError`.
"""

from __future__ import annotations

import json
import math
import time
from dataclasses import dataclass, field

import numpy as np

from .blas_probe import check_blas_orders
from .cost import CostBreakdown, CostParams
from .errors import ConfigError, EmptyBatch, NoValidDepth  # noqa: F401
from .geometry import RigidTransform, rotation_angle
from .model import LabeledCloud
from .proposals import (PoseProposalSet, compose_grid, compose_many, grid_proposals_3dof,
                        pose_proposals_6dof, rotation_proposals, translation_proposals)
from .raster import cloud_labels, frame_to_cloud
from .registration import GicpConfig


@dataclass(frozen=True)
class KnnConfig:
    """Accepted for signature compatibility; both strategies are exact and
    identical by contract (neighbors.py:32-43), the device path has one."""

    strategy: str = "streamed"
    k: int = 1

    def __post_init__(self):
        if self.strategy not in ("full", "streamed"):
            raise ValueError(f"unknown strategy {self.strategy!r}")
        if self.k < 1:
            raise ValueError("k must be >= 1")


@dataclass(frozen=True)
class SearchConfig:
    mode: str = "6dof"
    use_color: bool = True
    occluder_marking: bool = True
    knn_strategy: str = "streamed"
    stride: int = 2
    delta: float = 0.0075
    tau_c: float = 12.5
    refine: bool = True
    gicp: GicpConfig = field(default_factory=GicpConfig)
    workspace: tuple | None = None
    fixed_z: float = 0.0
    dt: float = 0.08
    dyaw: float = math.radians(22.5)
    viewpoints: int = 42
    n_inplane: int = 16
    z_step: float = 0.02
    workers: int = 1              # result-neutral; ignored on device
    chunk_size: int | None = None  # result-neutral; ignored on device
    trace_path: str | None = None
    max_proposals: int | None = None

    def __post_init__(self):
        if self.mode not in ("3dof", "6dof"):
            raise ConfigError(f"unknown mode {self.mode!r}")
        if self.knn_strategy not in ("full", "streamed"):
            raise ConfigError(f"unknown knn strategy {self.knn_strategy!r}")
        if self.stride < 1:
            raise ConfigError("stride must be >= 1")
        if self.mode == "3dof" and self.workspace is None:
            raise ConfigError("3dof mode requires workspace bounds")
        if self.workspace is not None:
            x0, x1, y0, y1 = self.workspace
            if x1 < x0 or y1 < y0:
                raise ConfigError("workspace bounds are inverted")
        if min(self.delta, self.tau_c, self.dt, self.dyaw, self.z_step) <= 0:
            raise ConfigError("scale parameters must be positive")
        if self.viewpoints < 1 or self.n_inplane < 1:
            raise ConfigError("proposal counts must be >= 1")
        if self.workers < 1:
            raise ConfigError("workers must be >= 1")

    @property
    def cost_params(self) -> CostParams:
        return CostParams(self.delta, self.tau_c, self.use_color)

    @property
    def knn_config(self) -> KnnConfig:
        return KnnConfig(self.knn_strategy, 1)

    def to_dict(self) -> dict:
        g = self.gicp
        return {
            "mode": self.mode, "use_color": self.use_color,
            "occluder_marking": self.occluder_marking, "knn_strategy": self.knn_strategy,
            "stride": self.stride, "delta": self.delta, "tau_c": self.tau_c,
            "refine": self.refine,
            "gicp": {"k_covariance": g.k_covariance, "epsilon": g.epsilon,
                     "max_iterations": g.max_iterations,
                     "translation_tolerance": g.translation_tolerance,
                     "rotation_tolerance": g.rotation_tolerance,
                     "max_correspondence_distance": g.max_correspondence_distance},
            "workspace": list(self.workspace) if self.workspace else None,
            "fixed_z": self.fixed_z, "dt": self.dt, "dyaw_degrees": math.degrees(self.dyaw),
            "viewpoints": self.viewpoints, "n_inplane": self.n_inplane,
            "z_step": self.z_step, "workers": self.workers,
        }

    _KEYS = frozenset({
        "mode", "use_color", "occluder_marking", "knn_strategy", "stride", "delta", "tau_c",
        "refine", "gicp", "workspace", "fixed_z", "dt", "dyaw_degrees", "viewpoints",
        "n_inplane", "z_step", "workers", "chunk_size", "trace_path", "max_proposals"})

    @staticmethod
    def from_dict(d: dict) -> "SearchConfig":
        extra = set(d) - SearchConfig._KEYS
        if extra:
            raise ConfigError(f"unknown config keys: {sorted(extra)}")
        kw = dict(d)
        if "dyaw_degrees" in kw:
            kw["dyaw"] = math.radians(kw.pop("dyaw_degrees"))
        if kw.get("workspace") is not None:
            kw["workspace"] = tuple(kw["workspace"])
        if "gicp" in kw:
            try:
                kw["gicp"] = GicpConfig(**kw["gicp"])
            except (TypeError, ValueError) as e:
                raise ConfigError(f"bad gicp config: {e}") from e
        try:
            return SearchConfig(**kw)
        except (TypeError, ValueError) as e:
            raise ConfigError(str(e)) from e


@dataclass(frozen=True)
class ObjectEstimate:
    object_id: int
    pose: RigidTransform | None
    cost: CostBreakdown | None
    provenance: tuple | None
    proposal_index: int | None
    refine_translation: float
    refine_rotation: float
    proposals_evaluated: int
    millis: float
    failed: bool = False
    failure: str | None = None


@dataclass(frozen=True)
class SearchResult:
    estimates: tuple
    stage_millis: dict
    total_millis: float
    proposals_evaluated: int
    max_rendered_points: int = 0
    observed_points: int = 0

    def estimate_for(self, object_id: int) -> ObjectEstimate:
        for e in self.estimates:
            if e.object_id == object_id:
                return e
        raise KeyError(object_id)


def select_best(costs) -> int:
    """Argmin over (total, index) (search.py:178-183)."""
    costs = list(costs)
    if not costs:
        raise EmptyBatch("no costs to select from")
    return min(range(len(costs)), key=lambda i: (costs[i].total, i))


# ---------------------------------------------------------------------------
# host-side plan


@dataclass
class SearchPlan:
    """Everything the per-candidate stages need, as flat arrays."""

    cfg: SearchConfig
    object_ids: list                 # order of the estimates
    failures: dict                   # oid -> failure string
    active: list                     # object ids with candidates, in order
    proposal_sets: dict              # oid -> PoseProposalSet
    observed: LabeledCloud
    obs_labels: np.ndarray           # (n_obs,) i32
    flat_oid: np.ndarray             # (N,) i32
    flat_local: np.ndarray           # (N,) i32  proposal index inside its object
    cam_poses: np.ndarray            # (N,3,4) f64 candidate model->camera
    target_offsets: np.ndarray | None = None  # (n_targets+1,) i64
    target_points: np.ndarray | None = None   # (sum,3) f64
    target_obs_index: np.ndarray | None = None  # (sum,) i64 index into observed
    target_idx: np.ndarray | None = None      # (N,) i32
    target_capsules: np.ndarray | None = None  # 3-DoF target specs (n_targets,5): x, y, z_lo, z_hi, radius
    target_labels: np.ndarray | None = None    # 6-DoF target specs (n_targets,) object ids
    c2w: np.ndarray | None = None    # (3,4)
    w2c: np.ndarray | None = None
    c2w_vec_order: int = 0           # 0: rotation C-contiguous, 1: transposed view
    w2c_vec_order: int = 1
    cam_to_world: RigidTransform | None = None  # the frame's own object (its array layout decides numpy's rounding order)
    # device-generated candidates (plan_lattice): per active object the outer x inner factors of its proposal set;
    # the flat arrays above stay None and the observed cloud is built on the device
    lattice: list | None = None      # [LatticeFactor]
    n_observed: int | None = None

    @property
    def n(self) -> int:
        if self.lattice is not None:
            return int(sum(f.n_outer * f.n_inner for f in self.lattice))
        return int(self.flat_oid.shape[0])

    def count_of(self, oid: int) -> int:
        """Candidates of one object (ObjectEstimate.proposals_evaluated, search.py:365)."""
        if self.lattice is not None:
            return int(sum(f.n_outer * f.n_inner for f in self.lattice if f.object_id == oid))
        return int(np.count_nonzero(self.flat_oid == oid))

    def provenance_of(self, oid: int, local: int) -> tuple:
        if self.lattice is not None:
            f = next(f for f in self.lattice if f.object_id == oid)
            return (int(local // f.n_inner), int(local % f.n_inner))
        return tuple(int(x) for x in self.proposal_sets[oid].provenance[local])

    def observed_count(self) -> int:
        return int(self.n_observed) if self.n_observed is not None else len(self.observed)

    def rank_in_object(self) -> np.ndarray:
        """Position of each candidate among its object's candidates: the index
        `select_best` ranks by (search.py:178-183, 346-360)."""
        cached = getattr(self, "_rank_cache", None)
        if cached is not None and cached.shape[0] == self.n:
            return cached
        rank = np.empty(self.n, dtype=np.int32)
        for oid in self.active:
            sel = np.nonzero(self.flat_oid == oid)[0]
            rank[sel] = np.arange(sel.size, dtype=np.int32)
        self._rank_cache = rank
        return rank


@dataclass
class LatticeFactor:
    """One object's proposal set as an outer x inner product (proposals.py:163-210): 3-DoF outer = grid cells
    (translations), inner = yaw spins (rotations); 6-DoF outer = rotations, inner = translations."""

    object_id: int
    n_outer: int
    n_inner: int
    rotations: np.ndarray      # (n_inner,3,3) in 3-DoF, (n_outer,3,3) in 6-DoF
    translations: np.ndarray   # (n_outer,3) in 3-DoF, (n_inner,3) in 6-DoF
    capsule: tuple = (0.0, 0.0, 0.0)  # 3-DoF GICP target capsule: z_lo, z_hi, radius (search.py:407-426)


def _capsule_mask(pw, x, y, z_lo, z_hi, radius):
    """search.py:205-214."""
    dx = pw[:, 0] - x
    dy = pw[:, 1] - y
    dz = np.maximum.reduce([z_lo - pw[:, 2], pw[:, 2] - z_hi, np.zeros(pw.shape[0])])
    return (dx * dx + dy * dy + dz * dz) <= radius * radius


def _proposals_for(oid, frame, model, cfg) -> PoseProposalSet:
    if cfg.mode == "3dof":
        return grid_proposals_3dof(cfg.workspace, cfg.dt, cfg.dyaw, cfg.fixed_z, oid,
                                   model.yaw_symmetric)
    det = next(d for d in frame.detections if d.object_id == oid)
    rot = rotation_proposals(cfg.viewpoints, 1 if model.yaw_symmetric else cfg.n_inplane)
    tr = translation_proposals(det, frame.depth, frame.labels, frame.intrinsics, cfg.z_step)
    return pose_proposals_6dof(oid, rot, tr)


def _vec_order(rotation: np.ndarray) -> int:
    return 0 if rotation.flags.c_contiguous else 1


def plan_search(frame, models: dict, cfg: SearchConfig, build_targets: bool = True,
                materialise_targets: bool = True) -> SearchPlan:
    """Host part of search.py:217-265 and :393-426.  With `materialise_targets`
    False only the target SPECS (capsule parameters / label ids) and the
    candidate -> target map are produced; the device crops the clouds itself
    (Engine.build_targets)."""
    check_blas_orders()  # once per process: the host BLAS must round like the device's baked-in orders (H2)
    k = frame.intrinsics
    cam_to_world = RigidTransform(k.camera_pose.rotation, k.camera_pose.translation)
    world_to_cam = cam_to_world.inverse()
    if frame.detections:
        object_ids = [d.object_id for d in frame.detections]
    else:
        object_ids = sorted(models)
    if cfg.mode == "6dof" and not frame.detections:
        raise ConfigError("6dof mode requires detections in the frame")

    observed = frame_to_cloud(frame, cfg.stride)
    obs_labels = cloud_labels(observed, frame.labels)

    failures, psets, cams = {}, {}, {}
    for oid in object_ids:
        if oid not in models:
            failures[oid] = "unknown_object"
            continue
        try:
            ps = _proposals_for(oid, frame, models[oid], cfg)
        except NoValidDepth:
            failures[oid] = "no_valid_depth"
            continue
        if len(ps) == 0:
            failures[oid] = "empty_proposal_set"
            continue
        psets[oid] = ps
        if cfg.mode == "3dof":
            r, t = compose_grid(world_to_cam, ps)
        else:
            r, t = ps.rotations, ps.translations
        cams[oid] = np.concatenate([r, t[:, :, None]], axis=2)

    active = [oid for oid in object_ids if oid in psets]
    flat_oid = np.concatenate([np.full(len(psets[o]), o, dtype=np.int32) for o in active]) \
        if active else np.zeros(0, np.int32)
    flat_local = np.concatenate([np.arange(len(psets[o]), dtype=np.int32) for o in active]) \
        if active else np.zeros(0, np.int32)
    cam_poses = np.concatenate([cams[o] for o in active]) if active else np.zeros((0, 3, 4))
    if cfg.max_proposals is not None and flat_oid.size > cfg.max_proposals:
        pick = np.unique(np.round(np.linspace(0, flat_oid.size - 1, cfg.max_proposals)).astype(int))
        flat_oid, flat_local, cam_poses = flat_oid[pick], flat_local[pick], cam_poses[pick]
        present = set(int(o) for o in np.unique(flat_oid))
        active = [o for o in active if o in present]

    plan = SearchPlan(cfg, object_ids, failures, active, psets, observed, obs_labels,
                      np.ascontiguousarray(flat_oid), np.ascontiguousarray(flat_local),
                      np.ascontiguousarray(cam_poses),
                      c2w=np.ascontiguousarray(cam_to_world.matrix3x4()),
                      w2c=np.ascontiguousarray(world_to_cam.matrix3x4()),
                      c2w_vec_order=_vec_order(cam_to_world.rotation),
                      w2c_vec_order=_vec_order(world_to_cam.rotation),
                      cam_to_world=cam_to_world)
    if cfg.refine and build_targets and plan.n:
        _plan_targets(plan, models, cam_to_world, materialise_targets)
    return plan


def plan_lattice(frame, models: dict, cfg: SearchConfig) -> SearchPlan | None:
    """The per-scene plan for device-side set-up (SURVEY 8(f) ranks 1 + 2): proposal FACTORS per object instead of
    per-candidate arrays -- the device forms every candidate's camera pose (px_search_upload_lattice) and builds
    the observed cloud from the frame (px_scene_upload_frame).  None when the configuration needs the flat host
    plan (`max_proposals` subsampling picks arbitrary candidates, search.py:259-265)."""
    if cfg.max_proposals is not None:
        return None
    check_blas_orders()
    k = frame.intrinsics
    cam_to_world = RigidTransform(k.camera_pose.rotation, k.camera_pose.translation)
    world_to_cam = cam_to_world.inverse()
    object_ids = [d.object_id for d in frame.detections] if frame.detections else sorted(models)
    if cfg.mode == "6dof" and not frame.detections:
        raise ConfigError("6dof mode requires detections in the frame")
    failures, factors = {}, []
    grid = None
    for oid in object_ids:
        if oid not in models:
            failures[oid] = "unknown_object"
            continue
        m = models[oid]
        if cfg.mode == "3dof":
            from .proposals import lattice_3dof
            if grid is None:
                grid = {}
            key = bool(m.yaw_symmetric)
            if key not in grid:
                grid[key] = lattice_3dof(cfg.workspace, cfg.dt, cfg.dyaw, cfg.fixed_z, key)
            cells, spins = grid[key]
            cyl = m.inscribed_cylinder
            cap = (cfg.fixed_z + cyl.z_min + 0.005, cfg.fixed_z + cyl.z_max, 1.5 * cyl.radius + cfg.dt)
            if cells.shape[0] == 0:
                failures[oid] = "empty_proposal_set"
                continue
            factors.append(LatticeFactor(oid, cells.shape[0], spins.shape[0], spins, cells, cap))
        else:
            try:
                det = next(d for d in frame.detections if d.object_id == oid)
                rot = rotation_proposals(cfg.viewpoints, 1 if m.yaw_symmetric else cfg.n_inplane)
                tr = translation_proposals(det, frame.depth, frame.labels, frame.intrinsics, cfg.z_step)
            except NoValidDepth:
                failures[oid] = "no_valid_depth"
                continue
            if len(rot) == 0 or len(tr) == 0:
                failures[oid] = "empty_proposal_set"
                continue
            factors.append(LatticeFactor(oid, len(rot), len(tr), rot.rotations, tr.translations))
    active = [f.object_id for f in factors]
    return SearchPlan(cfg, object_ids, failures, active, {}, None, None, None, None, None,
                      c2w=np.ascontiguousarray(cam_to_world.matrix3x4()),
                      w2c=np.ascontiguousarray(world_to_cam.matrix3x4()),
                      c2w_vec_order=_vec_order(cam_to_world.rotation),
                      w2c_vec_order=_vec_order(world_to_cam.rotation),
                      cam_to_world=cam_to_world, lattice=factors)


def _plan_targets(plan: SearchPlan, models, cam_to_world, materialise: bool = True) -> None:
    """GICP targets (search.py:393-426): the label sub-cloud per object in
    6-DoF; per (object, grid cell) a capsule crop of the observed cloud in
    3-DoF.  Slots are numbered by first appearance in the flat list."""
    cfg, obs = plan.cfg, plan.observed
    n_obs = len(obs)
    tidx = np.empty(plan.n, dtype=np.int32)
    if cfg.mode == "6dof":
        slot = {oid: s for s, oid in enumerate(plan.active)}
        for oid in plan.active:
            tidx[plan.flat_oid == oid] = slot[oid]
        plan.target_labels = np.asarray(plan.active, dtype=np.int32)
    else:
        caps = []
        for oid in plan.active:
            sel = np.nonzero(plan.flat_oid == oid)[0]
            ps = plan.proposal_sets[oid]
            loc = plan.flat_local[sel]
            cells = ps.provenance[loc, 0]
            uniq, first = np.unique(cells, return_index=True)
            order = np.argsort(first, kind="stable")
            cyl = models[oid].inscribed_cylinder
            z_lo, z_hi = cfg.fixed_z + cyl.z_min + 0.005, cfg.fixed_z + cyl.z_max
            radius = 1.5 * cyl.radius + cfg.dt
            lut = np.full(int(uniq.max()) + 1, -1, dtype=np.int32)
            lut[uniq[order]] = len(caps) + np.arange(order.size, dtype=np.int32)
            rows = loc[first[order]]
            block = np.empty((order.size, 5))
            block[:, 0], block[:, 1] = ps.translations[rows, 0], ps.translations[rows, 1]
            block[:, 2], block[:, 3], block[:, 4] = z_lo, z_hi, radius
            caps.extend(block)
            tidx[sel] = lut[cells]
        plan.target_capsules = np.ascontiguousarray(np.array(caps).reshape(-1, 5))
    plan.target_idx = tidx
    if not materialise:
        return
    if cfg.mode == "6dof":
        chunks = [np.nonzero(plan.obs_labels == oid)[0] for oid in plan.active]
    else:
        obs_world = cam_to_world.apply(obs.points) if n_obs else np.zeros((0, 3))
        chunks = [np.nonzero(_capsule_mask(obs_world, x, y, z_lo, z_hi, radius))[0]
                  for x, y, z_lo, z_hi, radius in plan.target_capsules]
    offs = np.zeros(len(chunks) + 1, dtype=np.int64)
    np.cumsum([c.size for c in chunks], out=offs[1:])
    index = np.concatenate(chunks) if chunks else np.zeros(0, np.int64)
    plan.target_offsets = offs
    plan.target_obs_index = index.astype(np.int64)
    plan.target_points = np.ascontiguousarray(obs.points[index]) if n_obs else np.zeros((0, 3))


# ---------------------------------------------------------------------------
# results


@dataclass
class StageOutputs:
    """Per-candidate outputs of the render / refine / cost stages."""

    refined_cam: np.ndarray   # (N,3,4)
    reg_T: np.ndarray         # (N,3,4) applied GICP correction (identity if none)
    j_o: np.ndarray           # (N,) i32
    j_r: np.ndarray           # (N,) i32
    iterations: np.ndarray | None = None
    flags: np.ndarray | None = None
    n_rendered: np.ndarray | None = None  # final render
    stage_millis: dict | None = None


def _winner_rows(plan: SearchPlan, out: StageOutputs, index=None) -> dict:
    """Per active object: (packed key, refined pose, applied correction, j_o, j_r) of the best
    candidate among `out`'s rows (rows = plan candidates `index`, all of them if None):
    argmin over (total, rank in object), search.py:178-183."""
    n = out.j_o.shape[0]
    index = np.arange(plan.n) if index is None else np.asarray(index)
    total = out.j_o.astype(np.int64) + out.j_r.astype(np.int64)
    key = (total << 32) | plan.rank_in_object()[index].astype(np.int64)
    oid = plan.flat_oid[index]
    rows = {}
    for o in plan.active:
        sel = np.nonzero(oid == o)[0]
        if sel.size:
            r = int(sel[np.argmin(key[sel])])
            rows[o] = (int(key[r]), out.refined_cam[r], out.reg_T[r], int(out.j_o[r]), int(out.j_r[r]))
    assert n == index.shape[0]
    return rows


def _assemble(plan: SearchPlan, winners: dict, stage_millis: dict, t_start: float, max_pts: int) -> SearchResult:
    """Result records from the per-object winners (search.py:346-377)."""
    per_stage_total = sum(stage_millis.values())
    # compose with the frame's own transform object: a transposed-view rotation rounds differently in numpy
    # than a contiguous copy would (search.py:363 uses k.camera_pose as it is)
    c2w = plan.cam_to_world if plan.cam_to_world is not None else RigidTransform.from_matrix3x4(plan.c2w)
    estimates = []
    for oid in plan.object_ids:
        if oid in plan.failures or oid not in plan.active or oid not in winners:
            estimates.append(ObjectEstimate(oid, None, None, None, None, 0.0, 0.0, 0, 0.0,
                                            failed=True,
                                            failure=plan.failures.get(oid, "empty_proposal_set")))
            continue
        key, refined, reg_T, j_o, j_r = winners[oid]
        best_local = key & 0xFFFFFFFF
        n_obj = plan.count_of(oid)
        world = c2w.compose(RigidTransform.from_matrix3x4(refined))
        delta = RigidTransform.from_matrix3x4(reg_T)
        share = per_stage_total * (n_obj / max(1, plan.n))
        estimates.append(ObjectEstimate(
            oid, world, CostBreakdown(j_o=j_o, j_r=j_r),
            plan.provenance_of(oid, best_local), best_local,
            float(np.linalg.norm(delta.translation)), rotation_angle(delta.rotation),
            n_obj, share))
    total_millis = (time.perf_counter() - t_start) * 1e3
    return SearchResult(tuple(estimates), stage_millis, total_millis, plan.n, max_pts, plan.observed_count())


def assemble_result(plan: SearchPlan, out: StageOutputs, t_start: float) -> SearchResult:
    """Per-object argmin and result records (search.py:346-377)."""
    cfg = plan.cfg
    stage_millis = {"render": 0.0, "refine": 0.0, "rerender": 0.0, "cost": 0.0}
    if out.stage_millis:
        stage_millis.update(out.stage_millis)
    total = out.j_o.astype(np.int64) + out.j_r.astype(np.int64)
    if cfg.trace_path:
        with open(cfg.trace_path, "w") as f:
            for j in range(plan.n):
                f.write(json.dumps({
                    "object_id": int(plan.flat_oid[j]), "proposal_index": int(plan.flat_local[j]),
                    "j_o": int(out.j_o[j]), "j_r": int(out.j_r[j]), "total": int(total[j]),
                }, sort_keys=True) + "\n")
    max_pts = int(out.n_rendered.max()) if out.n_rendered is not None and out.n_rendered.size else 0
    return _assemble(plan, _winner_rows(plan, out), stage_millis, t_start, max_pts)


def estimate_poses_distributed(frame, models: dict, cfg: SearchConfig, runner=None) -> SearchResult:
    """`estimate_poses` across the ranks of an initialised torch.distributed group (one
    process per GPU): every rank plans the scene, scores its shard of the candidates
    (dist.shard_index), and the ranks agree on the per-object winner with ONE
    all_reduce(MIN) of the packed (cost, pose-id) keys; the owning rank's refined pose
    travels in a second tiny all_reduce(SUM).  Every rank returns the same SearchResult,
    identical to the single-process one (the reference's worker-count invariance,
    tests/test_search.py:100-106).  `runner(frame, models, plan, index) -> StageOutputs`
    defaults to the device engine; the CPU tests of the host logic inject their own."""
    import torch
    import torch.distributed as dist

    from . import dist as pxd

    if cfg.trace_path:
        raise ConfigError("trace_path is not supported under torch.distributed (per-candidate rows live on their rank)")
    t_start = time.perf_counter()
    rank, world = dist.get_rank(), dist.get_world_size()
    device_run = runner is None
    if device_run:
        from .engine import default_engine
        runner = default_engine().run_plan
    plan = plan_search(frame, models, cfg, materialise_targets=not device_run)
    stage_millis = {"render": 0.0, "refine": 0.0, "rerender": 0.0, "cost": 0.0}
    if plan.n == 0:
        return _assemble(plan, {}, stage_millis, t_start, 0)
    idx = pxd.shard_index(plan, rank, world)
    if device_run and dist.get_backend() == "nccl":
        # the collective runs on the device: libpx's own NCCL communicator reduces the packed keys and
        # delivers the winners' records to every rank (px_search_reduce); nothing per-candidate leaves the GPU
        eng = default_engine()
        if eng.comm_world() != world:
            eng.comm_init_torch()
        lat = plan_lattice(frame, models, cfg)
        if lat is not None and lat.n:
            plan = lat
            winners, stage_millis, max_pts = _device_search(eng, frame, models, plan, (rank, world))
        else:
            winners, stage_millis, max_pts = _device_search(eng, frame, models, plan, idx)
        t = torch.tensor([stage_millis[k] for k in ("render", "refine", "rerender", "cost")], dtype=torch.float64,
                         device=torch.device("cuda", eng.device))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)  # stage times: slowest rank
        stage_millis = dict(zip(("render", "refine", "rerender", "cost"), (float(x) for x in t.cpu().numpy())))
        return _assemble(plan, winners, stage_millis, t_start, max_pts)
    out = runner(frame, models, plan, idx)
    if out.stage_millis:
        stage_millis.update(out.stage_millis)
    mine = _winner_rows(plan, out, idx)
    keys = np.array([mine[o][0] if o in mine else pxd.NO_KEY for o in plan.active], dtype=np.int64)
    dev = None  # host path (gloo / injected runner); the nccl path returned above
    best = pxd.allreduce_min(keys, dev)
    # payload of the winners: only the owning rank contributes non-zeros (keys are unique per candidate)
    pay = np.zeros((len(plan.active), 27))
    for s, o in enumerate(plan.active):
        if o in mine and mine[o][0] == int(best[s]) and best[s] < pxd.NO_KEY:
            pay[s, :12], pay[s, 12:24] = mine[o][1].reshape(-1), mine[o][2].reshape(-1)
            pay[s, 24], pay[s, 25], pay[s, 26] = mine[o][3], mine[o][4], 1.0
    t = torch.from_numpy(pay)
    t = t.to(dev) if dev is not None else t
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    pay = t.cpu().numpy()
    mp_t = torch.tensor([float(out.n_rendered.max()) if out.n_rendered is not None and out.n_rendered.size else 0.0]
                        + [stage_millis[k] for k in ("render", "refine", "rerender", "cost")], dtype=torch.float64)
    mp_t = mp_t.to(dev) if dev is not None else mp_t
    dist.all_reduce(mp_t, op=dist.ReduceOp.MAX)  # stage times: slowest rank
    mp_h = mp_t.cpu().numpy()
    stage_millis = dict(zip(("render", "refine", "rerender", "cost"), (float(x) for x in mp_h[1:])))
    winners = {}
    for s, o in enumerate(plan.active):
        if pay[s, 26] == 1.0:
            winners[o] = (int(best[s]), pay[s, :12].reshape(3, 4), pay[s, 12:24].reshape(3, 4), int(pay[s, 24]), int(pay[s, 25]))
    return _assemble(plan, winners, stage_millis, t_start, int(mp_h[0]))


def _device_search(eng, frame, models, plan: SearchPlan, index=None):
    """Upload, fused search, on-device argmin (+ NCCL reduction when a communicator is up); only the
    per-object winner records come back to the host.  -> (winners, stage_millis, max_rendered_points).
    `index`: candidate subset of a flat plan, or (rank, world) for a lattice plan (the device generates the shard)."""
    if plan.lattice is not None:
        rank, world = index if index is not None else (0, 1)
        plan.n_observed = eng.upload_frame(frame, plan.cfg.stride)
        eng.upload_models({oid: models[oid] for oid in plan.active})
        eng.search_upload_lattice(plan, rank, world)
    else:
        eng.prepare_plan(frame, models, plan)
        eng.search_upload(plan, index)
    eng.search_run(eng.search_cfg(plan))
    eng.search_reduce()
    win = eng.search_winners()
    winners = {o: win[o][:5] for o in plan.active if o in win}
    max_pts = max([win[o][5] for o in plan.active if o in win], default=0)
    return winners, eng.stage_millis(), max_pts


def estimate_poses(frame, models: dict, cfg: SearchConfig, engine=None) -> SearchResult:
    """Estimate a pose for every detected object (search.py:217-377).  `engine` (optional, not in the
    reference's signature) selects the device context; default: the process-wide one."""
    from .engine import default_engine as _default_engine

    def default_engine():
        return engine if engine is not None else _default_engine()

    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
            return estimate_poses_distributed(frame, models, cfg)
    except ImportError:
        pass
    t_start = time.perf_counter()
    if not cfg.trace_path:
        plan = plan_lattice(frame, models, cfg)  # candidates, observed cloud and targets are built on the device
        if plan is not None and plan.n:
            winners, stage_millis, max_pts = _device_search(default_engine(), frame, models, plan)
            sm = {"render": 0.0, "refine": 0.0, "rerender": 0.0, "cost": 0.0}
            sm.update(stage_millis)
            return _assemble(plan, winners, sm, t_start, max_pts)
    plan = plan_search(frame, models, cfg, materialise_targets=False)  # the device crops the GICP targets
    if plan.n == 0:
        out = StageOutputs(np.zeros((0, 3, 4)), np.zeros((0, 3, 4)), np.zeros(0, np.int32),
                           np.zeros(0, np.int32))
        return assemble_result(plan, out, t_start)
    if cfg.trace_path:  # the per-candidate trace needs every candidate's costs on the host
        out = default_engine().run_plan(frame, models, plan)
        return assemble_result(plan, out, t_start)
    winners, stage_millis, max_pts = _device_search(default_engine(), frame, models, plan)
    sm = {"render": 0.0, "refine": 0.0, "rerender": 0.0, "cost": 0.0}
    sm.update(stage_millis)
    return _assemble(plan, winners, sm, t_start, max_pts)


def result_to_json(result: SearchResult) -> str:
    objects = []
    for e in result.estimates:
        rec = {"object_id": e.object_id, "failed": e.failed}
        if e.failed:
            rec["failure"] = e.failure
        else:
            rec["pose"] = [float(x) for x in e.pose.matrix3x4().reshape(-1)]
            rec["j_o"] = e.cost.j_o
            rec["j_r"] = e.cost.j_r
            rec["total"] = e.cost.total
            rec["provenance"] = list(e.provenance)
            rec["proposal_index"] = e.proposal_index
            rec["proposals_evaluated"] = e.proposals_evaluated
        objects.append(rec)
    return json.dumps({"objects": objects, "proposals_evaluated": result.proposals_evaluated},
                      indent=2, sort_keys=True)


def timings_to_json(result: SearchResult) -> str:
    return json.dumps({
        "total_millis": result.total_millis,
        "stage_millis": result.stage_millis,
        "per_object_millis": {str(e.object_id): e.millis for e in result.estimates},
    }, indent=2, sort_keys=True)
