"""Batched generalized ICP: boundary types and device-backed entry points.

Reference: pkg/src/rvpose/registration.py:26-52, 219-230, 410-558.
`estimate_covariances`, `gicp_align` and `m2m_gicp` run on the device
(px_covariances / px_refine_batch); `icp_point2point` is not on the search
path and is not provided.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .errors import TooFewPoints
from .geometry import Pose3Dof, RigidTransform, canonical_yaw

FAILURES = (None, "too_few_points", "degenerate_correspondences",
            "singular_normal_equations", "no_decrease")


@dataclass(frozen=True)
class GicpConfig:
    k_covariance: int = 20
    epsilon: float = 1e-3
    max_iterations: int = 30
    translation_tolerance: float = 1e-4
    rotation_tolerance: float = 1e-3
    max_correspondence_distance: float = 0.05

    def __post_init__(self):
        if self.k_covariance < 4:
            raise ValueError("k_covariance must be >= 4")
        if not (0.0 < self.epsilon < 1.0):
            raise ValueError("epsilon must lie in (0, 1)")
        if min(self.translation_tolerance, self.rotation_tolerance,
               self.max_correspondence_distance) <= 0:
            raise ValueError("tolerances must be positive")


@dataclass(frozen=True)
class RegistrationResult:
    transform: RigidTransform
    iterations: int
    final_residual: float
    converged: bool
    failure: str | None = None
    objective_trace: tuple = field(default=())


def _pts(cloud) -> np.ndarray:
    p = getattr(cloud, "points", cloud)
    return np.ascontiguousarray(p, dtype=np.float64).reshape(-1, 3)


def estimate_covariances(cloud, k_covariance: int = 20, epsilon: float = 1e-3) -> np.ndarray:
    """(n,3,3) regularised neighbourhood covariances (registration.py:219-230)."""
    from .engine import default_engine

    pts = _pts(cloud)
    if pts.shape[0] <= k_covariance:
        raise TooFewPoints(f"need more than {k_covariance} points, have {pts.shape[0]}")
    return default_engine().covariances(pts, k_covariance, epsilon)


def m2m_gicp(sources, targets, inits, cfg: GicpConfig, target_indices=None,
             workers: int = 1, chunksize: int | None = None) -> list:
    """Align each source to its referenced target (registration.py:514-550).
    `workers` / `chunksize` are accepted and result-neutral."""
    from .engine import default_engine

    sources = [_pts(s) for s in sources]
    targets = [_pts(t) for t in targets]
    if target_indices is None:
        if len(targets) == 1:
            target_indices = [0] * len(sources)
        elif len(targets) == len(sources):
            target_indices = list(range(len(sources)))
        else:
            raise ValueError("target_indices required for this shape")
    if len(inits) != len(sources) or len(target_indices) != len(sources):
        raise ValueError("sources, inits, target_indices must align")
    return default_engine().m2m_gicp(sources, targets, inits, cfg, target_indices)


def gicp_align(source, target, source_covs, target_covs, init: RigidTransform,
               cfg: GicpConfig) -> RegistrationResult:
    """Single-pair GICP (registration.py:410-476).  The device rebuilds the covariances from the clouds
    with cfg's (k, epsilon) -- exactly what every caller on the search path passes (registration.py:500-511).
    Covariances that are NOT `estimate_covariances(cloud, cfg.k_covariance, cfg.epsilon)` would silently be
    ignored, so they are refused instead (DeviceError): a limit reported, never a different answer."""
    from .errors import DeviceError

    src, tgt = _pts(source), _pts(target)
    if src.shape[0] < 3 or tgt.shape[0] < 3:
        return RegistrationResult(init, 0, float("inf"), False, "degenerate_correspondences")
    for pts, covs, what in ((src, source_covs, "source"), (tgt, target_covs, "target")):
        if covs is None or pts.shape[0] <= cfg.k_covariance:
            continue
        given = np.asarray(covs, dtype=np.float64).reshape(-1, 3, 3)
        if given.shape[0] != pts.shape[0] or not np.array_equal(given, estimate_covariances(pts, cfg.k_covariance, cfg.epsilon)):
            raise DeviceError(f"gicp_align: the {what} covariances differ from estimate_covariances(cloud, "
                              f"{cfg.k_covariance}, {cfg.epsilon}); the device path builds its own and cannot honour others")
    return m2m_gicp([src], [tgt], [init], cfg, [0])[0]


def project_to_3dof(t: RigidTransform, fixed_z: float = 0.0) -> Pose3Dof:
    yaw = float(np.arctan2(t.rotation[1, 0], t.rotation[0, 0]))
    return Pose3Dof(float(t.translation[0]), float(t.translation[1]), canonical_yaw(yaw))
