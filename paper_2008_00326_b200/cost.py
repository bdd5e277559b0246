"""Explanation cost: boundary types and the device-backed cost functions.

Reference: pkg/src/rvpose/cost.py:23-162.  `rendered_cost` on arbitrary clouds
runs the brute-force exact-NN kernel (px_rendered_cost); inside
`estimate_poses` the per-candidate costs come from the organised-grid kernel
(px_cost_batch / px_search_run).  No CPU implementation exists here.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .geometry import RigidTransform
from .model import InscribedCylinder, LabeledCloud


@dataclass(frozen=True)
class CostParams:
    delta: float = 0.0075
    tau_c: float = 12.5
    use_color: bool = True

    def __post_init__(self):
        if self.delta <= 0 or self.tau_c <= 0:
            raise ValueError("delta and tau_c must be positive")


@dataclass(frozen=True)
class CostBreakdown:
    j_o: int
    j_r: int

    def __post_init__(self):
        if self.j_o < 0 or self.j_r < 0:
            raise ValueError("costs are counts")

    @property
    def total(self) -> int:
        return self.j_o + self.j_r


@dataclass(frozen=True)
class ObservedAssociation:
    """Which observed points belong to an object: inscribed cylinder of the pose
    (3-DoF) or pixel label (6-DoF) (cost.py:48-75)."""

    mode: str
    pose: RigidTransform | None = None
    cylinder: InscribedCylinder | None = None
    object_id: int | None = None

    def __post_init__(self):
        if self.mode == "cylinder":
            if self.pose is None or self.cylinder is None:
                raise ValueError("cylinder mode needs pose and cylinder")
        elif self.mode == "label":
            if self.object_id is None:
                raise ValueError("label mode needs object_id")
        else:
            raise ValueError(f"unknown association mode {self.mode!r}")

    @staticmethod
    def inscribed_cylinder(pose, cylinder) -> "ObservedAssociation":
        return ObservedAssociation("cylinder", pose=pose, cylinder=cylinder)

    @staticmethod
    def label_mask(object_id: int) -> "ObservedAssociation":
        return ObservedAssociation("label", object_id=int(object_id))


def rendered_cost(rendered: LabeledCloud, observed: LabeledCloud, params: CostParams,
                  knn_cfg=None) -> tuple:
    """(j_r, explained) exactly as cost.py:91-135; `knn_cfg` is result-neutral."""
    from .engine import default_engine

    return default_engine().rendered_cost(rendered, observed, params)


def select_observed(observed: LabeledCloud, frame, assoc: ObservedAssociation) -> np.ndarray:
    """Boolean mask of observed points associated to the object (cost.py:138-144).
    Per-scene helper kept on the host; the batched search evaluates the same
    predicate on the device only inside the cylinder's screen bound."""
    if assoc.mode == "label":
        if len(observed) == 0:
            return np.zeros(0, dtype=bool)
        sp = observed.source_pixel
        return frame.labels[sp[:, 1], sp[:, 0]] == assoc.object_id
    pose = RigidTransform(assoc.pose.rotation, assoc.pose.translation)
    return assoc.cylinder.contains(pose.inverse().apply(observed.points))


def observed_cost(observed: LabeledCloud, frame, assoc: ObservedAssociation,
                  explained: np.ndarray, params: CostParams | None = None) -> int:
    return int(np.count_nonzero(select_observed(observed, frame, assoc) & ~explained))


def proposal_cost(rendered: LabeledCloud, observed: LabeledCloud, frame,
                  assoc: ObservedAssociation, params: CostParams, knn_cfg=None) -> CostBreakdown:
    j_r, explained = rendered_cost(rendered, observed, params, knn_cfg)
    return CostBreakdown(j_o=observed_cost(observed, frame, assoc, explained, params), j_r=j_r)
