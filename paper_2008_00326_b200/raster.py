"""Rendering entry points: observed-cloud extraction (host, per scene) and the
device-backed `render_batch` / `rasterize`.

Reference: pkg/src/rvpose/raster.py:137-304.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .colorspace import srgb_encode, srgb_to_lab
from .errors import DimensionMismatch, EmptyMesh
from .geometry import CameraIntrinsics, unproject_pixel
from .model import DepthImage, LabeledCloud

NEAR_PLANE = 1e-4


@dataclass(frozen=True)
class RenderedView:
    depth: DepthImage
    color: np.ndarray
    valid: np.ndarray
    object_id: int = 0

    def __post_init__(self):
        c = np.ascontiguousarray(self.color, dtype=np.float64)
        m = np.ascontiguousarray(self.valid, dtype=bool)
        if c.shape[:2] != self.depth.values.shape or m.shape != self.depth.values.shape:
            raise DimensionMismatch("view buffers disagree on image size")
        c.setflags(write=False)
        m.setflags(write=False)
        object.__setattr__(self, "color", c)
        object.__setattr__(self, "valid", m)


def _grid_cloud(valid, depth, color, k, stride) -> LabeledCloud:
    """Stride-grid unprojection in row-major order (raster.py:197-210)."""
    if stride < 1:
        raise ValueError("stride must be >= 1")
    vs, us = np.nonzero(valid[::stride, ::stride])
    if vs.size == 0:
        return LabeledCloud.empty()
    u, v = us * stride, vs * stride
    pts = unproject_pixel(k, u + 0.5, v + 0.5, depth[v, u])
    return LabeledCloud(pts, srgb_to_lab(color[v, u]), np.stack([u, v], axis=1).astype(np.int32))


def frame_to_cloud(frame, stride: int = 1) -> LabeledCloud:
    return _grid_cloud(frame.depth.valid, frame.depth.values, frame.color, frame.intrinsics, stride)


def render_to_cloud(view: RenderedView, k: CameraIntrinsics, stride: int = 1) -> LabeledCloud:
    return _grid_cloud(view.valid, view.depth.values, view.color, k, stride)


def cloud_labels(cloud: LabeledCloud, labels: np.ndarray) -> np.ndarray:
    if len(cloud) == 0:
        return np.zeros(0, dtype=np.int32)
    return labels[cloud.source_pixel[:, 1], cloud.source_pixel[:, 0]]


def rasterize(mesh, model_to_camera, k: CameraIntrinsics, object_id: int = 0) -> RenderedView:
    """One mesh -> depth + sRGB view, nearest surface wins (raster.py:137-158);
    the z-buffer runs on the device (px_rasterize), the sRGB encode on the host."""
    from .engine import default_engine

    if mesh.num_triangles == 0:
        raise EmptyMesh("mesh has no triangles")
    zbuf, cbuf, valid, _owner = default_engine().rasterize_mesh(mesh, model_to_camera, k)
    color = np.zeros((k.height, k.width, 3))
    color[valid] = srgb_encode(cbuf[valid])
    return RenderedView(DepthImage(np.where(valid, zbuf, 0.0), valid), color, valid, object_id)


def mark_occluders(view: RenderedView, frame, delta_occ: float = 0.0075) -> RenderedView:
    """raster.py:161-182 (single view, host; the batch path marks on the device)."""
    if frame.depth.values.shape != view.depth.values.shape:
        raise DimensionMismatch("frame and view sizes differ")
    occluded = (view.valid & frame.depth.valid
                & (frame.depth.values < view.depth.values - delta_occ)
                & (frame.labels != view.object_id))
    if not occluded.any():
        return view
    keep = view.valid & ~occluded
    return RenderedView(DepthImage(np.where(keep, view.depth.values, 0.0), keep),
                        np.where(keep[..., None], view.color, 0.0), keep, view.object_id)


def render_batch(models: dict, proposals, frame, k: CameraIntrinsics, stride: int = 1,
                 occluder_marking: bool = True, delta_occ: float = 0.0075,
                 workers: int = 1, chunksize: int | None = None) -> list:
    """Render -> occluder-mark -> cloud per proposal (raster.py:283-304), one
    device launch for the whole flat list.  `workers`/`chunksize` are accepted
    and result-neutral."""
    from .engine import default_engine

    return default_engine().render_batch(models, proposals, frame, k, stride,
                                         occluder_marking, delta_occ)
