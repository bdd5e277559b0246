"""Scene and model directories of the reference's dataset layout.

A scene directory holds `scene.json` (intrinsics, camera pose, detections,
optional ground truth), `color.ppm` (8-bit P6), `depth.pgm` (16-bit big-endian
P5, millimetres, 0 = no measurement) and `labels.pgm` (8-bit P5); a models
directory holds `models.json` plus one ASCII PLY per object (reference:
pkg/src/rvpose/scenegen.py:542-625, model.py:223-350).  Reading goes through
numpy buffers rather than per-token Python loops; values are the ones the
reference's readers produce (x/255, mm/1000, uint8 -> int32), which
tests/test_host_api.py checks on files written by either side.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .errors import DatasetError
from .geometry import CameraIntrinsics, RigidTransform
from .model import (DepthImage, Detection, InscribedCylinder, ObjectModel, ObjectState, SceneFrame,
                    TriangleMesh)


# ---- PNM ---------------------------------------------------------------------

def _pnm(path):
    """(magic, width, height, maxval, raster bytes); `#` comments allowed in the header."""
    raw = Path(path).read_bytes()
    magic, pos, fields = raw[:2], 2, []
    while len(fields) < 3:
        end = raw.find(b"\n", pos)
        if end < 0:
            raise DatasetError(f"{path}: truncated PNM header")
        fields += [int(t) for t in raw[pos:end].split(b"#")[0].split()]
        pos = end + 1
    w, h, maxval = fields[:3]
    return magic, w, h, maxval, raw[pos:]


def _raster(path, data, dtype, shape):
    n = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if len(data) < n:
        raise DatasetError(f"{path}: truncated raster ({len(data)} of {n} bytes)")
    return np.frombuffer(data, dtype=dtype, count=int(np.prod(shape))).reshape(shape)


def load_ppm(path) -> np.ndarray:
    magic, w, h, maxval, data = _pnm(path)
    if magic != b"P6" or maxval != 255:
        raise DatasetError(f"{path}: expected 8-bit P6")
    return _raster(path, data, np.uint8, (h, w, 3)) / 255.0


def load_depth_pgm(path) -> DepthImage:
    magic, w, h, maxval, data = _pnm(path)
    if magic != b"P5" or maxval != 65535:
        raise DatasetError(f"{path}: expected 16-bit P5")
    mm = _raster(path, data, ">u2", (h, w)).astype(np.float64)
    valid = mm > 0
    return DepthImage(np.where(valid, mm / 1000.0, 0.0), valid)


def load_labels_pgm(path) -> np.ndarray:
    magic, w, h, maxval, data = _pnm(path)
    if magic != b"P5" or maxval != 255:
        raise DatasetError(f"{path}: expected 8-bit P5")
    return _raster(path, data, np.uint8, (h, w)).astype(np.int32)


def _write_pnm(path, magic, arr, maxval):
    h, w = arr.shape[:2]
    with open(path, "wb") as f:
        f.write(f"{magic}\n{w} {h}\n{maxval}\n".encode())
        f.write(arr.tobytes())


def save_ppm(path, image) -> None:
    _write_pnm(path, "P6", np.clip(np.rint(np.asarray(image, dtype=np.float64) * 255.0), 0, 255).astype(np.uint8), 255)


def save_depth_pgm(path, depth: DepthImage) -> None:
    mm = np.where(depth.valid, np.rint(depth.values * 1000.0), 0.0)
    _write_pnm(path, "P5", np.clip(mm, 0, 65535).astype(">u2"), 65535)


def save_labels_pgm(path, labels) -> None:
    _write_pnm(path, "P5", np.asarray(labels).astype(np.uint8), 255)


# ---- PLY ---------------------------------------------------------------------

def load_ply(path) -> TriangleMesh:
    lines = Path(path).read_text().splitlines()
    if not lines or lines[0].strip() != "ply":
        raise DatasetError(f"{path}: not a PLY file")
    n_vert = n_face = 0
    body = None
    for i, line in enumerate(lines[1:], 1):
        tok = line.split()
        if tok[:2] == ["element", "vertex"]:
            n_vert = int(tok[2])
        elif tok[:2] == ["element", "face"]:
            n_face = int(tok[2])
        elif tok[:1] == ["end_header"]:
            body = lines[i + 1:]
            break
    if body is None or len(body) < n_vert + n_face:
        raise DatasetError(f"{path}: truncated PLY body")
    try:
        vert = np.array([ln.split()[:6] for ln in body[:n_vert]], dtype=np.float64).reshape(n_vert, 6)
        face = np.array([ln.split()[:4] for ln in body[n_vert:n_vert + n_face]], dtype=np.int64).reshape(n_face, 4)
    except ValueError as e:
        raise DatasetError(f"{path}: malformed PLY body: {e}") from e
    if n_face and (face[:, 0] != 3).any():
        raise DatasetError(f"{path}: only triangle faces supported")
    return TriangleMesh(vert[:, :3], vert[:, 3:6].astype(np.int64) / 255.0, face[:, 1:].astype(np.int32))


def save_ply(path, mesh: TriangleMesh) -> None:
    v, t = mesh.vertices, mesh.triangles
    c = np.clip(np.rint(mesh.vertex_colors * 255.0), 0, 255).astype(int)
    head = ["ply", "format ascii 1.0", f"element vertex {v.shape[0]}", "property float x", "property float y",
            "property float z", "property uchar red", "property uchar green", "property uchar blue",
            f"element face {t.shape[0]}", "property list uchar int vertex_indices", "end_header"]
    rows = [f"{p[0]:.9g} {p[1]:.9g} {p[2]:.9g} {q[0]} {q[1]} {q[2]}" for p, q in zip(v, c)]
    rows += [f"3 {a} {b} {d}" for a, b, d in t]
    Path(path).write_text("\n".join(head + rows) + "\n")


# ---- directories -------------------------------------------------------------

def _pose(vals) -> RigidTransform:
    return RigidTransform.from_matrix3x4(np.asarray(vals, dtype=np.float64).reshape(3, 4))


def _pose_list(t) -> list:
    return [float(x) for x in t.matrix3x4().reshape(-1)]


def load_scene(scene_dir) -> SceneFrame:
    d = Path(scene_dir)
    try:
        meta = json.loads((d / "scene.json").read_text())
        color, depth, labels = load_ppm(d / "color.ppm"), load_depth_pgm(d / "depth.pgm"), load_labels_pgm(d / "labels.pgm")
    except FileNotFoundError as e:
        raise DatasetError(f"incomplete scene at {scene_dir}: {e}") from e
    except json.JSONDecodeError as e:
        raise DatasetError(f"bad scene.json in {scene_dir}: {e}") from e
    ki = meta["intrinsics"]
    k = CameraIntrinsics(ki["fx"], ki["fy"], ki["cx"], ki["cy"], ki["width"], ki["height"], _pose(ki["camera_pose"]))
    dets = [Detection(r["object_id"], tuple(r["full_bbox"]), labels == r["object_id"]) for r in meta["detections"]]
    gt = [ObjectState(r["object_id"], _pose(r["pose"])) for r in meta.get("ground_truth", [])] or None
    return SceneFrame(color, depth, labels, dets, k, gt)


def save_scene(scene_dir, frame: SceneFrame) -> None:
    d = Path(scene_dir)
    d.mkdir(parents=True, exist_ok=True)
    save_ppm(d / "color.ppm", frame.color)
    save_depth_pgm(d / "depth.pgm", frame.depth)
    save_labels_pgm(d / "labels.pgm", frame.labels)
    k = frame.intrinsics
    meta = {"intrinsics": {"fx": k.fx, "fy": k.fy, "cx": k.cx, "cy": k.cy, "width": k.width, "height": k.height,
                           "camera_pose": _pose_list(k.camera_pose)},
            "detections": [{"object_id": x.object_id, "full_bbox": list(x.full_bbox)} for x in frame.detections],
            "ground_truth": [{"object_id": s.object_id, "pose": _pose_list(s.pose)} for s in (frame.ground_truth or [])]}
    (d / "scene.json").write_text(json.dumps(meta, indent=2, sort_keys=True))


def load_models(models_dir) -> dict:
    d = Path(models_dir)
    try:
        index = json.loads((d / "models.json").read_text())
    except FileNotFoundError as e:
        raise DatasetError(f"no models.json in {models_dir}") from e
    out = {}
    for rec in index:
        r, z0, z1 = rec["inscribed_cylinder"]
        try:
            mesh = load_ply(d / rec["mesh"])
        except FileNotFoundError as e:
            raise DatasetError(f"missing mesh {rec['mesh']} in {models_dir}") from e
        out[rec["object_id"]] = ObjectModel(rec["object_id"], mesh, InscribedCylinder(r, z0, z1), rec["yaw_symmetric"])
    return out


def save_models(models_dir, models: dict) -> None:
    d = Path(models_dir)
    d.mkdir(parents=True, exist_ok=True)
    index = []
    for oid in sorted(models):
        m = models[oid]
        name = f"object_{oid:03d}.ply"
        save_ply(d / name, m.mesh)
        c = m.inscribed_cylinder
        index.append({"object_id": oid, "mesh": name, "inscribed_cylinder": [c.radius, c.z_min, c.z_max],
                      "yaw_symmetric": m.yaw_symmetric})
    (d / "models.json").write_text(json.dumps(index, indent=2, sort_keys=True))
