"""Device engine: owns one libpx context and maps the boundary types onto the
C-ABI calls.  One Engine per process / per GPU (one process per GPU under
torchrun).  Every method raises DeviceError if libpx.so or a CUDA device is
missing -- there is no CPU code path behind these calls.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .colorspace import srgb_decode
from .errors import DeviceError, EmptyMesh, UnknownObjectId
from .geometry import RigidTransform
from .model import LabeledCloud
from .registration import FAILURES, RegistrationResult

_ADHOC_ID = 2**31 - 1


def _pose3x4(t) -> np.ndarray:
    m = np.empty((3, 4))
    m[:, :3] = t.rotation
    m[:, 3] = t.translation
    return m


class Engine:
    def __init__(self, device: int = 0):
        self.lib = N.load()
        self.ctx = N.vp()
        rc = self.lib.px_ctx_create(int(device), C.byref(self.ctx))
        if rc != 0:
            msg = self.lib.px_last_error(None)
            raise DeviceError(f"px_ctx_create({device}) failed: {msg.decode() if msg else rc}")
        self.device = int(device)
        import os
        if os.environ.get("PX_SCRATCH_MB"):  # tuning knob: per-chunk candidate scratch (default 8 GiB)
            N.check(self.ctx, self.lib.px_ctx_set_scratch_budget(self.ctx, int(os.environ["PX_SCRATCH_MB"]) << 20),
                    "px_ctx_set_scratch_budget")
        self._scene_key = None
        self._model_keys = {}
        self._model_refs = {}
        self._keep = []

    def close(self):
        if self.ctx:
            self.lib.px_ctx_destroy(self.ctx)
            self.ctx = N.vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- state ---------------------------------------------------------------
    def set_stream(self, cuda_stream_ptr: int | None):
        N.check(self.ctx, self.lib.px_ctx_set_stream(self.ctx, cuda_stream_ptr), "px_ctx_set_stream")

    def sync(self):
        N.check(self.ctx, self.lib.px_ctx_sync(self.ctx), "px_ctx_sync")

    def launch_count(self) -> int:
        return int(self.lib.px_ctx_launch_count(self.ctx))

    def upload_scene(self, frame, stride: int, observed=None, obs_labels=None, force=False):
        from .raster import cloud_labels, frame_to_cloud

        key = (id(frame), int(stride))
        if not force and key == self._scene_key:
            return
        if observed is None:
            observed = frame_to_cloud(frame, stride)
        if obs_labels is None:
            obs_labels = cloud_labels(observed, frame.labels)
        k = frame.intrinsics
        depth = N.f64(frame.depth.values)
        valid = np.ascontiguousarray(frame.depth.valid, dtype=np.uint8)
        labels = N.i32(frame.labels)
        intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)
        pts, lab = N.f64(observed.points), N.f64(observed.lab_colors)
        src, ol = N.i32(observed.source_pixel), N.i32(obs_labels)
        rc = self.lib.px_scene_upload(self.ctx, k.height, k.width, N.ptr(depth, N.f64p), N.ptr(valid, N.u8p),
                                      N.ptr(labels, N.i32p), N.ptr(intr, N.f64p), int(stride),
                                      N.ptr(pts, N.f64p), N.ptr(lab, N.f64p), N.ptr(src, N.i32p),
                                      N.ptr(ol, N.i32p), len(observed))
        N.check(self.ctx, rc, "px_scene_upload")
        self._scene_key = key
        self._keep = [frame]

    def upload_frame(self, frame, stride: int, sample_on_host: bool = False) -> int:
        """Scene upload with the observed cloud built on the device (raster.frame_to_cloud + cloud_labels,
        raster.py:191-217); returns the number of observed points.  `sample_on_host` forces the path taken for planes
        that are not C-contiguous float64 / int32 / bool arrays (numpy samples the stride grid)."""
        k = frame.intrinsics
        dv, vv, lv, cv = frame.depth.values, frame.depth.valid, frame.labels, frame.color
        if (not sample_on_host and all(isinstance(a, np.ndarray) and a.flags.c_contiguous for a in (dv, vv, lv, cv)) and dv.dtype == np.float64
                and cv.dtype == np.float64 and lv.dtype == np.int32 and vv.dtype in (np.bool_, np.uint8)
                and dv.shape == vv.shape == lv.shape == (k.height, k.width) and cv.shape == (k.height, k.width, 3)):
            # the library samples the stride grid itself (C loop into pinned memory: numpy's strided copy of the colour
            # plane alone took longer than the whole upload)
            intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)
            n = C.c_int64(0)
            rc = self.lib.px_scene_upload_frame_full(self.ctx, k.height, k.width, N.ptr(dv, N.f64p), N.ptr(vv.view(np.uint8), N.u8p),
                                                     N.ptr(lv, N.i32p), N.ptr(cv, N.f64p), N.ptr(intr, N.f64p), int(stride),
                                                     C.cast(C.byref(n), N.i64p))
            N.check(self.ctx, rc, "px_scene_upload_frame_full")
            self._scene_key = None
            self._keep = [frame]
            return int(n.value)
        # other layouts / dtypes: sample on the host, upload a quarter of the bytes
        depth = N.f64(frame.depth.values[::stride, ::stride])
        valid = np.ascontiguousarray(frame.depth.valid[::stride, ::stride], dtype=np.uint8)
        labels = N.i32(frame.labels[::stride, ::stride])
        cgrid = np.ascontiguousarray(frame.color[::stride, ::stride], dtype=np.float64)
        intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)
        n = C.c_int64(0)
        rc = self.lib.px_scene_upload_frame(self.ctx, k.height, k.width, N.ptr(depth, N.f64p), N.ptr(valid, N.u8p),
                                            N.ptr(labels, N.i32p), N.ptr(cgrid, N.f64p), N.ptr(intr, N.f64p), int(stride),
                                            C.cast(C.byref(n), N.i64p))
        N.check(self.ctx, rc, "px_scene_upload_frame")
        self._scene_key = None
        self._keep = [frame]
        return int(n.value)

    def download_scene_cloud(self, n: int):
        """(points, lab, source_pixel, labels) of the resident observed cloud."""
        pts, lab = np.empty((n, 3)), np.empty((n, 3))
        src, lbl = np.empty((n, 2), dtype=np.int32), np.empty(n, dtype=np.int32)
        rc = self.lib.px_scene_download_cloud(self.ctx, N.ptr(pts, N.f64p), N.ptr(lab, N.f64p), N.ptr(src, N.i32p), N.ptr(lbl, N.i32p))
        N.check(self.ctx, rc, "px_scene_download_cloud")
        return pts, lab, src, lbl

    def search_upload_lattice(self, plan, rank: int = 0, world: int = 1) -> int:
        """Candidates (and GICP targets) of a lattice plan generated on the device; returns the local count."""
        cfg = plan.cfg
        arr = (N.Lattice * max(len(plan.lattice), 1))()
        keep = []
        for i, f in enumerate(plan.lattice):
            r, t = N.f64(f.rotations), N.f64(f.translations)
            keep += [r, t]
            arr[i].object_id, arr[i].n_outer, arr[i].n_inner = int(f.object_id), int(f.n_outer), int(f.n_inner)
            arr[i].rotations, arr[i].translations = N.ptr(r, N.f64p), N.ptr(t, N.f64p)
            arr[i].capsule[:] = [float(x) for x in f.capsule]
        w2c, c2w = N.f64(plan.w2c), N.f64(plan.c2w)
        g = self._gicp_cfg(cfg.gicp)
        n = C.c_int64(0)
        rc = self.lib.px_search_upload_lattice(self.ctx, int(cfg.mode == "3dof"), len(plan.lattice), arr, N.ptr(w2c, N.f64p),
                                               int(plan.w2c_vec_order), N.ptr(c2w, N.f64p),
                                               C.byref(g) if cfg.refine else None, int(rank), int(world),
                                               C.cast(C.byref(n), N.i64p))
        N.check(self.ctx, rc, "px_search_upload_lattice")
        return int(n.value)

    def download_candidates(self, n: int, with_targets: bool = True):
        slot, rank = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        pose = np.empty((n, 3, 4))
        tidx = np.zeros(n, dtype=np.int32) if with_targets else None
        rc = self.lib.px_search_candidates(self.ctx, N.ptr(slot, N.i32p), N.ptr(pose, N.f64p), N.ptr(tidx, N.i32p), N.ptr(rank, N.i32p))
        N.check(self.ctx, rc, "px_search_candidates")
        ids = np.zeros(max(int(self.lib.px_model_count(self.ctx)), 1), dtype=np.int32)
        self.lib.px_model_ids(self.ctx, N.ptr(ids, N.i32p))
        return ids[slot], pose, tidx, rank

    def upload_model(self, object_id: int, mesh, cylinder=None):
        if mesh.num_triangles == 0:
            raise EmptyMesh("mesh has no triangles")
        key = (id(mesh), None if cylinder is None else (cylinder.radius, cylinder.z_min, cylinder.z_max))
        if self._model_keys.get(object_id) == key:
            return
        verts = N.f64(mesh.vertices)
        col = N.f64(srgb_decode(mesh.vertex_colors))  # once per model, host numpy = reference bits
        tris = N.i32(mesh.triangles)
        if cylinder is None:
            cyl = np.array([1.0, 0.0, 1.0])
        else:
            cyl = np.array([cylinder.radius**2, cylinder.z_min, cylinder.z_max], dtype=np.float64)
        rc = self.lib.px_model_upload(self.ctx, int(object_id), N.ptr(verts, N.f64p), N.ptr(col, N.f64p),
                                      N.ptr(tris, N.i32p), verts.shape[0], tris.shape[0], N.ptr(cyl, N.f64p))
        N.check(self.ctx, rc, "px_model_upload")
        self._model_keys[object_id] = key
        self._model_refs[object_id] = mesh  # keeps id(mesh) from being reused while the key is cached

    def upload_models(self, models: dict):
        for oid, m in models.items():
            self.upload_model(oid, m.mesh, m.inscribed_cylinder)

    # -- clouds ----------------------------------------------------------------
    def _download_clouds(self, handle) -> list:
        n = int(self.lib.px_clouds_count(handle))
        counts = np.zeros(n, dtype=np.int32)
        if n:
            N.check(self.ctx, self.lib.px_clouds_counts(self.ctx, handle, N.ptr(counts, N.i32p)), "px_clouds_counts")
        tot = int(counts.sum())
        pts, lab = np.zeros((tot, 3)), np.zeros((tot, 3))
        src = np.zeros((tot, 2), dtype=np.int32)
        if tot:
            N.check(self.ctx, self.lib.px_clouds_download(self.ctx, handle, N.ptr(pts, N.f64p), N.ptr(lab, N.f64p),
                                                          N.ptr(src, N.i32p)), "px_clouds_download")
        out, o = [], 0
        for c in counts:
            c = int(c)
            out.append(LabeledCloud(pts[o:o + c], lab[o:o + c], src[o:o + c]) if c else LabeledCloud.empty())
            o += c
        return out

    def _upload_clouds(self, point_arrays, labs=None, srcs=None):
        counts = np.array([p.shape[0] for p in point_arrays], dtype=np.int32)
        pts = N.f64(np.concatenate(point_arrays)) if len(point_arrays) else np.zeros((0, 3))
        lab = N.f64(np.concatenate(labs)) if labs is not None and len(labs) else None
        src = N.i32(np.concatenate(srcs)) if srcs is not None and len(srcs) else None
        h = N.vp()
        rc = self.lib.px_clouds_upload(self.ctx, len(point_arrays), N.ptr(counts, N.i32p), N.ptr(pts, N.f64p),
                                       N.ptr(lab, N.f64p), N.ptr(src, N.i32p), C.byref(h))
        N.check(self.ctx, rc, "px_clouds_upload")
        return h

    # -- raster ------------------------------------------------------------------
    def render_clouds_handle(self, oids, poses, occluder_marking, delta_occ):
        oids, poses = N.i32(oids), N.f64(poses)
        h = N.vp()
        rc = self.lib.px_render_batch(self.ctx, N.ptr(oids, N.i32p), N.ptr(poses, N.f64p), oids.shape[0],
                                      int(bool(occluder_marking)), float(delta_occ), C.byref(h))
        N.check(self.ctx, rc, "px_render_batch")
        return h

    def render_batch(self, models, proposals, frame, k, stride, occluder_marking, delta_occ) -> list:
        oids, poses = [], []
        for oid, plist in proposals:
            if oid not in models:
                raise UnknownObjectId(f"no model registered for id {oid}")
            if models[oid].mesh.num_triangles == 0:
                raise EmptyMesh("mesh has no triangles")
            for p in plist:
                oids.append(oid)
                poses.append(_pose3x4(p))
        self.upload_scene(frame, stride)
        self.upload_models({oid: models[oid] for oid in set(oids)})
        if not oids:
            return []
        h = self.render_clouds_handle(np.array(oids), np.stack(poses), occluder_marking, delta_occ)
        try:
            return self._download_clouds(h)
        finally:
            self.lib.px_clouds_free(self.ctx, h)

    def rasterize_mesh(self, mesh, pose, k):
        """Full-image z-buffer of one mesh: (zbuf, cbuf_linear, valid, owner)."""
        class _F:  # minimal frame carrying only the camera
            pass
        h, w = k.height, k.width
        depth = np.zeros((h, w))
        valid = np.zeros((h, w), dtype=np.uint8)
        labels = np.zeros((h, w), dtype=np.int32)
        intr = np.array([k.fx, k.fy, k.cx, k.cy], dtype=np.float64)
        rc = self.lib.px_scene_upload(self.ctx, h, w, N.ptr(depth, N.f64p), N.ptr(valid, N.u8p),
                                      N.ptr(labels, N.i32p), N.ptr(intr, N.f64p), 1, None, None, None, None, 0)
        N.check(self.ctx, rc, "px_scene_upload")
        self._scene_key = None
        self._model_keys.pop(_ADHOC_ID, None)
        self.upload_model(_ADHOC_ID, mesh, None)
        zbuf, cbuf = np.empty((h, w)), np.empty((h, w, 3))
        val, owner = np.empty((h, w), dtype=np.uint8), np.empty((h, w), dtype=np.int32)
        p = N.f64(_pose3x4(pose))
        rc = self.lib.px_rasterize(self.ctx, _ADHOC_ID, N.ptr(p, N.f64p), N.ptr(zbuf, N.f64p), N.ptr(cbuf, N.f64p),
                                   N.ptr(val, N.u8p), N.ptr(owner, N.i32p))
        N.check(self.ctx, rc, "px_rasterize")
        return zbuf, cbuf, val.astype(bool), owner

    # -- registration --------------------------------------------------------------
    def covariances(self, pts, k, eps) -> np.ndarray:
        pts = N.f64(pts)
        out = np.empty((pts.shape[0], 3, 3))
        rc = self.lib.px_covariances(self.ctx, N.ptr(pts, N.f64p), pts.shape[0], int(k), float(eps), N.ptr(out, N.f64p))
        N.check(self.ctx, rc, "px_covariances")
        return out

    def upload_targets(self, offsets, points, gicp_cfg, obs_index=None):
        offsets = np.ascontiguousarray(offsets, dtype=np.int64)
        points = N.f64(points)
        oi = None if obs_index is None else np.ascontiguousarray(obs_index, dtype=np.int64)
        g = self._gicp_cfg(gicp_cfg)
        rc = self.lib.px_targets_upload(self.ctx, offsets.shape[0] - 1, N.ptr(offsets, N.i64p), N.ptr(points, N.f64p),
                                        N.ptr(oi, N.i64p), C.byref(g))
        N.check(self.ctx, rc, "px_targets_upload")

    def build_targets(self, plan):
        """GICP targets cropped from the resident observed cloud on the device
        (search.py:393-426) from the plan's target specs."""
        g = self._gicp_cfg(plan.cfg.gicp)
        if plan.cfg.mode == "3dof":
            prm = N.f64(plan.target_capsules)
            c2w = N.f64(plan.c2w)
            rc = self.lib.px_targets_build_capsules(self.ctx, prm.shape[0], N.ptr(prm, N.f64p), N.ptr(c2w, N.f64p), C.byref(g))
            N.check(self.ctx, rc, "px_targets_build_capsules")
        else:
            ids = N.i32(plan.target_labels)
            rc = self.lib.px_targets_build_labels(self.ctx, ids.shape[0], N.ptr(ids, N.i32p), C.byref(g))
            N.check(self.ctx, rc, "px_targets_build_labels")

    def download_targets(self):
        """(offsets, points, obs_index) of the resident targets."""
        n, tot = C.c_int32(0), C.c_int64(0)
        N.check(self.ctx, self.lib.px_targets_info(self.ctx, C.byref(n), C.byref(tot)), "px_targets_info")
        off = np.zeros(n.value + 1, dtype=np.int64)
        pts = np.empty((tot.value, 3))
        oi = np.zeros(tot.value, dtype=np.int32)
        rc = self.lib.px_targets_download(self.ctx, N.ptr(off, N.i64p), N.ptr(pts, N.f64p), N.ptr(oi, N.i32p))
        N.check(self.ctx, rc, "px_targets_download")
        return off, pts, oi

    def target_covariances(self, total) -> np.ndarray:
        out = np.empty((total, 3, 3))
        N.check(self.ctx, self.lib.px_targets_covariances(self.ctx, N.ptr(out, N.f64p)), "px_targets_covariances")
        return out

    @staticmethod
    def _gicp_cfg(cfg) -> N.GicpCfg:
        return N.GicpCfg(cfg.k_covariance, cfg.max_iterations, cfg.epsilon, cfg.translation_tolerance,
                         cfg.rotation_tolerance, cfg.max_correspondence_distance)

    def refine_handle(self, handle, target_idx, cfg, inits=None, want_residual=False, want_trace=False):
        n = int(self.lib.px_clouds_count(handle))
        tidx = N.i32(target_idx)
        init = None if inits is None else N.f64(inits)
        out_T = np.empty((n, 3, 4))
        iters, flags, ntr = (np.zeros(n, dtype=np.int32) for _ in range(3))
        resid = np.empty(n) if want_residual else None
        trace = np.zeros((n, max(cfg.max_iterations, 1), 2)) if want_trace else None
        g = self._gicp_cfg(cfg)
        rc = self.lib.px_refine_batch(self.ctx, handle, N.ptr(tidx, N.i32p), N.ptr(init, N.f64p), C.byref(g),
                                      N.ptr(out_T, N.f64p), N.ptr(iters, N.i32p), N.ptr(flags, N.i32p),
                                      N.ptr(resid, N.f64p), N.ptr(trace, N.f64p), N.ptr(ntr, N.i32p))
        N.check(self.ctx, rc, "px_refine_batch")
        return out_T, iters, flags, resid, trace, ntr

    def m2m_gicp(self, sources, targets, inits, cfg, target_indices) -> list:
        offs = np.zeros(len(targets) + 1, dtype=np.int64)
        np.cumsum([t.shape[0] for t in targets], out=offs[1:])
        tp = np.concatenate(targets) if targets else np.zeros((0, 3))
        self.upload_targets(offs, tp, cfg)
        if not sources:
            return []
        h = self._upload_clouds(sources)
        try:
            init_m = np.stack([_pose3x4(t) for t in inits])
            T, iters, flags, resid, trace, ntr = self.refine_handle(h, target_indices, cfg, init_m, True, True)
        finally:
            self.lib.px_clouds_free(self.ctx, h)
        out = []
        for i in range(len(sources)):
            code = int(flags[i]) & 0xff
            if code == 1:  # too_few_points: init returned as given (registration.py:504-510)
                out.append(RegistrationResult(inits[i], 0, float("inf"), False, "too_few_points"))
                continue
            tr = tuple((float(a), float(b)) for a, b in trace[i, :int(ntr[i])])
            out.append(RegistrationResult(RigidTransform.from_matrix3x4(T[i]), int(iters[i]), float(resid[i]),
                                          bool(int(flags[i]) & 0x100), FAILURES[code], tr))
        return out

    def gicp_linearize(self, src, tgt, T, cfg):
        """registration._gicp_linearize through the production kernels (test export):
        -> (f0, n_corr, h (6,6), g (6,), corr (n,) i64, w (n,3,3))."""
        src, tgt, T = N.f64(src), N.f64(tgt), N.f64(T)
        n = src.shape[0]
        h, g, f0 = np.zeros((6, 6)), np.zeros(6), C.c_double(0.0)
        nc = C.c_int32(0)
        corr, w = np.zeros(n, dtype=np.int64), np.zeros((n, 3, 3))
        gc = self._gicp_cfg(cfg)
        rc = self.lib.px_gicp_linearize(self.ctx, N.ptr(src, N.f64p), n, N.ptr(tgt, N.f64p), tgt.shape[0], N.ptr(T, N.f64p),
                                        C.byref(gc), N.ptr(h, N.f64p), N.ptr(g, N.f64p), C.cast(C.byref(f0), N.f64p),
                                        C.cast(C.byref(nc), N.i32p), N.ptr(corr, N.i64p), N.ptr(w, N.f64p))
        N.check(self.ctx, rc, "px_gicp_linearize")
        return float(f0.value), int(nc.value), h, g, corr, w

    def ciede2000(self, lab_a, lab_b) -> np.ndarray:
        a, b = N.f64(lab_a).reshape(-1, 3), N.f64(lab_b).reshape(-1, 3)
        out = np.zeros(a.shape[0])
        N.check(self.ctx, self.lib.px_ciede2000(self.ctx, N.ptr(a, N.f64p), N.ptr(b, N.f64p), a.shape[0], N.ptr(out, N.f64p)),
                "px_ciede2000")
        return out

    def srgb_to_lab(self, rgb, linear_input=False) -> np.ndarray:
        a = N.f64(rgb).reshape(-1, 3)
        out = np.zeros_like(a)
        N.check(self.ctx, self.lib.px_srgb_to_lab(self.ctx, N.ptr(a, N.f64p), a.shape[0], int(bool(linear_input)),
                                                  N.ptr(out, N.f64p)), "px_srgb_to_lab")
        return out

    # -- cost ------------------------------------------------------------------------
    def rendered_cost(self, rendered, observed, params):
        n_obs, n_r = len(observed), len(rendered)
        explained = np.zeros(n_obs, dtype=np.uint8)
        jr = C.c_int32(0)
        rp, rl = N.f64(rendered.points), N.f64(rendered.lab_colors)
        op, ol = N.f64(observed.points), N.f64(observed.lab_colors)
        rc = self.lib.px_rendered_cost(self.ctx, N.ptr(rp, N.f64p), N.ptr(rl, N.f64p), n_r, N.ptr(op, N.f64p),
                                       N.ptr(ol, N.f64p), n_obs, float(params.delta), float(params.tau_c),
                                       int(bool(params.use_color)), C.byref(jr), N.ptr(explained, N.u8p))
        N.check(self.ctx, rc, "px_rendered_cost")
        return int(jr.value), explained.astype(bool)

    def cost_handle(self, handle, oids, cyl_poses, delta, tau_c, use_color):
        n = int(self.lib.px_clouds_count(handle))
        oids = N.i32(oids)
        poses = None if cyl_poses is None else N.f64(cyl_poses)
        jo, jr = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        rc = self.lib.px_cost_batch(self.ctx, handle, N.ptr(oids, N.i32p), N.ptr(poses, N.f64p), float(delta),
                                    float(tau_c), int(bool(use_color)), N.ptr(jo, N.i32p), N.ptr(jr, N.i32p))
        N.check(self.ctx, rc, "px_cost_batch")
        return jo, jr

    def knn(self, queries, targets, k):
        q, t = N.f64(queries).reshape(-1, 3), N.f64(targets).reshape(-1, 3)
        idx = np.full((q.shape[0], k), -1, dtype=np.int64)
        d2 = np.full((q.shape[0], k), np.inf)
        if q.shape[0] and t.shape[0]:
            rc = self.lib.px_knn(self.ctx, N.ptr(q, N.f64p), q.shape[0], N.ptr(t, N.f64p), t.shape[0], int(k),
                                 N.ptr(idx, N.i64p), N.ptr(d2, N.f64p))
            N.check(self.ctx, rc, "px_knn")
        return idx, d2

    # -- fused search --------------------------------------------------------------
    def search_cfg(self, plan) -> N.SearchCfg:
        cfg = plan.cfg
        sc = N.SearchCfg()
        sc.mode3dof = int(cfg.mode == "3dof")
        sc.use_color, sc.occluder_marking, sc.refine = int(cfg.use_color), int(cfg.occluder_marking), int(cfg.refine)
        sc.delta, sc.tau_c = float(cfg.delta), float(cfg.tau_c)
        sc.gicp = self._gicp_cfg(cfg.gicp)
        sc.cam_to_world[:] = list(np.asarray(plan.c2w).reshape(-1))
        sc.world_to_cam[:] = list(np.asarray(plan.w2c).reshape(-1))
        sc.c2w_vec_order, sc.w2c_vec_order = int(plan.c2w_vec_order), int(plan.w2c_vec_order)
        sc.fixed_z = float(cfg.fixed_z)
        return sc

    def search_upload(self, plan, index=None):
        """Make the plan's candidates (or the subset `index`) device-resident."""
        oid, pose, rank = plan.flat_oid, plan.cam_poses, plan.rank_in_object()
        tidx = plan.target_idx
        if index is not None:
            oid, pose, rank = oid[index], pose[index], rank[index]
            tidx = None if tidx is None else tidx[index]
        oid, pose, rank = N.i32(oid), N.f64(pose), N.i32(rank)
        tidx = None if tidx is None else N.i32(tidx)
        rc = self.lib.px_search_upload(self.ctx, oid.shape[0], N.ptr(oid, N.i32p), N.ptr(pose, N.f64p),
                                       N.ptr(tidx, N.i32p), N.ptr(rank, N.i32p))
        N.check(self.ctx, rc, "px_search_upload")
        return oid.shape[0]

    def search_run(self, sc: N.SearchCfg):
        N.check(self.ctx, self.lib.px_search_run(self.ctx, C.byref(sc)), "px_search_run")

    def search_download(self, n, full=True):
        from .search import StageOutputs

        nm = int(self.lib.px_model_count(self.ctx))
        keys = np.zeros(max(nm, 1), dtype=np.uint64)
        ms = np.zeros(4)
        jo, jr = np.zeros(n, dtype=np.int32), np.zeros(n, dtype=np.int32)
        ref = np.empty((n, 3, 4)) if full else None
        regT = np.empty((n, 3, 4)) if full else None
        it, fl, nf, nl = ((np.zeros(n, dtype=np.int32) if full else None) for _ in range(4))
        rc = self.lib.px_search_download(self.ctx, N.ptr(ref, N.f64p), N.ptr(regT, N.f64p), N.ptr(it, N.i32p),
                                         N.ptr(fl, N.i32p), N.ptr(jo, N.i32p), N.ptr(jr, N.i32p),
                                         N.ptr(nf, N.i32p), N.ptr(nl, N.i32p), N.ptr(keys, N.u64p), N.ptr(ms, N.f64p))
        N.check(self.ctx, rc, "px_search_download")
        ids = np.zeros(max(nm, 1), dtype=np.int32)
        self.lib.px_model_ids(self.ctx, N.ptr(ids, N.i32p))
        out = StageOutputs(ref, regT, jo, jr, it, fl, nl,
                           dict(zip(("render", "refine", "rerender", "cost"), (float(x) for x in ms))))
        out.n_first = nf
        out.best_keys = {int(i): int(k) for i, k in zip(ids[:nm], keys[:nm])}
        return out

    # -- multi-GPU (include/px.h: px_comm_*, px_search_reduce) ---------------------------
    @staticmethod
    def nccl_library() -> bytes | None:
        """Path of the NCCL shared library torch ships (site-packages/nvidia/nccl/lib), or None to let
        libpx pick the copy already mapped into the process / the loader path."""
        import importlib.util
        import os

        env = os.environ.get("PX_NCCL_LIB")
        if env:
            return env.encode()
        try:
            spec = importlib.util.find_spec("nvidia.nccl")
        except (ImportError, ValueError):
            spec = None
        for base in (list(spec.submodule_search_locations) if spec and spec.submodule_search_locations else []):
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                return cand.encode()
        return None

    def comm_init(self, rank: int, world: int, unique_id: np.ndarray):
        uid = np.ascontiguousarray(unique_id, dtype=np.uint8)
        assert uid.shape == (128,)
        rc = self.lib.px_comm_init(self.ctx, self.nccl_library(), N.ptr(uid, N.u8p), int(rank), int(world))
        N.check(self.ctx, rc, "px_comm_init")

    def comm_unique_id(self) -> np.ndarray:
        uid = np.zeros(128, dtype=np.uint8)
        N.check(self.ctx, self.lib.px_comm_unique_id(self.ctx, self.nccl_library(), N.ptr(uid, N.u8p)), "px_comm_unique_id")
        return uid

    def comm_init_torch(self):
        """Join the ranks of the initialised torch.distributed group in libpx's own NCCL communicator: rank 0
        creates the unique id, torch.distributed (the plumbing) broadcasts it, every rank calls px_comm_init."""
        import torch
        import torch.distributed as dist

        rank, world = dist.get_rank(), dist.get_world_size()
        uid = self.comm_unique_id() if rank == 0 else np.zeros(128, dtype=np.uint8)
        t = torch.from_numpy(uid)
        if dist.get_backend() == "nccl":
            t = t.to(torch.device("cuda", self.device))
        dist.broadcast(t, src=0)
        self.comm_init(rank, world, t.cpu().numpy())

    def comm_world(self) -> int:
        r, w, v = C.c_int32(0), C.c_int32(1), C.c_int32(0)
        N.check(self.ctx, self.lib.px_comm_info(self.ctx, C.byref(r), C.byref(w), C.byref(v)), "px_comm_info")
        return int(w.value)

    def nccl_version(self) -> int:
        r, w, v = C.c_int32(0), C.c_int32(1), C.c_int32(0)
        N.check(self.ctx, self.lib.px_comm_info(self.ctx, C.byref(r), C.byref(w), C.byref(v)), "px_comm_info")
        return int(v.value)

    def search_reduce(self):
        """Enqueue the argmin all-reduce + winner extraction behind the last search_run (no host sync)."""
        N.check(self.ctx, self.lib.px_search_reduce(self.ctx), "px_search_reduce")

    def search_winners(self) -> dict:
        """{object_id: (key, refined (3,4), reg_T (3,4), j_o, j_r, max_points)} for every model with a
        candidate on any rank."""
        nm = int(self.lib.px_model_count(self.ctx))
        keys = np.zeros(max(nm, 1), dtype=np.uint64)
        ref, reg = np.zeros((max(nm, 1), 3, 4)), np.zeros((max(nm, 1), 3, 4))
        jo, jr, mp = (np.zeros(max(nm, 1), dtype=np.int32) for _ in range(3))
        rc = self.lib.px_search_winners(self.ctx, N.ptr(keys, N.u64p), N.ptr(ref, N.f64p), N.ptr(reg, N.f64p),
                                        N.ptr(jo, N.i32p), N.ptr(jr, N.i32p), N.ptr(mp, N.i32p))
        N.check(self.ctx, rc, "px_search_winners")
        ids = np.zeros(max(nm, 1), dtype=np.int32)
        self.lib.px_model_ids(self.ctx, N.ptr(ids, N.i32p))
        no_key = np.uint64(0xFFFFFFFFFFFFFFFF)
        return {int(ids[s]): (int(keys[s]), ref[s].copy(), reg[s].copy(), int(jo[s]), int(jr[s]), int(mp[s]))
                for s in range(nm) if keys[s] != no_key}

    def stage_millis(self) -> dict:
        ms = np.zeros(4)
        rc = self.lib.px_search_download(self.ctx, None, None, None, None, None, None, None, None, None, N.ptr(ms, N.f64p))
        N.check(self.ctx, rc, "px_search_download")
        return dict(zip(("render", "refine", "rerender", "cost"), (float(x) for x in ms)))

    def knife_edges(self) -> dict:
        """How close any gate decision of the last search came to its threshold."""
        m = np.zeros(2)
        N.check(self.ctx, self.lib.px_search_knife_edges(self.ctx, N.ptr(m, N.f64p)), "px_search_knife_edges")
        return {"min_abs_d2_minus_delta2": float(m[0]), "min_abs_dE_minus_tau_c": float(m[1])}

    def search_stats(self, n):
        nc, nm, nfp = (np.zeros(n, dtype=np.int32) for _ in range(3))
        c0, c1 = np.zeros(n, dtype=np.int64), np.zeros(n, dtype=np.int64)
        rc = self.lib.px_search_stats(self.ctx, N.ptr(nc, N.i32p), N.ptr(c0, N.i64p), N.ptr(c1, N.i64p),
                                      N.ptr(nm, N.i32p), N.ptr(nfp, N.i32p))
        N.check(self.ctx, rc, "px_search_stats")
        return nc, c0, c1, nm, nfp

    # gicp_step_kernel = linearise + solve + step halving fused (the default build); a -DPX_GICP_SPLIT build runs
    # gicp_lin_kernel (+ solve) and gicp_halve_kernel instead and reports them in the third / fourth slot
    KERNELS = ("gicp_init_kernel", "gicp_nn_kernel", "gicp_step_kernel", "gicp_halve_kernel", "gicp_finish_kernel")

    def set_kernel_timing(self, on: bool):
        N.check(self.ctx, self.lib.px_ctx_set_kernel_timing(self.ctx, int(on)), "px_ctx_set_kernel_timing")

    def kernel_ms(self):
        """{kernel: (total ms, launches)} of the refine stage of the last search_run."""
        ms, nl = np.zeros(5, dtype=np.float64), np.zeros(5, dtype=np.int64)
        N.check(self.ctx, self.lib.px_search_kernel_ms(self.ctx, N.ptr(ms, N.f64p), N.ptr(nl, N.i64p)), "px_search_kernel_ms")
        return {k: (float(m), int(c)) for k, m, c in zip(self.KERNELS, ms, nl)}

    def prepare_plan(self, frame, models, plan):
        self.upload_scene(frame, plan.cfg.stride, plan.observed, plan.obs_labels)
        self.upload_models({oid: models[oid] for oid in plan.active})
        if plan.cfg.refine and plan.target_offsets is not None:
            self.upload_targets(plan.target_offsets, plan.target_points, plan.cfg.gicp, plan.target_obs_index)
        elif plan.cfg.refine and plan.target_idx is not None:
            self.build_targets(plan)

    def run_plan(self, frame, models, plan, index=None):
        """Scene/model/target upload + fused search for the plan's candidates."""
        self.prepare_plan(frame, models, plan)
        n = self.search_upload(plan, index)
        self.search_run(self.search_cfg(plan))
        return self.search_download(n)


_default = None


def default_engine() -> Engine:
    """Process-wide engine on the current device (LOCAL_RANK under torchrun)."""
    global _default
    if _default is None:
        import os

        _default = Engine(int(os.environ.get("LOCAL_RANK", "0")))
    return _default
