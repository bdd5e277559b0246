"""ctypes wrapper around oracle/liborc.so (px_oracle.c).

TEST INFRASTRUCTURE, NOT PRODUCT.  It takes the same prepared inputs the device
engine takes (a `SearchPlan`, boundary dataclasses) so that the two can be
compared on identical operands; the arithmetic lives in px_oracle.c, which
restates the reference (each C function cites the reference file:line).
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB = None

f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)

FAILURES = (None, "too_few_points", "degenerate_correspondences", "singular_normal_equations",
            "no_decrease")


class Scene(C.Structure):
    _fields_ = [("H", C.c_int32), ("W", C.c_int32), ("stride", C.c_int32), ("pad_", C.c_int32),
                ("depth", f64p), ("valid", u8p), ("labels", i32p),
                ("fx", C.c_double), ("fy", C.c_double), ("cx", C.c_double), ("cy", C.c_double),
                ("n_obs", C.c_int64), ("obs_pts", f64p), ("obs_lab", f64p), ("obs_labels", i32p)]


class Model(C.Structure):
    _fields_ = [("object_id", C.c_int32), ("V", C.c_int32), ("T", C.c_int32), ("pad_", C.c_int32),
                ("verts", f64p), ("col_lin", f64p), ("tris", i32p),
                ("cyl_r2", C.c_double), ("cyl_zmin", C.c_double), ("cyl_zmax", C.c_double)]


class GicpCfg(C.Structure):
    _fields_ = [("k_cov", C.c_int32), ("max_iter", C.c_int32), ("eps", C.c_double),
                ("tol_t", C.c_double), ("tol_r", C.c_double), ("gate", C.c_double)]


class SearchCfg(C.Structure):
    _fields_ = [("mode3dof", C.c_int32), ("use_color", C.c_int32), ("occluder_marking", C.c_int32),
                ("refine", C.c_int32), ("delta", C.c_double), ("tau_c", C.c_double), ("gicp", GicpCfg),
                ("c2w", C.c_double * 12), ("w2c", C.c_double * 12),
                ("c2w_vec_order", C.c_int32), ("w2c_vec_order", C.c_int32), ("fixed_z", C.c_double),
                ("n_threads", C.c_int32), ("cloud_cap", C.c_int32)]


def build(force: bool = False) -> Path:
    so = _HERE / "liborc.so"
    src = _HERE / "px_oracle.c"
    if force or not so.exists() or so.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-C", os.fspath(_HERE), "-B", "liborc.so"], check=True,
                       stdout=subprocess.DEVNULL)
    return so


def lib():
    global _LIB
    if _LIB is None:
        L = C.CDLL(os.fspath(build()))
        L.orc_ciede2000.restype = C.c_double
        L.orc_ciede2000.argtypes = [f64p, f64p]
        L.orc_gicp_linearize.restype = C.c_double
        L.orc_rms_residual.restype = C.c_double
        L.orc_rms_residual.argtypes = [f64p, C.c_int64, f64p, C.c_int64, f64p, C.c_double]
        _LIB = L
    return _LIB


def _f(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a, t=f64p):
    return None if a is None else a.ctypes.data_as(t)


def _gicp_cfg(cfg) -> GicpCfg:
    return GicpCfg(cfg.k_covariance, cfg.max_iterations, cfg.epsilon, cfg.translation_tolerance,
                   cfg.rotation_tolerance, cfg.max_correspondence_distance)


class OracleScene:
    """Keeps the numpy operands alive behind an `orc_scene`."""

    def __init__(self, frame, stride, observed, obs_labels):
        k = frame.intrinsics
        self.depth = _f(frame.depth.values)
        self.valid = np.ascontiguousarray(frame.depth.valid, dtype=np.uint8)
        self.labels = np.ascontiguousarray(frame.labels, dtype=np.int32)
        self.obs_pts, self.obs_lab = _f(observed.points), _f(observed.lab_colors)
        self.obs_labels = np.ascontiguousarray(obs_labels, dtype=np.int32)
        self.c = Scene(k.height, k.width, stride, 0, _p(self.depth), _p(self.valid, u8p), _p(self.labels, i32p),
                       k.fx, k.fy, k.cx, k.cy, self.obs_pts.shape[0], _p(self.obs_pts), _p(self.obs_lab),
                       _p(self.obs_labels, i32p))
        self.cap = ((k.height + stride - 1) // stride) * ((k.width + stride - 1) // stride)


class OracleModel:
    def __init__(self, object_id, mesh, cylinder=None):
        from paper_2008_00326_b200.colorspace import srgb_decode  # host-side operand prep, shared input

        self.verts = _f(mesh.vertices)
        self.col = _f(srgb_decode(mesh.vertex_colors))
        self.tris = np.ascontiguousarray(mesh.triangles, dtype=np.int32)
        r2, z0, z1 = (1.0, 0.0, 1.0) if cylinder is None else (cylinder.radius**2, cylinder.z_min, cylinder.z_max)
        self.c = Model(int(object_id), self.verts.shape[0], self.tris.shape[0], 0, _p(self.verts), _p(self.col),
                       _p(self.tris, i32p), r2, z0, z1)


def pose3x4(t) -> np.ndarray:
    m = np.empty((3, 4))
    m[:, :3] = t.rotation
    m[:, 3] = t.translation
    return m


def rasterize(model: OracleModel, pose, k):
    h, w = k.height, k.width
    z, c = np.empty((h, w)), np.empty((h, w, 3))
    v, o = np.empty((h, w), dtype=np.uint8), np.empty((h, w), dtype=np.int32)
    p = _f(pose)
    lib().orc_rasterize(C.byref(model.c), _p(p), C.c_double(k.fx), C.c_double(k.fy), C.c_double(k.cx),
                        C.c_double(k.cy), k.width, k.height, _p(z), _p(c), _p(v, u8p), _p(o, i32p))
    return z, c, v.astype(bool), o


def render_one(scene: OracleScene, model: OracleModel, pose, occluder_marking=True, delta_occ=0.0075):
    cap = scene.cap
    pts, lab = np.empty((cap, 3)), np.empty((cap, 3))
    src = np.empty((cap, 2), dtype=np.int32)
    p = _f(pose)
    n = lib().orc_render_one(C.byref(scene.c), C.byref(model.c), _p(p), int(bool(occluder_marking)),
                             C.c_double(delta_occ), _p(pts), _p(lab), _p(src, i32p), cap)
    assert n >= 0
    return pts[:n].copy(), lab[:n].copy(), src[:n].copy()


def knn(q, t, k):
    q, t = _f(q).reshape(-1, 3), _f(t).reshape(-1, 3)
    idx = np.empty((q.shape[0], k), dtype=np.int64)
    d2 = np.empty((q.shape[0], k))
    lib().orc_knn(_p(q), C.c_int64(q.shape[0]), _p(t), C.c_int64(t.shape[0]), k, _p(idx, i64p), _p(d2))
    return idx, d2


def covariances(pts, k=20, eps=1e-3):
    pts = _f(pts)
    out = np.empty((pts.shape[0], 3, 3))
    lib().orc_covariances(_p(pts), C.c_int64(pts.shape[0]), int(k), C.c_double(eps), _p(out))
    return out


def gicp_linearize(src, tgt, ca, cb, r, t, gate2):
    src, tgt, ca, cb, r, t = (_f(x) for x in (src, tgt, ca, cb, r, t))
    n = src.shape[0]
    h, g = np.zeros((6, 6)), np.zeros(6)
    corr = np.empty(n, dtype=np.int64)
    w = np.zeros((n, 3, 3))
    nc = C.c_int64(0)
    f0 = lib().orc_gicp_linearize(_p(src), C.c_int64(n), _p(tgt), C.c_int64(tgt.shape[0]), _p(ca), _p(cb), _p(r),
                                  _p(t), C.c_double(gate2), _p(h), _p(g), _p(corr, i64p), _p(w), C.byref(nc))
    return f0, int(nc.value), h, g, corr, w


def gicp_align(src, tgt, ca, cb, init3x4, cfg):
    """-> (T 3x4, iterations, converged, failure, trace, r_raw)"""
    src, tgt, ca, cb, init = (_f(x) for x in (src, tgt, ca, cb, init3x4))
    T = np.empty((3, 4))
    it, conv, ntr = C.c_int32(0), C.c_int32(0), C.c_int32(0)
    trace = np.zeros((max(cfg.max_iterations, 1), 2))
    rraw = np.empty((3, 3))
    g = _gicp_cfg(cfg)
    code = lib().orc_gicp_align(_p(src), C.c_int64(src.shape[0]), _p(tgt), C.c_int64(tgt.shape[0]), _p(ca), _p(cb),
                                _p(init), C.byref(g), _p(T), C.byref(it), C.byref(conv), _p(trace), C.byref(ntr),
                                _p(rraw))
    return T, int(it.value), bool(conv.value), FAILURES[code], trace[:ntr.value].copy(), rraw


def rms_residual(src, tgt, T, gate):
    src, tgt, T = _f(src), _f(tgt), _f(T)
    return float(lib().orc_rms_residual(_p(src), src.shape[0], _p(tgt), tgt.shape[0], _p(T), gate))


def refine_apply(reg_T, cam_in, mode3dof, c2w, c2w_order, w2c, w2c_order, fixed_z):
    out = np.empty((3, 4))
    a, b, c, d = _f(reg_T), _f(cam_in), _f(c2w), _f(w2c)
    lib().orc_refine_apply(_p(a), _p(b), int(mode3dof), _p(c), int(c2w_order), _p(d), int(w2c_order),
                           C.c_double(fixed_z), _p(out))
    return out


def rendered_cost(rp, rlab, op, olab, delta, tau_c, use_color):
    rp, rlab, op, olab = (_f(x).reshape(-1, 3) for x in (rp, rlab, op, olab))
    ex = np.zeros(op.shape[0], dtype=np.uint8)
    lib().orc_rendered_cost.restype = C.c_int
    jr = lib().orc_rendered_cost(_p(rp), _p(rlab), rp.shape[0], _p(op), _p(olab), C.c_int64(op.shape[0]),
                                 C.c_double(delta), C.c_double(tau_c), int(bool(use_color)), _p(ex, u8p))
    return int(jr), ex.astype(bool)


def observed_cost_cyl(op, pose3x4_, r2, zmin, zmax, explained):
    op, P = _f(op).reshape(-1, 3), _f(pose3x4_)
    ex = np.ascontiguousarray(explained, dtype=np.uint8)
    sel = np.zeros(op.shape[0], dtype=np.uint8)
    jo = lib().orc_observed_cost_cyl(_p(op), C.c_int64(op.shape[0]), _p(P), C.c_double(r2), C.c_double(zmin),
                                     C.c_double(zmax), _p(ex, u8p), _p(sel, u8p))
    return int(jo), sel.astype(bool)


def srgb_to_lab(rgb):
    rgb = _f(rgb).reshape(-1, 3)
    out = np.empty_like(rgb)
    lib().orc_srgb_to_lab(_p(rgb), C.c_int64(rgb.shape[0]), _p(out))
    return out


def ciede2000(a, b):
    a, b = _f(a), _f(b)
    return float(lib().orc_ciede2000(_p(a), _p(b)))


def run_plan(frame, models, plan, n_threads=None, index=None):
    """Per-candidate stages of estimate_poses on the CPU for the plan's
    candidates (search.py:268-336) -> StageOutputs (+ .n_first, .stage_seconds)."""
    from paper_2008_00326_b200.search import StageOutputs

    cfg = plan.cfg
    scene = OracleScene(frame, cfg.stride, plan.observed, plan.obs_labels)
    slot_of = {oid: i for i, oid in enumerate(plan.active)}
    oms = [OracleModel(oid, models[oid].mesh, models[oid].inscribed_cylinder) for oid in plan.active]
    marr = (Model * max(len(oms), 1))(*[m.c for m in oms])
    flat_oid, poses, tidx = plan.flat_oid, plan.cam_poses, plan.target_idx
    if index is not None:
        flat_oid, poses = flat_oid[index], poses[index]
        tidx = None if tidx is None else tidx[index]
    n = flat_oid.shape[0]
    slots = np.array([slot_of[int(o)] for o in flat_oid], dtype=np.int32)
    poses = _f(poses)
    sc = SearchCfg()
    sc.mode3dof = int(cfg.mode == "3dof")
    sc.use_color, sc.occluder_marking, sc.refine = int(cfg.use_color), int(cfg.occluder_marking), int(cfg.refine)
    sc.delta, sc.tau_c, sc.gicp = cfg.delta, cfg.tau_c, _gicp_cfg(cfg.gicp)
    sc.c2w[:] = list(np.asarray(plan.c2w).reshape(-1))
    sc.w2c[:] = list(np.asarray(plan.w2c).reshape(-1))
    sc.c2w_vec_order, sc.w2c_vec_order, sc.fixed_z = plan.c2w_vec_order, plan.w2c_vec_order, cfg.fixed_z
    sc.n_threads = int(n_threads or os.cpu_count() or 1)
    sc.cloud_cap = scene.cap
    if cfg.refine and plan.target_offsets is not None:
        # only targets referenced by these candidates get covariances (m2m_gicp
        # builds them per distinct target of the call, registration.py:533-540)
        used = np.unique(tidx)
        remap = np.full(plan.target_offsets.shape[0] - 1, -1, dtype=np.int32)
        remap[used] = np.arange(used.size, dtype=np.int32)
        sizes = np.diff(plan.target_offsets)[used]
        toff = np.zeros(used.size + 1, dtype=np.int64)
        np.cumsum(sizes, out=toff[1:])
        if used.size == remap.size:
            tpts = _f(plan.target_points)
        else:
            tpts = _f(np.concatenate([plan.target_points[plan.target_offsets[t]:plan.target_offsets[t + 1]]
                                      for t in used])) if used.size else np.zeros((0, 3))
        tix = np.ascontiguousarray(remap[tidx], dtype=np.int32)
        ntg = used.size
    else:
        toff, tpts, tix, ntg = np.zeros(1, dtype=np.int64), np.zeros((0, 3)), np.zeros(max(n, 1), dtype=np.int32), 0
    refined, regT = np.empty((n, 3, 4)), np.empty((n, 3, 4))
    it, fl, jo, jr, nf, nl = (np.zeros(n, dtype=np.int32) for _ in range(6))
    st = np.zeros(5)
    lib().orc_search(C.byref(scene.c), marr, C.c_int64(n), _p(slots, i32p), _p(poses), ntg, _p(toff, i64p), _p(tpts),
                     _p(tix, i32p), C.byref(sc), _p(refined), _p(regT), _p(it, i32p), _p(fl, i32p), _p(jo, i32p),
                     _p(jr, i32p), _p(nf, i32p), _p(nl, i32p), _p(st))
    if (fl < 0).any():
        raise RuntimeError("oracle cloud capacity overflow")
    nth = sc.n_threads
    out = StageOutputs(refined, regT, jo, jr, it, fl, nl,
                       {"render": st[0] / nth * 1e3, "refine": (st[1] / nth + st[4]) * 1e3,
                        "rerender": st[2] / nth * 1e3, "cost": st[3] / nth * 1e3})
    out.n_first = nf
    return out
