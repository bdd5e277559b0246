"""ctypes binding of libpx.so (include/px.h).  No fallback: if the library is
missing or no CUDA device is present, every entry point raises DeviceError."""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

from .errors import DeviceError, UnknownObjectId

_LIB_PATH = Path(__file__).resolve().parent / "libpx.so"
_lib = None

f64p = C.POINTER(C.c_double)
i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
u8p = C.POINTER(C.c_uint8)
u64p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class GicpCfg(C.Structure):
    _fields_ = [("k_covariance", C.c_int32), ("max_iterations", C.c_int32),
                ("epsilon", C.c_double), ("translation_tolerance", C.c_double),
                ("rotation_tolerance", C.c_double), ("max_correspondence_distance", C.c_double)]


class SearchCfg(C.Structure):
    _fields_ = [("mode3dof", C.c_int32), ("use_color", C.c_int32),
                ("occluder_marking", C.c_int32), ("refine", C.c_int32),
                ("delta", C.c_double), ("tau_c", C.c_double), ("gicp", GicpCfg),
                ("cam_to_world", C.c_double * 12), ("world_to_cam", C.c_double * 12),
                ("c2w_vec_order", C.c_int32), ("w2c_vec_order", C.c_int32),
                ("fixed_z", C.c_double)]


class Lattice(C.Structure):
    _fields_ = [("object_id", C.c_int32), ("n_outer", C.c_int32), ("n_inner", C.c_int32),
                ("rotations", f64p), ("translations", f64p), ("capsule", C.c_double * 3)]


_SIGS = {
    "px_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
    "px_ctx_destroy": (None, [vp]),
    "px_last_error": (C.c_char_p, [vp]),
    "px_ctx_set_stream": (C.c_int, [vp, vp]),
    "px_ctx_sync": (C.c_int, [vp]),
    "px_ctx_set_scratch_budget": (C.c_int, [vp, C.c_int64]),
    "px_ctx_launch_count": (C.c_int64, [vp]),
    "px_scene_upload": (C.c_int, [vp, C.c_int32, C.c_int32, f64p, u8p, i32p, f64p, C.c_int32,
                                  f64p, f64p, i32p, i32p, C.c_int64]),
    "px_scene_upload_frame": (C.c_int, [vp, C.c_int32, C.c_int32, f64p, u8p, i32p, f64p, f64p, C.c_int32, i64p]),
    "px_scene_upload_frame_full": (C.c_int, [vp, C.c_int32, C.c_int32, f64p, u8p, i32p, f64p, f64p, C.c_int32, i64p]),
    "px_scene_download_cloud": (C.c_int, [vp, f64p, f64p, i32p, i32p]),
    "px_search_upload_lattice": (C.c_int, [vp, C.c_int32, C.c_int32, C.POINTER(Lattice), f64p, C.c_int32, f64p,
                                           C.POINTER(GicpCfg), C.c_int32, C.c_int32, i64p]),
    "px_search_candidates": (C.c_int, [vp, i32p, f64p, i32p, i32p]),
    "px_model_upload": (C.c_int, [vp, C.c_int32, f64p, f64p, i32p, C.c_int64, C.c_int64, f64p]),
    "px_render_batch": (C.c_int, [vp, i32p, f64p, C.c_int64, C.c_int32, C.c_double, C.POINTER(vp)]),
    "px_clouds_count": (C.c_int64, [vp]),
    "px_clouds_counts": (C.c_int, [vp, vp, i32p]),
    "px_clouds_download": (C.c_int, [vp, vp, f64p, f64p, i32p]),
    "px_clouds_upload": (C.c_int, [vp, C.c_int64, i32p, f64p, f64p, i32p, C.POINTER(vp)]),
    "px_clouds_free": (None, [vp, vp]),
    "px_rasterize": (C.c_int, [vp, C.c_int32, f64p, f64p, f64p, u8p, i32p]),
    "px_covariances": (C.c_int, [vp, f64p, C.c_int64, C.c_int32, C.c_double, f64p]),
    "px_targets_upload": (C.c_int, [vp, C.c_int32, i64p, f64p, i64p, C.POINTER(GicpCfg)]),
    "px_targets_covariances": (C.c_int, [vp, f64p]),
    "px_refine_batch": (C.c_int, [vp, vp, i32p, f64p, C.POINTER(GicpCfg), f64p, i32p, i32p, f64p,
                                  f64p, i32p]),
    "px_gicp_linearize": (C.c_int, [vp, f64p, C.c_int64, f64p, C.c_int64, f64p, C.POINTER(GicpCfg), f64p, f64p, f64p,
                                    i32p, i64p, f64p]),
    "px_ciede2000": (C.c_int, [vp, f64p, f64p, C.c_int64, f64p]),
    "px_srgb_to_lab": (C.c_int, [vp, f64p, C.c_int64, C.c_int32, f64p]),
    "px_cost_batch": (C.c_int, [vp, vp, i32p, f64p, C.c_double, C.c_double, C.c_int32, i32p, i32p]),
    "px_rendered_cost": (C.c_int, [vp, f64p, f64p, C.c_int64, f64p, f64p, C.c_int64, C.c_double,
                                   C.c_double, C.c_int32, i32p, u8p]),
    "px_knn": (C.c_int, [vp, f64p, C.c_int64, f64p, C.c_int64, C.c_int32, i64p, f64p]),
    "px_search_upload": (C.c_int, [vp, C.c_int64, i32p, f64p, i32p, i32p]),
    "px_search_run": (C.c_int, [vp, C.POINTER(SearchCfg)]),
    "px_search_download": (C.c_int, [vp, f64p, f64p, i32p, i32p, i32p, i32p, i32p, i32p, u64p, f64p]),
    "px_search_stats": (C.c_int, [vp, i32p, i64p, i64p, i32p, i32p]),
    "px_targets_build_capsules": (C.c_int, [vp, C.c_int32, f64p, f64p, C.POINTER(GicpCfg)]),
    "px_targets_build_labels": (C.c_int, [vp, C.c_int32, i32p, C.POINTER(GicpCfg)]),
    "px_targets_info": (C.c_int, [vp, i32p, i64p]),
    "px_targets_download": (C.c_int, [vp, i64p, f64p, i32p]),
    "px_ctx_set_kernel_timing": (C.c_int, [vp, C.c_int32]),
    "px_search_kernel_ms": (C.c_int, [vp, f64p, i64p]),
    "px_comm_unique_id": (C.c_int, [vp, C.c_char_p, u8p]),
    "px_comm_init": (C.c_int, [vp, C.c_char_p, u8p, C.c_int32, C.c_int32]),
    "px_comm_destroy": (C.c_int, [vp]),
    "px_comm_info": (C.c_int, [vp, i32p, i32p, i32p]),
    "px_search_reduce": (C.c_int, [vp]),
    "px_search_winners": (C.c_int, [vp, u64p, f64p, f64p, i32p, i32p, i32p]),
    "px_search_knife_edges": (C.c_int, [vp, f64p]),
    "px_model_count": (C.c_int, [vp]),
    "px_model_ids": (C.c_int, [vp, i32p]),
}

EXPORTS = tuple(_SIGS)


def lib_path() -> Path:
    return _LIB_PATH


def load():
    """Load libpx.so; raises DeviceError when it has not been built."""
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            raise DeviceError(f"{_LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (there is no CPU fallback)")
        try:
            lib = C.CDLL(os.fspath(_LIB_PATH))
        except OSError as e:
            raise DeviceError(f"cannot load {_LIB_PATH}: {e}") from e
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype, fn.argtypes = res, args
        _lib = lib
    return _lib


def ptr(a, ctype):
    """Pointer to a C-contiguous numpy array (None -> NULL)."""
    if a is None:
        return None
    return a.ctypes.data_as(ctype)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def check(ctx, rc: int, what: str = ""):
    if rc == 0:
        return
    msg = load().px_last_error(ctx)
    msg = msg.decode() if msg else "unknown error"
    if "no model registered" in msg:
        raise UnknownObjectId(msg)
    raise DeviceError(f"{what or 'libpx'} failed ({rc}): {msg}")
