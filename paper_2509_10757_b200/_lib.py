"""ctypes binding of libfasttrack_b200.so (the C ABI in include/fasttrack_b200.h).

The library is built in-tree by ``build()`` (nvcc, sm_100a).  There is no CPU
fallback: if the shared object is missing or a call fails, this module raises.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libfasttrack_b200.so"
CSRC = PKG / "csrc"

FT_MAX_LEVELS = 16
FT_STEREO_PHASE1 = 0x1
FT_STEREO_REFINE = 0x2
FT_STEREO_FROM_CAND = 0x4
FT_STEREO_REJECT = 0x8
FT_PROJ_RESOLVE = 0x1
FT_PROJ_ROTATION = 0x2
FT_PROJ_SKIP_SLOTS = 0x4
FT_PROJ_WRITE_SLOTS = 0x8

vp = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
f64 = ctypes.c_double


class FtWorkspace(ctypes.Structure):
    _fields_ = [("base", vp), ("bytes", ctypes.c_size_t), ("n_frames", i32), ("cap_left", i32),
                ("cap_points", i32)]


class FtKeypoints(ctypes.Structure):
    _fields_ = [("rec", vp), ("count", vp), ("cap", i32)]


class FtPyramid(ctypes.Structure):
    _fields_ = [("data", vp), ("frame_bytes", i64), ("n_levels", i32),
                ("offsets", i64 * FT_MAX_LEVELS), ("widths", i32 * FT_MAX_LEVELS),
                ("heights", i32 * FT_MAX_LEVELS)]


class FtStereoParams(ctypes.Structure):
    _fields_ = [("t_match", i32), ("band_factor", f64), ("min_disparity", f64),
                ("max_disparity", f64), ("half_window", i32), ("half_slide", i32),
                ("outlier_multiplier", f64), ("ratio", f64), ("baseline_times_fx", f64),
                ("height", i32), ("n_levels", i32), ("scale_pow", f64 * FT_MAX_LEVELS)]


class FtStereoOut(ctypes.Structure):
    _fields_ = [("cand_idx", vp), ("cand_dist", vp), ("right_idx", vp), ("distance", vp),
                ("disparity", vp), ("refined_u", vp), ("depth", vp), ("sad", vp),
                ("n_matched", vp)]


class FtMapPoints(ctypes.Structure):
    _fields_ = [("rec", vp), ("count", vp), ("cap", i32), ("index", vp)]


# numpy views of the packed records (include/fasttrack_b200.h)
import numpy as _np  # noqa: E402

KP_RECORD = _np.dtype([("u", "<f8"), ("v", "<f8"), ("desc", "<u8", (4,)), ("angle", "<f8"),
                       ("octave", "<i4"), ("pad", "<i4")])
POINT_RECORD = _np.dtype([("desc", "<u8", (4,)), ("pos", "<f8", (3,)), ("nrm", "<f8", (3,)),
                          ("min_dist", "<f8"), ("max_dist", "<f8"), ("id", "<i8"),
                          ("pad", "<i8")])
assert KP_RECORD.itemsize == 64 and POINT_RECORD.itemsize == 112


class FtProjectParams(ctypes.Structure):
    _fields_ = [("cam_kind", i32), ("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64),
                ("k1", f64), ("k2", f64), ("k3", f64), ("k4", f64), ("width", f64),
                ("height", f64), ("cell_px", i32), ("grid_nx", i32), ("grid_ny", i32),
                ("n_levels", i32), ("scale_pow", f64 * FT_MAX_LEVELS), ("inv_log_scale", f64),
                ("window_px", f64), ("t_proj", i32), ("ratio", f64), ("view_cos_min", f64),
                ("u_offset", f64), ("histogram_bins", i32), ("histogram_keep", i32)]


class FtProjectIO(ctypes.Structure):
    _fields_ = [("rot", vp), ("trans", vp), ("skip", vp), ("ref_angles", vp), ("slots_in", vp),
                ("slots_out", vp)]


class FtProjectOut(ctypes.Structure):
    _fields_ = [("out_kp", vp), ("out_dist", vp), ("out_oct", vp), ("corr_point", vp),
                ("corr_kp", vp), ("corr_dist", vp), ("corr_oct", vp), ("corr_count", vp),
                ("slot_count", vp)]


class FtFisheyeTri(ctypes.Structure):
    _fields_ = [("fx", f64), ("fy", f64), ("cx", f64), ("cy", f64), ("k1", f64), ("k2", f64),
                ("k3", f64), ("k4", f64), ("rot_rl", f64 * 9), ("trans_rl", f64 * 3),
                ("rot_lr", f64 * 9), ("trans_lr", f64 * 3), ("ray_gap_ceiling", f64),
                ("corrected", i32)]


class FtError(RuntimeError):
    """A C-ABI call returned a non-zero status."""


_lib = None

EXPORTS = ("ft_abi_version", "ft_status_string", "ft_workspace_bytes", "ft_workspace_init",
           "ft_hamming_pairs", "ft_stereo_pinhole", "ft_stereo_fisheye_bf", "ft_project_search",
           "ft_track_frames", "ft_resolve_conflicts", "ft_rotation_filter", "ft_bench_popc",
           "ft_pack_keypoints", "ft_pack_points", "ft_build_pyramids", "ft_stereo_fisheye",
           "ft_gather_points", "ft_scatter_points", "ft_copy_ranges", "ft_runner_create", "ft_runner_create_n", "ft_runner_submit", "ft_runner_submit_range", "ft_runner_submit_ranges", "ft_runner_submit_batch",
           "ft_runner_wait", "ft_runner_destroy", "ft_runner_create_persistent",
           "ft_track_plan", "ft_track_plan_groups", "ft_track_plan_bytes", "ft_track_frames_ring", "ft_session_create",
           "ft_session_destroy", "ft_session_stats", "ft_session_stereo", "ft_session_project", "ft_session_fisheye",
           "ft_host_pack_keypoints", "ft_host_pack_points", "ft_update_local_map",
           "ft_session_update_local_map")


def build(force: bool = False) -> Path:
    """Compile the CUDA sources into LIB_PATH (nvcc, -gencode sm_100a)."""
    (PKG.parent / "build").mkdir(exist_ok=True)
    if force and LIB_PATH.exists():
        LIB_PATH.unlink()
    subprocess.run(["make", "-s", "-C", str(CSRC)], check=True)
    return LIB_PATH


def load() -> ctypes.CDLL:
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise FtError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(str(LIB_PATH))
    P = ctypes.POINTER
    L.ft_abi_version.restype = ctypes.c_int
    L.ft_status_string.argtypes = [ctypes.c_int]
    L.ft_status_string.restype = ctypes.c_char_p
    L.ft_workspace_bytes.argtypes = [i32, i32, i32]
    L.ft_workspace_bytes.restype = ctypes.c_size_t
    W = P(FtWorkspace)
    L.ft_workspace_init.argtypes = [W, vp]
    L.ft_hamming_pairs.argtypes = [vp, vp, i64, vp, vp]
    L.ft_stereo_pinhole.argtypes = [i32, P(FtKeypoints), P(FtKeypoints), P(FtPyramid),
                                    P(FtPyramid), P(FtStereoParams), i32, P(FtStereoOut), W, vp]
    L.ft_stereo_fisheye_bf.argtypes = [i32, P(FtKeypoints), P(FtKeypoints), i32, f64, vp, vp,
                                       W, vp]
    L.ft_stereo_fisheye.argtypes = [i32, P(FtKeypoints), P(FtKeypoints), i32, f64,
                                    P(FtFisheyeTri), vp, vp, vp, vp, W, vp]
    L.ft_gather_points.argtypes = [i32, vp, i64, vp, vp, i32, vp, vp, vp]
    L.ft_scatter_points.argtypes = [i32, vp, vp, vp, i64, vp]
    L.ft_copy_ranges.argtypes = [vp, vp, i32, vp]
    L.ft_runner_create.argtypes = [vp * 2, vp * 2, ctypes.c_size_t, vp * 2, vp * 2,
                                   ctypes.c_size_t, P(vp)]
    L.ft_runner_create_n.argtypes = [i32, vp, vp, ctypes.c_size_t, vp, vp, ctypes.c_size_t,
                                     P(vp)]
    L.ft_runner_submit.argtypes = [vp, i64, vp]
    L.ft_runner_submit_range.argtypes = [vp, i64, vp, ctypes.c_size_t, ctypes.c_size_t]
    L.ft_runner_submit_ranges.argtypes = [vp, i64, vp, vp, i32]
    L.ft_runner_submit_batch.argtypes = [vp, i64, i32, vp, ctypes.c_size_t, vp, i32]
    L.ft_runner_wait.argtypes = [vp, i64]
    L.ft_runner_destroy.argtypes = [vp]
    L.ft_runner_create_persistent.argtypes = [i32, vp, vp, ctypes.c_size_t, vp, vp,
                                              ctypes.c_size_t, P(vp)]
    L.ft_track_frames_ring.argtypes = [i32, vp, i64, vp]
    L.ft_track_plan_bytes.restype = ctypes.c_size_t
    L.ft_track_plan_bytes.argtypes = []
    L.ft_track_plan.argtypes = [i32, P(FtKeypoints), P(FtKeypoints), P(FtPyramid),
                                P(FtPyramid), P(FtStereoParams), i32, P(FtStereoOut),
                                P(FtMapPoints), P(FtProjectParams), P(FtProjectIO), i32,
                                P(FtProjectOut), W, vp, ctypes.c_size_t]
    L.ft_track_plan_groups.argtypes = [i32, P(FtKeypoints), P(FtKeypoints), P(FtPyramid),
                                       P(FtPyramid), P(FtStereoParams), i32, P(FtStereoOut),
                                       P(FtMapPoints), P(FtProjectParams), P(FtProjectIO), i32,
                                       P(FtProjectOut), W, i32, vp, ctypes.c_size_t]
    L.ft_project_search.argtypes = [i32, P(FtMapPoints), P(FtKeypoints), P(FtProjectParams),
                                    P(FtProjectIO), i32, P(FtProjectOut), W, vp]
    L.ft_track_frames.argtypes = [i32, P(FtKeypoints), P(FtKeypoints), P(FtPyramid),
                                  P(FtPyramid), P(FtStereoParams), i32, P(FtStereoOut),
                                  P(FtMapPoints), P(FtProjectParams), P(FtProjectIO), i32,
                                  P(FtProjectOut), W, vp]
    L.ft_resolve_conflicts.argtypes = [i32, vp, vp, vp, i32, P(FtProjectOut), W, vp]
    L.ft_rotation_filter.argtypes = [i32, vp, vp, vp, vp, vp, vp, i32, i32, vp, vp]
    L.ft_bench_popc.argtypes = [i32, i32, i32, vp, vp]
    L.ft_pack_keypoints.argtypes = [i32, vp, vp, vp, vp, vp, vp, i32, vp, vp]
    L.ft_pack_points.argtypes = [i32, vp, vp, vp, vp, vp, vp, vp, i32, vp, vp]
    L.ft_build_pyramids.argtypes = [i32, P(FtPyramid), vp, i64, W, vp]
    _lib = L
    return L


def check(status: int, what: str) -> None:
    if status != 0:
        msg = load().ft_status_string(status).decode()
        raise FtError(f"{what} failed with status {status}: {msg}")
