"""CPU-side checks of the C ABI: the library loads, exports every entry
include/fasttrack_b200.h declares, and validates arguments without a GPU."""

import ctypes
import re
from pathlib import Path

import pytest

from paper_2509_10757_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "fasttrack_b200.h"


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(ft_\w+)\s*\(", text, re.M)))


def test_header_declares_entries():
    names = declared_functions()
    for must in ("ft_stereo_pinhole", "ft_stereo_fisheye_bf", "ft_project_search",
                 "ft_resolve_conflicts", "ft_rotation_filter", "ft_workspace_bytes",
                 "ft_workspace_init", "ft_hamming_pairs"):
        assert must in names


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    for name in declared_functions():
        assert hasattr(L, name), name
    assert set(_lib.EXPORTS) <= set(declared_functions())


def test_abi_version_and_status_strings():
    L = _lib.load()
    assert L.ft_abi_version() == 1
    assert L.ft_status_string(0) == b"ok"
    assert b"NULL" in L.ft_status_string(-1)


def test_workspace_sizing_monotone():
    L = _lib.load()
    a = L.ft_workspace_bytes(1, 1024, 1024)
    b = L.ft_workspace_bytes(1, 2048, 1024)
    c = L.ft_workspace_bytes(4, 2048, 8192)
    assert 0 < a < b < c
    assert L.ft_workspace_bytes(0, 1024, 1024) == 0


def test_argument_validation_without_gpu():
    """Null / range errors are returned before any CUDA call."""
    L = _lib.load()
    kp = _lib.FtKeypoints()
    kp.cap = 0
    params = _lib.FtStereoParams()
    out = _lib.FtStereoOut()
    ws = _lib.FtWorkspace()
    assert L.ft_stereo_pinhole(1, None, None, None, None, None, 0, None, None, None) == -1
    assert L.ft_stereo_pinhole(1, kp, kp, None, None, params, 1, out, ws, None) == -2
    assert L.ft_stereo_fisheye_bf(1, kp, kp, 100, 0.8, None, None, ws, None) == -1
    assert L.ft_resolve_conflicts(0, None, None, None, 0, None, None, None) == -1
    assert L.ft_rotation_filter(0, None, None, None, None, None, None, 0, 1,
                                ctypes.byref(ctypes.c_int32()), None) == -4


def test_new_entries_validate_without_gpu():
    """Entries added with the resident map, the fisheye triangulation, the
    pyramid build and the native runner reject bad arguments before any CUDA
    call."""
    L = _lib.load()
    kp = _lib.FtKeypoints()
    ws = _lib.FtWorkspace()
    # ft_stereo_fisheye: missing triangulation terms / outputs
    assert L.ft_stereo_fisheye(1, kp, kp, 100, 0.8, None, None, None, None, None, ws, None) == -1
    tri = _lib.FtFisheyeTri()
    assert L.ft_stereo_fisheye(1, kp, kp, 100, 0.8, tri, None, None, None, None, ws, None) == -4
    tri.fx = tri.fy = 190.0
    assert L.ft_stereo_fisheye(1, kp, kp, 100, 0.8, tri, None, None, None, None, ws, None) == -1
    # map table gather / scatter
    assert L.ft_gather_points(1, None, 10, None, None, 4, None, None, None) == -1
    assert L.ft_scatter_points(0, None, None, None, 10, None) == 0  # empty delta: no-op
    assert L.ft_scatter_points(3, None, None, None, 10, None) == -1
    # packed-upload scatter
    assert L.ft_copy_ranges(None, None, 1, None) == -1
    assert L.ft_copy_ranges(ctypes.c_void_p(16), None, 0, None) == 0  # nothing to place
    assert L.ft_copy_ranges(ctypes.c_void_p(16), ctypes.c_void_p(16), -1, None) == -2
    # pyramid build
    assert L.ft_build_pyramids(1, None, None, 0, ws, None) == -1
    # native runner
    vp2 = ctypes.c_void_p * 2
    out = ctypes.c_void_p()
    assert L.ft_runner_create(vp2(None, None), vp2(None, None), 16, vp2(None, None),
                              vp2(None, None), 16, ctypes.byref(out)) == -1
    assert L.ft_runner_submit(None, 0, None) == -1
    assert L.ft_runner_submit_range(None, 0, None, 0, 0) == -1
    assert L.ft_runner_submit_ranges(None, 0, None, None, 0) == -1
    assert L.ft_runner_submit_batch(None, 0, 2, None, 0, None, 0) == -1
    assert L.ft_runner_wait(None, 0) == -1
    assert L.ft_runner_destroy(None) == 0
    # persistent runner / plans / resident ring
    assert L.ft_runner_create_persistent(2, None, None, 16, None, None, 16,
                                         ctypes.byref(out)) == -1
    assert L.ft_runner_create_persistent(1, vp2(None, None), vp2(None, None), 16,
                                         vp2(None, None), vp2(None, None), 16,
                                         ctypes.byref(out)) == -2  # needs >= 2 slots
    assert L.ft_track_plan_bytes() > 0
    buf = (ctypes.c_ubyte * 16)()
    assert L.ft_track_plan(1, kp, kp, None, None, None, 0, None, None, None, None, 0, None,
                           ws, None, 0) == -1  # no plan buffer
    assert L.ft_track_plan(1, kp, kp, None, None, None, 0, None, None, None, None, 0, None,
                           ws, buf, 16) == -2  # plan buffer too small
    assert L.ft_track_frames_ring(1, None, 1, None) == -1
    assert L.ft_track_frames_ring(0, vp2(None, None), 1, None) == -2
    assert L.ft_track_frames_ring(1, vp2(None, None), -1, None) == -2


def test_session_entries_validate_without_gpu():
    """The host-array session entries (csrc/ft_session.cu) reject missing
    arguments before any CUDA call; creating a session needs a device."""
    from paper_2509_10757_b200 import session as S
    L = _lib.load()
    S._bind(L)
    f = S.FtHostFeatures()
    assert L.ft_session_destroy(None) == 0
    assert L.ft_session_stereo(None, f, f, None, None, _lib.FtStereoParams(), 1, None, None,
                               None) == -1
    assert L.ft_session_project(None, S.FtHostPoints(), None, 0, None, f, _lib.FtProjectParams(),
                                None, None, None, None, None, 1, S.FtHostProjectOut()) == -1
    assert L.ft_session_fisheye(None, f, f, 100, 0.8, None, None, None, None, None) == -1
    import torch
    if not torch.cuda.is_available():
        h = ctypes.c_void_p()
        assert L.ft_session_create(0, ctypes.byref(h)) > 0  # a cudaError_t: no device


def test_host_packers_match_numpy_layout():
    """ft_host_pack_keypoints / ft_host_pack_points (C loops, no GPU) write
    exactly the include/fasttrack_b200.h record layout."""
    import numpy as np
    import golden_io as G
    from paper_2509_10757_b200.runtime import fill_kp_records, fill_point_records
    d = G.load("cfg2_frame_map.npz")
    left, pts = G.feats(d, "left"), G.soa(d)
    n, m = len(left.u), len(pts.point_ids)
    rec = np.zeros(n + 3, _lib.KP_RECORD)
    fill_kp_records(rec, left, with_angle=True)
    want = np.zeros(n, _lib.KP_RECORD)
    want["u"], want["v"], want["desc"] = left.u, left.v, left.descriptors
    want["angle"], want["octave"] = left.angle, left.octave
    assert rec[:n].tobytes() == want.tobytes()
    prec = np.zeros(m, _lib.POINT_RECORD)
    fill_point_records(prec, pts)
    pw = np.zeros(m, _lib.POINT_RECORD)
    pw["desc"], pw["pos"], pw["nrm"] = pts.descriptors, pts.positions, pts.normals
    pw["min_dist"], pw["max_dist"], pw["id"] = pts.min_distances, pts.max_distances, pts.point_ids
    assert prec.tobytes() == pw.tobytes()
