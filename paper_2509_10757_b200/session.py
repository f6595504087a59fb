"""Host-array drop-in calls through the native session (csrc/ft_session.cu).

Each reference stage function becomes ONE C call that packs the reference
objects' numpy arrays (passed in place, no copies in Python), copies them to
the device, launches the fused kernel, and copies the outputs into numpy
arrays the caller allocated -- the per-call Python work is a few pointer
fields.  One native session (stream, pinned staging, device arena, workspace)
per CUDA device, reused by every call (reference buffers.py:13-55: buffers
reserved once, reused per frame).  No CPU fallback: the session needs the
library and a CUDA device.
"""

from __future__ import annotations

import ctypes
import threading
from functools import lru_cache

import numpy as np

from . import _lib

vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64


class FtHostFeatures(ctypes.Structure):
    _fields_ = [("n", i64), ("u", vp), ("v", vp), ("octave", vp), ("angle", vp), ("desc", vp)]


class FtHostPyramid(ctypes.Structure):
    _fields_ = [("data", vp), ("n_levels", i32), ("offsets", i64 * (_lib.FT_MAX_LEVELS + 1)),
                ("widths", i32 * _lib.FT_MAX_LEVELS), ("heights", i32 * _lib.FT_MAX_LEVELS)]


class FtHostMatches(ctypes.Structure):
    _fields_ = [("right_idx", vp), ("distance", vp), ("disparity", vp), ("refined_u", vp),
                ("depth", vp), ("sad", vp)]


class FtHostPoints(ctypes.Structure):
    _fields_ = [("m", i64), ("positions", vp), ("normals", vp), ("min_dist", vp),
                ("max_dist", vp), ("desc", vp), ("ids", vp)]


class FtHostProjectOut(ctypes.Structure):
    _fields_ = [("out_kp", vp), ("out_dist", vp), ("out_oct", vp), ("corr_point", vp),
                ("corr_kp", vp), ("corr_dist", vp), ("corr_oct", vp), ("corr_count", vp),
                ("slots_out", vp), ("slot_count", vp)]


class FtWorldDev(ctypes.Structure):
    _fields_ = [("kf_obs", vp), ("kf_off", vp), ("n_kf", i32), ("id_slot", vp), ("id_cap", i64)]


_bound = False


def _bind(L) -> None:
    global _bound
    if _bound:
        return
    P = ctypes.POINTER
    L.ft_session_create.argtypes = [i32, P(vp)]
    L.ft_session_destroy.argtypes = [vp]
    L.ft_session_stats.argtypes = [vp, vp, i32]
    L.ft_session_stereo.argtypes = [vp, P(FtHostFeatures), P(FtHostFeatures), P(FtHostPyramid),
                                    P(FtHostPyramid), P(_lib.FtStereoParams), i32, vp, vp,
                                    P(FtHostMatches)]
    L.ft_session_project.argtypes = [vp, P(FtHostPoints), vp, i64, vp, P(FtHostFeatures),
                                     P(_lib.FtProjectParams), vp, vp, vp, vp, vp, i32,
                                     P(FtHostProjectOut)]
    L.ft_session_fisheye.argtypes = [vp, P(FtHostFeatures), P(FtHostFeatures), i32,
                                     ctypes.c_double, P(_lib.FtFisheyeTri), vp, vp, vp, vp]
    L.ft_session_update_local_map.argtypes = [vp, vp, i64, P(FtWorldDev), i64, vp, vp, vp, vp]
    L.ft_update_local_map.argtypes = [vp, i32, vp, vp, i32, vp, i64, vp, vp, vp, vp, vp]
    L.ft_host_pack_keypoints.argtypes = [P(FtHostFeatures), vp]
    L.ft_host_pack_points.argtypes = [P(FtHostPoints), vp]
    _bound = True


def lib():
    """The library with the session entries bound (no device needed)."""
    L = _lib.load()
    _bind(L)
    return L


class Session:
    """One native ft_session on one CUDA device (lock-guarded: the session
    is single-threaded, like the reference's tracking thread)."""

    def __init__(self, device: int):
        self.lib = _lib.load()
        _bind(self.lib)
        h = vp()
        _lib.check(self.lib.ft_session_create(int(device), ctypes.byref(h)), "ft_session_create")
        self.handle = h
        self.lock = threading.Lock()

    def stats(self, reset: bool = False) -> dict:
        """Host phase times (us, summed over calls) of the native calls."""
        out = np.zeros(6)
        _lib.check(self.lib.ft_session_stats(self.handle, out.ctypes.data, int(reset)),
                   "ft_session_stats")
        return dict(zip(("pack", "issue", "kernel", "sync", "unpack", "calls"), out.tolist()))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            try:
                self.lib.ft_session_destroy(h)
            except Exception:  # noqa: BLE001  (interpreter shutdown)
                pass


_SESSIONS: dict[int, Session] = {}


def session() -> Session:
    import torch
    if not torch.cuda.is_available():
        raise _lib.FtError("no CUDA device: the B200 path has no CPU fallback")
    dev = torch.cuda.current_device()
    from . import _guard
    _guard.check(dev, "drop-in call")
    s = _SESSIONS.get(dev)
    if s is None:
        s = _SESSIONS[dev] = Session(dev)
    return s


# ---------------------------------------------------------------------------
# reference objects -> native structs (arrays passed in place)

def _c(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a) -> int | None:
    return a.ctypes.data if a is not None and a.size else None


def features(f, with_angle: bool = False, keep: list | None = None) -> FtHostFeatures:
    """FeatureSet (u, v, octave, angle, descriptors) -> ft_host_features."""
    u, v = _c(f.u, np.float64), _c(f.v, np.float64)
    o = _c(f.octave, np.int32)
    d = _c(f.descriptors, np.uint64)
    a = _c(f.angle, np.float64) if with_angle else None
    if keep is not None:
        keep.extend((u, v, o, d, a))
    return FtHostFeatures(len(u), _ptr(u), _ptr(v), _ptr(o), _ptr(a), _ptr(d))


def points(pts, keep: list) -> FtHostPoints:
    """MapPointSoA -> ft_host_points."""
    arrs = (_c(pts.positions, np.float64), _c(pts.normals, np.float64),
            _c(pts.min_distances, np.float64), _c(pts.max_distances, np.float64),
            _c(pts.descriptors, np.uint64), _c(pts.point_ids, np.int64))
    keep.extend(arrs)
    return FtHostPoints(len(arrs[5]), *(_ptr(a) for a in arrs))


@lru_cache(maxsize=64)
def _pyr_geometry(offsets: tuple, widths: tuple, heights: tuple) -> FtHostPyramid:
    p = FtHostPyramid()
    n = len(widths)
    if n < 1 or n > _lib.FT_MAX_LEVELS:
        raise ValueError(f"need 1..{_lib.FT_MAX_LEVELS} pyramid levels, got {n}")
    p.n_levels = n
    p.offsets[:n + 1] = offsets
    p.widths[:n] = widths
    p.heights[:n] = heights
    return p


_PYR_BY_BYTES: dict = {}


def _geometry_of(pyr) -> FtHostPyramid:
    # keyed by the level table's raw bytes (a new ImagePyramid per frame, the
    # same geometry): ~1 us instead of converting 25 numpy scalars per call
    try:
        key = (pyr.offsets.tobytes(), pyr.widths.tobytes(), pyr.heights.tobytes())
    except AttributeError:  # plain sequences
        key = None
    g = _PYR_BY_BYTES.get(key) if key is not None else None
    if g is None:
        g = _pyr_geometry(tuple(int(x) for x in pyr.offsets), tuple(int(x) for x in pyr.widths),
                          tuple(int(x) for x in pyr.heights))
        if key is not None:
            if len(_PYR_BY_BYTES) > 64:
                _PYR_BY_BYTES.clear()
            _PYR_BY_BYTES[key] = g
    return g


def pyramid(pyr, keep: list) -> FtHostPyramid:
    """ImagePyramid -> ft_host_pyramid (level table cached per geometry)."""
    g = _geometry_of(pyr)
    data = _c(pyr.data, np.uint8)
    if len(data) < g.offsets[g.n_levels]:
        raise ValueError("pyramid data shorter than its level table")
    keep.append(data)
    p = FtHostPyramid.from_buffer_copy(g)  # the cached level table
    p.data = data.ctypes.data
    return p


_MFIELDS = ("right_idx", "distance", "disparity", "refined_u", "depth", "sad")


def matches_struct(m) -> FtHostMatches:
    one = getattr(m, "_ft_rows", None)
    if one is not None and all(getattr(m, k) is r for k, r in zip(_MFIELDS, one[1])):
        # one allocation (empty_matches), fields not rebound: six rows of 8 * n bytes
        base, n = one[0], len(m.right_idx)
        return FtHostMatches(base, base + 8 * n, base + 16 * n, base + 24 * n, base + 32 * n,
                             base + 40 * n)
    return FtHostMatches(*(getattr(m, k).ctypes.data for k in _MFIELDS))


def empty_matches(n: int):
    """A StereoMatches whose six arrays are rows of ONE (6, n) allocation
    (int64 rows, the three fp64 fields as float64 views): one allocation and
    one pointer lookup per call instead of six."""
    from .types import StereoMatches
    buf = np.empty((6, n), np.int64)
    m = StereoMatches(right_idx=buf[0], distance=buf[1], disparity=buf[2].view(np.float64),
                      refined_u=buf[3].view(np.float64), depth=buf[4].view(np.float64),
                      sad=buf[5])
    try:
        m._ft_rows = (buf.ctypes.data, tuple(getattr(m, k) for k in _MFIELDS))
    except AttributeError:  # slotted / frozen result type: the generic path
        pass
    return m


def check(status: int, what: str) -> None:
    _lib.check(status, what)


# ---------------------------------------------------------------------------
# parameter structs, cached per configuration (the dataclass configs are
# frozen; cameras are keyed by their numeric fields)

_SP: dict = {}
_PP: dict = {}


def stereo_params(cfg, height: int, scale_pow, bf: float) -> _lib.FtStereoParams:
    from .runtime import stereo_params as build
    sp = np.asarray(scale_pow, dtype=np.float64)
    try:
        key = (cfg, int(height), sp.tobytes(), float(bf))
        hash(key)
    except TypeError:
        return build(cfg, height, sp, bf)
    p = _SP.get(key)
    if p is None:
        if len(_SP) > 256:
            _SP.clear()
        p = _SP[key] = build(cfg, height, sp, bf)
    return p


def _cam_key(cam) -> tuple:
    return tuple(float(getattr(cam, k, 0.0)) for k in
                 ("fx", "fy", "cx", "cy", "k1", "k2", "k3", "k4", "width", "height")) + (
        hasattr(cam, "k1"),)


_CAM_KEYS: dict = {}


def _cam_key_cached(cam) -> tuple:
    # the tracker's camera lives as long as the tracker: key it by identity,
    # keeping the object alive in the cache so its id is never reused
    hit = _CAM_KEYS.get(id(cam))
    if hit is not None and hit[0] is cam:
        return hit[1]
    k = _cam_key(cam)
    if len(_CAM_KEYS) > 64:
        _CAM_KEYS.clear()
    _CAM_KEYS[id(cam)] = (cam, k)
    return k


def project_params(cam, cfg, scale, levels, cell, nx, ny, window_px, u_offset):
    from .runtime import project_params as build
    try:
        key = (_cam_key_cached(cam), cfg, float(scale), int(levels), int(cell), int(nx), int(ny),
               None if window_px is None else float(window_px), float(u_offset))
        hash(key)
    except TypeError:
        return build(cam, cfg, scale, levels, cell, nx, ny, window_px, u_offset)
    p = _PP.get(key)
    if p is None:
        if len(_PP) > 256:
            _PP.clear()
        p = _PP[key] = build(cam, cfg, scale, levels, cell, nx, ny, window_px, u_offset)
    return p
