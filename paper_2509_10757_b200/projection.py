"""Search by projection drop-in: the reference's stage functions on B200.

Signatures, argument meaning, outputs and error behaviour follow the
reference module ``trackfront.projection`` (pkg/src/trackfront/projection.py).
Phase A (projection + windowed descriptor search), phase B (conflict
resolution) and phase C (rotation histogram) run fused in
``ft_project_search`` (csrc/ft_project.cu); ``run_phase_a`` /
``resolve_conflicts`` / ``rotation_consistency_filter`` are also callable on
their own through their own C-ABI entries.  ``engine`` / ``pool`` are accepted
for signature compatibility and ignored.
"""

from __future__ import annotations

import math

import numpy as np

from . import _lib
from .runtime import (Layout, add_keypoints, fill_point_records, keypoints_struct,
                      project_params, put_keypoints, runtime)
from .types import Correspondences, ProjectionSearchConfig, NO_POINT

__all__ = ["ProjectionSearchConfig", "Correspondences", "predict_scale", "frustum_and_cone_check",
           "run_phase_a", "resolve_conflicts", "rotation_consistency_filter",
           "search_by_projection", "search_prev_frame"]


def predict_scale(distance: float, max_distance: float, scale: float, levels: int) -> int:
    """Scalar twin of the kernel's level prediction (reference projection.py:70-77)."""
    r = math.log(max_distance / distance) / math.log(scale)
    return int(min(max(math.ceil(r - 1e-9), 0), levels - 1))


def frustum_and_cone_check(position, normal, min_distance, max_distance, pose, cam,
                           cfg: ProjectionSearchConfig, scale: float, levels: int):
    """Scalar visibility gate for one map point (reference projection.py:80-107);
    host helper for callers, the kernels inline the same test."""
    position = np.asarray(position, dtype=np.float64)
    p = pose.rotation @ position + pose.translation
    if p[2] <= 1e-6:
        return None
    x, y, z = float(p[0]), float(p[1]), float(p[2])
    if hasattr(cam, "k1"):
        r = math.hypot(x, y)
        if r < 1e-12:
            u, v = cam.cx, cam.cy
        else:
            th = math.atan2(r, z)
            t2 = th * th
            d = th * (1.0 + t2 * (cam.k1 + t2 * (cam.k2 + t2 * (cam.k3 + t2 * cam.k4))))
            u, v = cam.fx * d * x / r + cam.cx, cam.fy * d * y / r + cam.cy
    else:
        u, v = cam.fx * x / z + cam.cx, cam.fy * y / z + cam.cy
    if not (0.0 <= u < cam.width and 0.0 <= v < cam.height):
        return None
    dist = float(np.linalg.norm(p))
    if dist < min_distance or dist > max_distance:
        return None
    center = -pose.rotation.T @ pose.translation
    cosang = float((position - center) @ np.asarray(normal)) / dist
    if cosang < cfg.view_cos_min:
        return None
    return predict_scale(dist, max_distance, scale, levels), u, v, cosang


# ---------------------------------------------------------------------------

def _grid_geometry(frame, cam) -> tuple[int, int, int]:
    g = getattr(frame, "grid", None)
    if g is not None:
        return int(g.cell_px), int(g.nx), int(g.ny)
    cell = 48
    return cell, max(1, (int(cam.width) + cell - 1) // cell), max(1, (int(cam.height) + cell - 1) // cell)


def project_search(points, frame, pose, cam, cfg: ProjectionSearchConfig, scale: float,
                   levels: int, *, skip_mask=None, ref_angles=None, rotation: bool = False,
                   window_px=None, u_offset: float = 0.0, slots=None, skip_slotted=False,
                   write_slots=False, resolve=True, phase_a_out=False, table=None,
                   table_slots=None, want_corr=True):
    """One fused ``ft_project_search`` launch on one frame, through the
    native session (csrc/ft_session.cu: the reference objects' arrays are
    packed, shipped, searched and the requested outputs copied back in one
    C call).  table: a resident MapTable -- the points are read in place
    through their table slots (points missing from it are uploaded first:
    the map delta).

    Returns a dict with any of: out_kp/out_dist/out_oct (phase A),
    corr (Correspondences), slots (updated copy), count (filled slots)."""
    from . import session as S
    ses = S.session()
    left = frame.left
    n_kp, m = len(left.u), len(points.point_ids)
    cell, nx, ny = _grid_geometry(frame, cam)
    with_angle = bool(rotation and ref_angles is not None)
    keep: list = []
    kf = S.features(left, with_angle=with_angle, keep=keep)
    if table is None:
        pts = S.points(points, keep)
        tptr, tsize, tidx = None, 0, None
    else:
        if table_slots is not None:  # resident local map: slots already known
            tidx = np.ascontiguousarray(table_slots, np.int32)
        else:
            if m and getattr(points, "positions", None) is not None:
                table.upsert(points.point_ids, points, only_missing=True)
            tidx = np.ascontiguousarray(table.slots(points.point_ids), np.int32)
        pts = S.FtHostPoints(m, None, None, None, None, None, None)
        tptr, tsize = table.ptr, table.capacity
    mode = 0
    if resolve:
        mode |= _lib.FT_PROJ_RESOLVE
    if with_angle:
        mode |= _lib.FT_PROJ_ROTATION
    if skip_slotted:
        mode |= _lib.FT_PROJ_SKIP_SLOTS
    if write_slots:
        mode |= _lib.FT_PROJ_WRITE_SLOTS
    params = S.project_params(cam, cfg, scale, levels, cell, nx, ny, window_px, u_offset)
    rot = np.ascontiguousarray(pose.rotation, np.float64).reshape(9)
    trans = np.ascontiguousarray(pose.translation, np.float64).reshape(3)
    skip = np.ascontiguousarray(skip_mask, np.uint8) if skip_mask is not None else None
    ref = np.ascontiguousarray(ref_angles, np.float64) if with_angle else None
    sl = np.ascontiguousarray(slots, np.int64) if slots is not None else None
    res, out = {}, S.FtHostProjectOut()
    if phase_a_out:
        res["out_kp"], res["out_dist"], res["out_oct"] = (np.empty(m, np.int64) for _ in range(3))
        out.out_kp, out.out_dist, out.out_oct = (res[k].ctypes.data for k in
                                                 ("out_kp", "out_dist", "out_oct"))
    want_corr = want_corr and resolve
    cbuf = np.empty((4, max(m, 1)), np.int64) if want_corr else None
    counts = np.zeros(2, np.int32)
    if want_corr:  # (search_local_points needs only the slots and the count)
        out.corr_point, out.corr_kp, out.corr_dist, out.corr_oct = (cbuf[q].ctypes.data
                                                                    for q in range(4))
    out.corr_count = counts.ctypes.data
    out.slot_count = counts.ctypes.data + 4
    slots_out = np.empty(n_kp, np.int64) if sl is not None else None
    if slots_out is not None:
        out.slots_out = slots_out.ctypes.data
    with ses.lock:
        st = ses.lib.ft_session_project(ses.handle, pts, tptr, tsize,
                                        tidx.ctypes.data if tidx is not None and m else None,
                                        kf, params, rot.ctypes.data, trans.ctypes.data,
                                        skip.ctypes.data if skip is not None and m else None,
                                        ref.ctypes.data if ref is not None and m else None,
                                        sl.ctypes.data if sl is not None and n_kp else None,
                                        mode, out)
    _lib.check(st, "ft_session_project")
    if want_corr:
        c = int(counts[0])
        res["corr"] = Correspondences(*(cbuf[q, :c].copy() for q in range(4)))
    if slots_out is not None:
        res["slots"] = slots_out
    if write_slots:
        res["count"] = int(counts[1])
    return res


def run_phase_a(points, frame, pose, cam, cfg: ProjectionSearchConfig, scale: float,
                levels: int, engine=None, skip_mask: np.ndarray | None = None,
                window_px: float | None = None, u_offset: float = 0.0, pool=None
                ) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """Per-point candidate keypoint, distance and predicted octave
    (reference projection.py:118-158 -> kernels.py:470-579)."""
    n = len(points.point_ids)
    if n == 0:
        z = np.empty(0, dtype=np.int64)
        return z, z.copy(), z.copy()
    r = project_search(points, frame, pose, cam, cfg, scale, levels, skip_mask=skip_mask,
                       window_px=window_px, u_offset=u_offset, resolve=False, phase_a_out=True)
    return r["out_kp"], r["out_dist"], r["out_oct"]


def resolve_conflicts(out_kp: np.ndarray, out_dist: np.ndarray,
                      out_oct: np.ndarray) -> Correspondences:
    """Phase B (reference projection.py:161-178): per keypoint the lowest
    distance wins, ties to the lower point index; output in point order."""
    out_kp = np.asarray(out_kp)
    n = len(out_kp)
    if n == 0 or not (out_kp >= 0).any():
        return Correspondences.empty()
    n_kp = int(out_kp.max()) + 1
    rt = runtime()
    cap_kp, cap_pts = rt.caps(n_kp, n)
    lay = Layout()
    for k in ("kp", "dist", "oct"):
        lay.add(k, 8 * n)
    in_end = lay.total
    for k in ("c_point", "c_kp", "c_dist", "c_oct"):
        lay.add(k, 8 * n)
    lay.add("c_n", 4)
    with rt.lock:
        rt.reserve(lay.total)
        rt.put(lay, "kp", out_kp, np.int64)
        rt.put(lay, "dist", out_dist, np.int64)
        rt.put(lay, "oct", out_oct, np.int64)
        rt.h2d(0, in_end)
        o = _lib.FtProjectOut()
        o.corr_point, o.corr_kp = rt.ptr(lay, "c_point"), rt.ptr(lay, "c_kp")
        o.corr_dist, o.corr_oct, o.corr_count = (rt.ptr(lay, "c_dist"), rt.ptr(lay, "c_oct"),
                                                 rt.ptr(lay, "c_n"))
        st = rt.lib.ft_resolve_conflicts(n, rt.ptr(lay, "kp"), rt.ptr(lay, "dist"),
                                         rt.ptr(lay, "oct"), n_kp, o, rt.workspace(),
                                         rt.stream.cuda_stream)
        _lib.check(st, "ft_resolve_conflicts")
        rt.d2h(in_end, lay.total)
        rt.sync()
        c = int(rt.host_view(lay, "c_n", np.int32, (1,))[0])
        return Correspondences(*(rt.host_view(lay, k, np.int64, (c,)).copy()
                                 for k in ("c_point", "c_kp", "c_dist", "c_oct")))


def rotation_consistency_filter(corr: Correspondences, ref_angles: np.ndarray,
                                kp_angles: np.ndarray,
                                cfg: ProjectionSearchConfig) -> Correspondences:
    """Phase C (reference projection.py:181-200): keep correspondences in
    the K most populated of B angle-difference bins (ties: lower bin)."""
    m = len(corr.point_idx)
    if m == 0:
        return corr
    rt = runtime()
    lay = Layout()
    for k in ("c_point", "c_kp", "c_dist", "c_oct"):
        lay.add(k, 8 * m)
    lay.add("ref", 8 * len(ref_angles))
    lay.add("kpa", 8 * len(kp_angles))
    in_end = lay.total
    lay.add("c_n", 4)
    with rt.lock:
        rt.reserve(lay.total)
        for k, arr in (("c_point", corr.point_idx), ("c_kp", corr.keypoint_idx),
                       ("c_dist", corr.distance), ("c_oct", corr.octave)):
            rt.put(lay, k, arr, np.int64)
        rt.put(lay, "ref", ref_angles, np.float64)
        rt.put(lay, "kpa", kp_angles, np.float64)
        rt.h2d(0, in_end)
        st = rt.lib.ft_rotation_filter(m, rt.ptr(lay, "c_point"), rt.ptr(lay, "c_kp"),
                                       rt.ptr(lay, "c_dist"), rt.ptr(lay, "c_oct"),
                                       rt.ptr(lay, "ref"), rt.ptr(lay, "kpa"),
                                       int(cfg.histogram_bins), int(cfg.histogram_keep),
                                       rt.ptr(lay, "c_n"), rt.stream.cuda_stream)
        _lib.check(st, "ft_rotation_filter")
        rt.d2h(0, lay.total)
        rt.sync()
        c = int(rt.host_view(lay, "c_n", np.int32, (1,))[0])
        return Correspondences(*(rt.host_view(lay, k, np.int64, (c,)).copy()
                                 for k in ("c_point", "c_kp", "c_dist", "c_oct")))


def search_by_projection(points, frame, pose, cam, cfg: ProjectionSearchConfig, scale: float,
                         levels: int, engine=None, skip_mask: np.ndarray | None = None,
                         ref_angles: np.ndarray | None = None, rotation_check: bool = False,
                         window_px: float | None = None, u_offset: float = 0.0,
                         pool=None, table=None) -> Correspondences:
    """Project map points into the frame and resolve the best associations
    (reference projection.py:203-221) -- phases A, B and C in ONE launch.
    table: optional resident MapTable (the points are read in place through
    their slots; only points missing from it are uploaded)."""
    if len(points.point_ids) == 0:
        return Correspondences.empty()
    r = project_search(points, frame, pose, cam, cfg, scale, levels, skip_mask=skip_mask,
                       ref_angles=ref_angles, rotation=bool(rotation_check),
                       window_px=window_px, u_offset=u_offset, table=table)
    return r["corr"]


_RESIDENT_WORLD = False  # set by install(resident_world=True)


def search_prev_frame(prev, cur, pose, world, cam, cfg: ProjectionSearchConfig, scale: float,
                      levels: int, engine=None, soa_out=None, pool=None, table=None):
    """Match the previous frame's map points into the current frame
    (reference projection.py:224-253).  Without a table the previous frame's
    slotted points are decomposed on the host (mapping.py:204-235), as in the
    reference; with a resident MapTable only points missing from the table
    are decomposed and uploaded (the map delta) and the search reads the rest
    in place.  soa_out, when given (the tracker's pooled
    buffers, tracker.py:304-314), receives the decomposed points as in the
    reference and the returned point ids are a view of it."""
    from .types import MapPointSoA
    slot_idx = np.nonzero(prev.slots != NO_POINT)[0]
    if len(slot_idx) == 0:
        return Correspondences.empty(), np.empty(0, dtype=np.int64)
    pids = np.asarray(prev.slots[slot_idx], dtype=np.int64)
    if table is None and _RESIDENT_WORLD and world is not None:
        # install(resident_world=True): the world update_local_map mirrors in
        # HBM serves the previous frame's points in place (soa_out untouched)
        from .worldmap import world_table
        wt = world_table(world)
        wt.sync(world)
        table = wt.table

    def decompose(ids):
        from .maptable import decompose_points
        return decompose_points([world.points[int(p)] for p in ids])

    if table is None:
        points = decompose(pids)
        if soa_out is not None:  # reference: decompose_map_points(mps, out=soa_out)
            k = len(pids)
            for name in ("positions", "descriptors", "normals", "min_distances",
                         "max_distances", "point_ids"):
                getattr(soa_out, name)[:k] = getattr(points, name)
            points = MapPointSoA(*(getattr(soa_out, name)[:k] for name in
                                   ("positions", "descriptors", "normals", "min_distances",
                                    "max_distances", "point_ids")))
    else:
        # resident mode: the points are read in place from the table, nothing
        # is decomposed, soa_out is left untouched
        missing = pids[table._lookup(pids) < 0]
        if len(missing):
            table.upsert(missing, decompose(missing))
        points = _IdsOnly(pids)
    ref_angles = prev.left.angle[slot_idx]
    rel = pose.matrix() @ np.linalg.inv(prev.pose.matrix())
    forward = float(rel[2, 3])
    u_offset = math.copysign(cfg.prev_u_offset_px, forward) if abs(forward) > 1e-9 else 0.0
    corr = search_by_projection(points, cur, pose, cam, cfg, scale, levels, ref_angles=ref_angles,
                                rotation_check=cfg.rotation_check_prev,
                                window_px=cfg.window_prev_px, u_offset=u_offset, table=table)
    return corr, np.asarray(points.point_ids)


class _IdsOnly:
    """Points named by id only (their records are resident in a MapTable)."""

    def __init__(self, point_ids):
        self.point_ids = np.asarray(point_ids, dtype=np.int64)
        self.positions = None
