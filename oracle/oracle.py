"""CPU oracle for the tracking hot path -- TEST INFRASTRUCTURE ONLY.

Restates the reference (trackfront; /root/reference/pkg/src/trackfront) stage
functions on top of the plain-C kernels in ft_oracle.c (loaded via ctypes).
Host-side numpy steps follow the reference lines cited in each docstring.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may
import this module; the product package never does.  The oracle is pinned
against the reference's own outputs by tests/test_oracle_golden.py using the
fixtures that tests/golden/make_golden.py produced by running the reference.

All objects are duck-typed on the reference's attribute names (FeatureSet.u,
.v, .octave, .angle, .descriptors; MapPointSoA.positions, ...; Pose.rotation,
.translation; cameras with fx/fy/cx/cy[/k1..k4]; the dataclass configs), so
reference objects and paper_2509_10757_b200 objects both work.
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_LIB_PATH = _HERE / "_build" / "libft_oracle.so"
_lib = None

c_dp = ctypes.POINTER(ctypes.c_double)
c_i64p = ctypes.POINTER(ctypes.c_int64)
c_i32p = ctypes.POINTER(ctypes.c_int32)
c_u64p = ctypes.POINTER(ctypes.c_uint64)
c_u8p = ctypes.POINTER(ctypes.c_uint8)
I64 = ctypes.c_int64
F64 = ctypes.c_double
INT = ctypes.c_int


def build() -> Path:
    """Compile ft_oracle.c into oracle/_build/ (make)."""
    subprocess.run(["make", "-s", "-C", str(_HERE)], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not _LIB_PATH.exists():
            build()
        L = ctypes.CDLL(str(_LIB_PATH))
        L.fto_hamming_pairs.argtypes = [c_u64p, c_u64p, I64, c_i64p, INT]
        L.fto_build_row_buckets.argtypes = [c_dp, I64, I64, c_i64p, c_i64p]
        L.fto_stereo_phase1.argtypes = [c_dp, c_dp, c_i32p, c_u64p, I64, c_dp, c_dp, c_i32p,
                                        c_u64p, c_i64p, c_i64p, I64, c_dp, F64, F64, F64, I64,
                                        c_i64p, c_i64p, INT]
        L.fto_stereo_phase2.argtypes = [c_u8p, c_i64p, c_i64p, c_i64p, c_u8p, c_i64p, c_i64p,
                                        c_i64p, c_dp, c_dp, c_i32p, c_dp, c_i64p, I64, c_dp,
                                        I64, I64, F64, F64, c_dp, c_dp, c_i64p, c_u8p, INT]
        L.fto_bruteforce.argtypes = [c_u64p, I64, c_u64p, I64, I64, F64, c_i64p, c_i64p, INT]
        L.fto_frame_grid.argtypes = [c_dp, c_dp, I64, I64, I64, I64, c_i64p, c_i64p]
        L.fto_project_search.argtypes = (
            [c_dp, c_dp, c_dp, c_dp, c_u64p, c_u8p, I64, c_dp, c_dp, I64]
            + [F64] * 10
            + [c_dp, c_dp, c_i32p, c_u64p, c_i64p, c_i64p, I64, I64, I64, c_dp, I64, F64, F64,
               I64, F64, F64, F64, c_i64p, c_i64p, c_i64p, INT, c_i64p])
        L.fto_resolve_conflicts.argtypes = [c_i64p, c_i64p, c_i64p, I64, I64, c_i64p, c_i64p,
                                            c_i64p, c_i64p]
        L.fto_resolve_conflicts.restype = I64
        L.fto_rotation_filter.argtypes = [c_i64p, c_i64p, I64, c_dp, c_dp, I64, I64, c_u8p]
        L.fto_rotation_filter.restype = I64
        L.fto_median_i64.argtypes = [c_i64p, I64]
        L.fto_median_i64.restype = F64
        L.fto_num_threads_available.restype = INT
        L.fto_build_pyramid.argtypes = [c_u8p, I64, c_i64p, c_i64p, c_i64p, c_u8p]
        _lib = L
    return _lib


def _p(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(ctype)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _u64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.uint64).reshape(-1, 4)


def max_threads() -> int:
    return int(lib().fto_num_threads_available())


# ---------------------------------------------------------------------------
# result containers (field names of the reference dataclasses)

@dataclass
class OStereoMatches:
    """stereo.py:45-64 StereoMatches."""
    right_idx: np.ndarray
    distance: np.ndarray
    disparity: np.ndarray
    refined_u: np.ndarray
    depth: np.ndarray
    sad: np.ndarray

    def matched_mask(self) -> np.ndarray:
        return self.right_idx >= 0


@dataclass
class OCorrespondences:
    """projection.py:48-67 Correspondences."""
    point_idx: np.ndarray
    keypoint_idx: np.ndarray
    distance: np.ndarray
    octave: np.ndarray

    def __len__(self) -> int:
        return len(self.point_idx)


# ---------------------------------------------------------------------------
# stereo

def hamming_pairs(a, b, nthreads: int = 1) -> np.ndarray:
    a, b = _u64(a), _u64(b)
    out = np.empty(len(a), dtype=np.int64)
    lib().fto_hamming_pairs(_p(a, c_u64p), _p(b, c_u64p), len(a), _p(out, c_i64p), nthreads)
    return out


def build_row_buckets(v, height: int) -> tuple[np.ndarray, np.ndarray]:
    """stereo.py:67-74."""
    v = _f64(v)
    start = np.empty(int(height) + 1, dtype=np.int64)
    items = np.empty(len(v), dtype=np.int64)
    lib().fto_build_row_buckets(_p(v, c_dp), len(v), int(height), _p(start, c_i64p),
                                _p(items, c_i64p))
    return start, items


def match_pinhole_phase1(left, right, height: int, scale_pow, cfg, nthreads: int = 1,
                         row_buckets=None) -> tuple[np.ndarray, np.ndarray]:
    """stereo.py:77-103 -> kernels.py:300-345."""
    n = len(left.u)
    if row_buckets is None:
        row_buckets = build_row_buckets(right.v, height)
    rs, ri = _i64(row_buckets[0]), _i64(row_buckets[1])
    idx = np.empty(n, dtype=np.int64)
    dist = np.empty(n, dtype=np.int64)
    if n == 0:
        return idx, dist
    lu, lv, lo, ld = _f64(left.u), _f64(left.v), _i32(left.octave), _u64(left.descriptors)
    ru, rv, ro, rd = _f64(right.u), _f64(right.v), _i32(right.octave), _u64(right.descriptors)
    sp = _f64(scale_pow)
    lib().fto_stereo_phase1(_p(lu, c_dp), _p(lv, c_dp), _p(lo, c_i32p), _p(ld, c_u64p), n,
                            _p(ru, c_dp), _p(rv, c_dp), _p(ro, c_i32p), _p(rd, c_u64p),
                            _p(rs, c_i64p), _p(ri, c_i64p), len(rs) - 1, _p(sp, c_dp),
                            float(cfg.band_factor), float(cfg.min_disparity),
                            float(cfg.max_disparity), int(cfg.t_match),
                            _p(idx, c_i64p), _p(dist, c_i64p), nthreads)
    return idx, dist


def refine_match_phase2(left_pyr, right_pyr, left, right, cand_idx, cand_dist, cam, cfg,
                        nthreads: int = 1) -> OStereoMatches:
    """stereo.py:106-140 -> kernels.py:351-428, host post-processing :129-140."""
    n = len(left.u)
    scale_pow = float(left_pyr.scale) ** np.arange(len(left_pyr.widths), dtype=np.float64)
    disp = np.zeros(n)
    ur = np.zeros(n)
    sad = np.zeros(n, dtype=np.int64)
    ok = np.zeros(n, dtype=np.uint8)
    cand_idx = _i64(cand_idx)
    if n:
        ld = np.ascontiguousarray(left_pyr.data, dtype=np.uint8)
        rdat = np.ascontiguousarray(right_pyr.data, dtype=np.uint8)
        lo_, lw, lh = _i64(left_pyr.offsets), _i64(left_pyr.widths), _i64(left_pyr.heights)
        ro_, rw, rh = _i64(right_pyr.offsets), _i64(right_pyr.widths), _i64(right_pyr.heights)
        lu, lv, loct, ru = _f64(left.u), _f64(left.v), _i32(left.octave), _f64(right.u)
        lib().fto_stereo_phase2(_p(ld, c_u8p), _p(lo_, c_i64p), _p(lw, c_i64p), _p(lh, c_i64p),
                                _p(rdat, c_u8p), _p(ro_, c_i64p), _p(rw, c_i64p),
                                _p(rh, c_i64p), _p(lu, c_dp), _p(lv, c_dp), _p(loct, c_i32p),
                                _p(ru, c_dp), _p(cand_idx, c_i64p), n, _p(scale_pow, c_dp),
                                int(cfg.half_window), int(cfg.half_slide),
                                float(cfg.min_disparity), float(cfg.max_disparity),
                                _p(disp, c_dp), _p(ur, c_dp), _p(sad, c_i64p), _p(ok, c_u8p),
                                nthreads)
    accepted = ok.astype(bool)
    right_idx = np.where(accepted, cand_idx, -1)
    depth = np.zeros(n)
    depth[accepted] = cam.baseline_times_fx / disp[accepted]
    return OStereoMatches(right_idx=right_idx,
                          distance=np.where(accepted, cand_dist, 10000),
                          disparity=np.where(accepted, disp, 0.0),
                          refined_u=np.where(accepted, ur, 0.0),
                          depth=depth,
                          sad=np.where(accepted, sad, 0))


def matches_from_candidates(cand_idx, cand_dist, left, right, cam, cfg) -> OStereoMatches:
    """stereo.py:143-168 (numpy, restated)."""
    n = len(cand_idx)
    right_idx = _i64(cand_idx).copy()
    disp = np.zeros(n)
    depth = np.zeros(n)
    ur = np.zeros(n)
    m = right_idx >= 0
    disp[m] = left.u[m] - right.u[right_idx[m]]
    bad = m & ((disp < cfg.min_disparity) | (disp > cfg.max_disparity))
    right_idx[bad] = -1
    m = right_idx >= 0
    depth[m] = cam.baseline_times_fx / disp[m]
    ur[m] = right.u[right_idx[m]]
    return OStereoMatches(right_idx=right_idx,
                          distance=np.where(m, cand_dist, 10000),
                          disparity=np.where(m, disp, 0.0),
                          refined_u=ur,
                          depth=np.where(m, depth, 0.0),
                          sad=np.zeros(n, dtype=np.int64))


def reject_outliers(matches, cfg):
    """stereo.py:171-188, in place (median via the C port of np.median)."""
    m = matches.right_idx >= 0
    if not m.any():
        return matches
    vals = _i64(matches.sad[m])
    med = float(lib().fto_median_i64(_p(vals, c_i64p), len(vals)))
    bad = m & (matches.sad > cfg.outlier_multiplier * med)
    matches.right_idx[bad] = -1
    matches.distance[bad] = 10000
    matches.disparity[bad] = 0.0
    matches.refined_u[bad] = 0.0
    matches.depth[bad] = 0.0
    matches.sad[bad] = 0
    return matches


def bruteforce(ldesc, rdesc, t_match: int, ratio: float,
               nthreads: int = 1) -> tuple[np.ndarray, np.ndarray]:
    """kernels.py:434-464 (as launched by stereo.py:238-244)."""
    a, b = _u64(ldesc), _u64(rdesc)
    idx = np.empty(len(a), dtype=np.int64)
    dist = np.empty(len(a), dtype=np.int64)
    lib().fto_bruteforce(_p(a, c_u64p), len(a), _p(b, c_u64p), len(b), int(t_match),
                         float(ratio), _p(idx, c_i64p), _p(dist, c_i64p), nthreads)
    return idx, dist


def fisheye_unproject(cam, u: float, v: float) -> np.ndarray:
    """cameras.py:139-157 FisheyeCamera.unproject (Kannala-Brandt Newton
    inversion), term for term."""
    mx = (u - cam.cx) / cam.fx
    my = (v - cam.cy) / cam.fy
    rd = float(np.hypot(mx, my))
    if rd < 1e-12:
        return np.array([0.0, 0.0, 1.0])
    theta = min(rd, np.pi / 2)
    for _ in range(20):
        t2 = theta * theta
        f = theta * (1.0 + t2 * (cam.k1 + t2 * (cam.k2 + t2 * (cam.k3 + t2 * cam.k4)))) - rd
        df = 1.0 + t2 * (3 * cam.k1 + t2 * (5 * cam.k2 + t2 * (7 * cam.k3 + t2 * 9 * cam.k4)))
        step = f / df
        theta -= step
        if abs(step) < 1e-14:
            break
    s = np.sin(theta) / rd
    ray = np.array([s * mx, s * my, np.cos(theta)])
    return ray / np.linalg.norm(ray)


def closest_ray_points(oa, da, ob, db, corrected: bool = False):
    """stereo.py:200-220 _closest_ray_points.  corrected=False keeps the
    reference's t = (a11 b2 - a12 b1) / den (stereo.py:216); corrected=True is
    the least-squares t = (a12 b1 - a11 b2) / den."""
    da = np.asarray(da, dtype=np.float64)
    db = np.asarray(db, dtype=np.float64)
    oa = np.asarray(oa, dtype=np.float64)
    ob = np.asarray(ob, dtype=np.float64)
    if np.linalg.norm(np.cross(da, db)) < 1e-9:
        return None, None, None, None
    r = ob - oa
    a11 = da @ da
    a12 = da @ db
    a22 = db @ db
    b1 = da @ r
    b2 = db @ r
    den = a11 * a22 - a12 * a12
    s = (b1 * a22 - a12 * b2) / den
    t = ((a12 * b1 - a11 * b2) if corrected else (a11 * b2 - a12 * b1)) / den
    pa = oa + s * da
    pb = ob + t * db
    gap = float(np.linalg.norm(pa - pb))
    return (pa + pb) / 2.0, gap, s, t


def fisheye_triangulate(left, right, idx, dist, cam, ray_gap_ceiling: float,
                        corrected: bool = False):
    """stereo.py:245-273: triangulate the accepted brute-force pairs ->
    (left_ids, right_ids, points, dists)."""
    rot_rl = np.asarray(cam.right_extrinsic.rotation, dtype=np.float64)
    tr_rl = np.asarray(cam.right_extrinsic.translation, dtype=np.float64)
    rot_lr = rot_rl.T
    tr_lr = -rot_lr @ tr_rl
    left_ids, right_ids, points, dists = [], [], [], []
    for i in np.nonzero(np.asarray(idx) >= 0)[0]:
        j = int(idx[i])
        ray_l = fisheye_unproject(cam, float(left.u[i]), float(left.v[i]))
        ray_r = fisheye_unproject(cam, float(right.u[j]), float(right.v[j]))
        dir_r = rot_lr @ ray_r
        pt, gap, _, _ = closest_ray_points(np.zeros(3), ray_l, tr_lr, dir_r, corrected)
        if pt is None or gap is None or gap > ray_gap_ceiling:
            continue
        p_right = rot_rl @ pt + tr_rl
        if pt[2] <= 0 or p_right[2] <= 0:
            continue
        left_ids.append(int(i))
        right_ids.append(j)
        points.append(pt)
        dists.append(int(dist[i]))
    if not left_ids:
        return (np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64), np.empty((0, 3)),
                np.empty(0, dtype=np.int64))
    return (np.asarray(left_ids, dtype=np.int64), np.asarray(right_ids, dtype=np.int64),
            np.asarray(points), np.asarray(dists, dtype=np.int64))


# ---------------------------------------------------------------------------
# search by projection

def frame_grid(u, v, width: int, height: int, cell_px: int = 48):
    """mapping.py:68-100 FrameGrid -> (start, indices, nx, ny)."""
    cell_px = int(cell_px)
    nx = max(1, (int(width) + cell_px - 1) // cell_px)
    ny = max(1, (int(height) + cell_px - 1) // cell_px)
    u, v = _f64(u), _f64(v)
    start = np.empty(nx * ny + 1, dtype=np.int64)
    idx = np.empty(len(u), dtype=np.int64)
    lib().fto_frame_grid(_p(u, c_dp), _p(v, c_dp), len(u), cell_px, nx, ny,
                         _p(start, c_i64p), _p(idx, c_i64p))
    return start, idx, nx, ny


def camera_args(cam) -> tuple:
    """projection.py:110-115 _camera_args (duck-typed: fisheye has k1..k4)."""
    if hasattr(cam, "k1"):
        return (1, cam.fx, cam.fy, cam.cx, cam.cy, cam.k1, cam.k2, cam.k3, cam.k4,
                float(cam.width), float(cam.height))
    return (0, cam.fx, cam.fy, cam.cx, cam.cy, 0.0, 0.0, 0.0, 0.0,
            float(cam.width), float(cam.height))


def run_phase_a(points, kp_u, kp_v, kp_oct, kp_desc, grid, pose, cam, cfg, scale: float,
                levels: int, skip_mask=None, window_px=None, u_offset: float = 0.0,
                nthreads: int = 1, ham_count: list | None = None):
    """projection.py:118-158 -> kernels.py:470-579.  ``grid`` is
    (start, indices, nx, ny, cell_px).  ``ham_count`` (a list) receives the
    number of Hamming evaluations performed (work accounting for bench.py)."""
    n = len(points.point_ids)
    out_kp = np.empty(n, dtype=np.int64)
    out_dist = np.empty(n, dtype=np.int64)
    out_oct = np.empty(n, dtype=np.int64)
    if n == 0:
        return out_kp, out_dist, out_oct
    skip = (np.zeros(n, dtype=np.uint8) if skip_mask is None
            else np.ascontiguousarray(skip_mask, dtype=np.uint8))
    scale_pow = scale ** np.arange(levels, dtype=np.float64)
    window = cfg.window_px if window_px is None else window_px
    ca = camera_args(cam)
    pos, nor = _f64(points.positions), _f64(points.normals)
    mind, maxd = _f64(points.min_distances), _f64(points.max_distances)
    pdesc = _u64(points.descriptors)
    rot, tr = _f64(pose.rotation), _f64(pose.translation)
    ku, kv, ko, kd = _f64(kp_u), _f64(kp_v), _i32(kp_oct), _u64(kp_desc)
    gs, gi = _i64(grid[0]), _i64(grid[1])
    hc = ctypes.c_int64(0)
    lib().fto_project_search(
        _p(pos, c_dp), _p(nor, c_dp), _p(mind, c_dp), _p(maxd, c_dp), _p(pdesc, c_u64p),
        _p(skip, c_u8p), n, _p(rot, c_dp), _p(tr, c_dp), int(ca[0]),
        *[float(x) for x in ca[1:]],
        _p(ku, c_dp), _p(kv, c_dp), _p(ko, c_i32p), _p(kd, c_u64p), _p(gs, c_i64p),
        _p(gi, c_i64p), int(grid[2]), int(grid[3]), int(grid[4]), _p(scale_pow, c_dp),
        int(levels), 1.0 / math.log(scale), float(window), int(cfg.t_proj), float(cfg.ratio),
        float(cfg.view_cos_min), float(u_offset),
        _p(out_kp, c_i64p), _p(out_dist, c_i64p), _p(out_oct, c_i64p), nthreads,
        ctypes.byref(hc))
    if ham_count is not None:
        ham_count.append(int(hc.value))
    return out_kp, out_dist, out_oct


def resolve_conflicts(out_kp, out_dist, out_oct, n_kp: int | None = None) -> OCorrespondences:
    """projection.py:161-178."""
    out_kp, out_dist, out_oct = _i64(out_kp), _i64(out_dist), _i64(out_oct)
    n = len(out_kp)
    if n_kp is None:
        n_kp = int(out_kp.max()) + 1 if n and out_kp.max() >= 0 else 0
    pi = np.empty(n, dtype=np.int64)
    ki = np.empty(n, dtype=np.int64)
    di = np.empty(n, dtype=np.int64)
    oi = np.empty(n, dtype=np.int64)
    m = lib().fto_resolve_conflicts(_p(out_kp, c_i64p), _p(out_dist, c_i64p),
                                    _p(out_oct, c_i64p), n, int(n_kp), _p(pi, c_i64p),
                                    _p(ki, c_i64p), _p(di, c_i64p), _p(oi, c_i64p))
    return OCorrespondences(pi[:m].copy(), ki[:m].copy(), di[:m].copy(), oi[:m].copy())


def rotation_consistency_filter(corr, ref_angles, kp_angles, cfg) -> OCorrespondences:
    """projection.py:181-200."""
    m = len(corr.point_idx)
    if m == 0:
        return corr
    pi, ki = _i64(corr.point_idx), _i64(corr.keypoint_idx)
    ra, ka = _f64(ref_angles), _f64(kp_angles)
    keep = np.empty(m, dtype=np.uint8)
    lib().fto_rotation_filter(_p(pi, c_i64p), _p(ki, c_i64p), m, _p(ra, c_dp), _p(ka, c_dp),
                              int(cfg.histogram_bins), int(cfg.histogram_keep), _p(keep, c_u8p))
    mask = keep.astype(bool)
    return OCorrespondences(corr.point_idx[mask], corr.keypoint_idx[mask],
                            corr.distance[mask], corr.octave[mask])


def search_by_projection(points, kp_u, kp_v, kp_oct, kp_desc, kp_angle, grid, pose, cam, cfg,
                         scale, levels, skip_mask=None, ref_angles=None,
                         rotation_check=False, window_px=None, u_offset=0.0,
                         nthreads: int = 1) -> OCorrespondences:
    """projection.py:203-221."""
    kp, kd, ko = run_phase_a(points, kp_u, kp_v, kp_oct, kp_desc, grid, pose, cam, cfg, scale,
                             levels, skip_mask, window_px, u_offset, nthreads)
    corr = resolve_conflicts(kp, kd, ko, len(kp_u))
    if rotation_check and ref_angles is not None:
        corr = rotation_consistency_filter(corr, ref_angles, kp_angle, cfg)
    return corr


def skip_from_slots(point_ids, slots) -> np.ndarray:
    """localmap.py:93-96: skip[i] = point_ids[i] in unique(slots != -1)."""
    slotted = np.unique(slots[slots != -1])
    return np.isin(point_ids, slotted).astype(np.uint8)


def search_local_points(point_ids, soa, kp_u, kp_v, kp_oct, kp_desc, grid, slots, pose, cam,
                        cfg, scale, levels, nthreads: int = 1) -> int:
    """localmap.py:79-122 without the world-map flag updates; mutates slots."""
    if len(point_ids) == 0:
        return int(np.count_nonzero(slots != -1))
    skip = skip_from_slots(point_ids, slots)
    corr = search_by_projection(soa, kp_u, kp_v, kp_oct, kp_desc, None, grid, pose, cam, cfg,
                                scale, levels, skip_mask=skip, nthreads=nthreads)
    for pi, ki in zip(corr.point_idx, corr.keypoint_idx):
        if slots[ki] != -1:
            continue
        slots[ki] = point_ids[pi]
    return int(np.count_nonzero(slots != -1))


def stereo_pinhole(left, right, left_pyr, right_pyr, cam, cfg, scale_pow,
                   nthreads: int = 1) -> OStereoMatches:
    """tracker.py:415-427 pinhole _run_stereo: phase 1, then phase 2 when
    pyramids exist (else matches_from_candidates), then reject_outliers."""
    idx, dist = match_pinhole_phase1(left, right, cam.height, scale_pow, cfg, nthreads)
    if left_pyr is None:
        m = matches_from_candidates(idx, dist, left, right, cam, cfg)
    else:
        m = refine_match_phase2(left_pyr, right_pyr, left, right, idx, dist, cam, cfg, nthreads)
    return reject_outliers(m, cfg)


def pyramid_level_dims(width: int, height: int, scale: float, levels: int):
    """extraction.py:58-64: floor(dims / scale ** level)."""
    powers = scale ** np.arange(levels, dtype=np.float64)
    return (np.floor(width / powers).astype(np.int64), np.floor(height / powers).astype(np.int64))


def build_pyramid(image, levels: int = 8, scale: float = 1.2):
    """extraction.py:97-125 build_pyramid -> (data u8[total], offsets, widths,
    heights), via fto_build_pyramid (kernels.py:230-268)."""
    image = np.ascontiguousarray(image, dtype=np.uint8)
    h, w = image.shape
    ws, hs = pyramid_level_dims(w, h, scale, levels)
    offsets = np.zeros(levels + 1, dtype=np.int64)
    np.cumsum(ws * hs, out=offsets[1:])
    data = np.zeros(int(offsets[-1]), dtype=np.uint8)
    lib().fto_build_pyramid(_p(image, c_u8p), levels, _p(offsets, c_i64p), _p(ws, c_i64p),
                            _p(hs, c_i64p), _p(data, c_u8p))
    return data, offsets, ws, hs


def _env_threads() -> int:
    try:
        return max(1, int(os.environ.get("FT_ORACLE_THREADS", "1")))
    except ValueError:
        return 1


# ---------------------------------------------------------------------------
# local map gathering

def update_local_map(slots, kf_obs, kf_off, n_kf: int):
    """localmap.py:42-76 update_local_map over a world given as keyframe
    observation lists (keyframe k observes kf_obs[kf_off[k]:kf_off[k+1]],
    KeyFrame.observed_point_ids, mapping.py:142-145): seeds = the frame's
    slotted ids; keyframes = those observing any seed (a point's
    observations are exactly the (keyframe, slot) pairs whose keyframe holds
    it, mapping.py:262-266); points = every id those keyframes observe.
    Returns (keyframe indices ascending, point ids ascending); empty seeds ->
    both empty (LocalMap.empty())."""
    slots = np.asarray(slots, dtype=np.int64)
    seeds = np.unique(slots[slots != -1])
    if len(seeds) == 0:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    kf_off = np.asarray(kf_off, dtype=np.int64)
    kf_obs = np.asarray(kf_obs, dtype=np.int64)
    kfs = [k for k in range(int(n_kf))
           if np.isin(kf_obs[kf_off[k]:kf_off[k + 1]], seeds, assume_unique=False).any()]
    if not kfs:
        return np.empty(0, np.int64), np.empty(0, np.int64)
    pts = np.unique(np.concatenate([kf_obs[kf_off[k]:kf_off[k + 1]] for k in kfs]))
    return np.asarray(kfs, dtype=np.int64), pts.astype(np.int64)
