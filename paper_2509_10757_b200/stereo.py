"""Stereo matching drop-in: the reference's stage functions on B200.

Signatures, argument meaning, outputs and error behaviour follow the
reference module ``trackfront.stereo`` (pkg/src/trackfront/stereo.py); the
work runs in the fused sm_100a kernel ``ft_stereo_pinhole`` /
``ft_stereo_fisheye_bf`` (csrc/ft_stereo.cu, csrc/ft_fisheye.cu) via the C ABI.
``engine`` / ``pool`` arguments are accepted for signature compatibility and
ignored: the device is the engine.

ORB-SLAM-style aliases: ``compute_stereo_matches`` (pinhole: phase 1 ->
phase 2 | from-candidates -> reject, ONE launch) and
``compute_stereo_fisheye_matches``.
"""

from __future__ import annotations

from types import SimpleNamespace

import numpy as np

from . import _lib
from .types import StereoMatchConfig, StereoMatches

__all__ = ["StereoMatchConfig", "StereoMatches", "build_row_buckets", "match_pinhole_phase1",
           "refine_match_phase2", "matches_from_candidates", "reject_outliers",
           "triangulate_rays", "match_fisheye", "matches_to_csv_rows",
           "compute_stereo_matches", "compute_stereo_fisheye_matches"]


def build_row_buckets(v: np.ndarray, height: int) -> tuple[np.ndarray, np.ndarray]:
    """CSR of keypoint indices by rounded row (reference stereo.py:67-74).

    Provided for API completeness; the device kernels build the same buckets
    in shared memory and never call this."""
    rows = np.clip(np.round(np.asarray(v)).astype(np.int64), 0, height - 1)
    order = np.argsort(rows, kind="stable")
    start = np.zeros(height + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=height), out=start[1:])
    return start, order.astype(np.int64)


def _empty_matches(n: int) -> StereoMatches:
    return StereoMatches(right_idx=np.empty(n, np.int64), distance=np.empty(n, np.int64),
                         disparity=np.empty(n), refined_u=np.empty(n), depth=np.empty(n),
                         sad=np.empty(n, np.int64))


def _run_stereo(mode: int, left, right, cam, cfg, scale_pow, height: int,
                left_pyr=None, right_pyr=None, cand=None, matches=None,
                out_cand=None):
    """One ft_session_stereo call: pack -> H2D -> ft_stereo_pinhole -> D2H,
    with the reference objects' arrays passed in place (csrc/ft_session.cu).
    Returns (matches or None, cand_idx, cand_dist)."""
    from . import session as S
    ses = S.session()
    n = len(left.u)
    keep: list = []
    lf = S.features(left, keep=keep)
    rf = lf if right is left else S.features(right, keep=keep)
    pl = pr = None
    if mode & _lib.FT_STEREO_REFINE:
        pl, pr = S.pyramid(left_pyr, keep), S.pyramid(right_pyr, keep)
    params = S.stereo_params(cfg, height, scale_pow, getattr(cam, "baseline_times_fx", 1.0))
    if cand is not None:
        ci, cd = np.ascontiguousarray(cand[0], np.int64), np.ascontiguousarray(cand[1], np.int64)
    elif out_cand is not None:
        ci, cd = out_cand
    else:
        ci = cd = None
    res = None
    if matches is not None:
        res = matches
    elif mode & ~_lib.FT_STEREO_PHASE1:
        res = S.empty_matches(n)
    ms = S.matches_struct(res) if res is not None else None
    with ses.lock:
        st = ses.lib.ft_session_stereo(ses.handle, lf, rf, pl, pr, params, mode,
                                       ci.ctypes.data if ci is not None else None,
                                       cd.ctypes.data if cd is not None else None, ms)
    _lib.check(st, "ft_session_stereo")
    return res, ci, cd


def match_pinhole_phase1(left, right, height: int, scale_pow: np.ndarray,
                         cfg: StereoMatchConfig, engine=None, row_buckets=None,
                         out_idx: np.ndarray | None = None,
                         out_dist: np.ndarray | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Best-candidate right index (or -1) and distance per left keypoint
    (reference stereo.py:77-103 -> kernels.py:300-345).

    ``row_buckets`` is accepted for compatibility; the kernel rebuilds the
    buckets of ``build_row_buckets`` on the device (same rows, same sets)."""
    n = len(left.u)
    idx = out_idx if out_idx is not None else np.empty(n, dtype=np.int64)
    dist = out_dist if out_dist is not None else np.empty(n, dtype=np.int64)
    if n == 0:
        return idx, dist
    direct = (idx.dtype == np.int64 and dist.dtype == np.int64 and idx.flags.c_contiguous
              and dist.flags.c_contiguous and len(idx) >= n and len(dist) >= n)
    ci, cd = (idx, dist) if direct else (np.empty(n, np.int64), np.empty(n, np.int64))
    _run_stereo(_lib.FT_STEREO_PHASE1, left, right, None, cfg, scale_pow, height,
                out_cand=(ci, cd))
    if not direct:
        idx[:n] = ci
        dist[:n] = cd
    return idx, dist


def refine_match_phase2(left_pyr, right_pyr, left, right, cand_idx: np.ndarray,
                        cand_dist: np.ndarray, cam, cfg: StereoMatchConfig,
                        engine=None) -> StereoMatches:
    """Sub-pixel SAD refinement of phase-1 candidates (reference
    stereo.py:106-140 -> kernels.py:351-428)."""
    n = len(left.u)
    if n == 0:
        z = np.zeros(0)
        zi = np.zeros(0, dtype=np.int64)
        return StereoMatches(zi.copy(), zi.copy(), z.copy(), z.copy(), z.copy(), zi.copy())
    scale_pow = left_pyr.scale ** np.arange(len(left_pyr.widths), dtype=np.float64)
    res, _, _ = _run_stereo(_lib.FT_STEREO_REFINE, left, right, cam, cfg, scale_pow,
                            int(cam.height), left_pyr, right_pyr,
                            cand=(np.asarray(cand_idx), np.asarray(cand_dist)))
    return res


def matches_from_candidates(cand_idx: np.ndarray, cand_dist: np.ndarray, left, right, cam,
                            cfg: StereoMatchConfig) -> StereoMatches:
    """Accept phase-1 candidates at their raw disparity (reference
    stereo.py:143-168)."""
    n = len(cand_idx)
    if n == 0:
        z = np.zeros(0)
        zi = np.zeros(0, dtype=np.int64)
        return StereoMatches(zi.copy(), zi.copy(), z.copy(), z.copy(), z.copy(), zi.copy())
    res, _, _ = _run_stereo(_lib.FT_STEREO_FROM_CAND, left, right, cam, cfg, np.ones(1),
                            int(getattr(cam, "height", 1)),
                            cand=(np.asarray(cand_idx), np.asarray(cand_dist)))
    return res


def reject_outliers(matches: StereoMatches, cfg: StereoMatchConfig) -> StereoMatches:
    """Drop matches whose SAD exceeds outlier_multiplier x median, in place
    (reference stereo.py:171-188).  SADs must lie in [0, 2^32)."""
    m = matches.right_idx >= 0
    if not m.any():
        return matches

    n = len(matches.right_idx)
    names = ("right_idx", "distance", "disparity", "refined_u", "depth", "sad")
    types = (np.int64, np.int64, np.float64, np.float64, np.float64, np.int64)
    direct = all(getattr(matches, k).dtype == t and getattr(matches, k).flags.c_contiguous and
                 getattr(matches, k).flags.writeable for k, t in zip(names, types))
    work = matches if direct else StereoMatches(*(np.ascontiguousarray(getattr(matches, k), t)
                                                  for k, t in zip(names, types)))
    counts = SimpleNamespace(u=np.zeros(n), v=np.zeros(n), octave=np.zeros(n, np.int32),
                             descriptors=np.zeros((0, 4), np.uint64))
    _run_stereo(_lib.FT_STEREO_REJECT, counts, counts, None, cfg, np.ones(1), 1, matches=work)
    if not direct:  # in place, as the reference (stereo.py:181-188)
        for k in names:
            getattr(matches, k)[...] = getattr(work, k)
    return matches


def compute_stereo_matches(left, right, cam, cfg: StereoMatchConfig | None = None,
                           scale_pow: np.ndarray | None = None, left_pyr=None,
                           right_pyr=None) -> StereoMatches:
    """ORB-SLAM ComputeStereoMatches: the reference tracker's pinhole
    ``_run_stereo`` (tracker.py:415-427) as ONE fused launch -- phase 1, then
    phase 2 when pyramids are given (else matches_from_candidates), then
    reject_outliers."""
    cfg = cfg or StereoMatchConfig()
    if scale_pow is None:
        scale_pow = (left_pyr.scale ** np.arange(len(left_pyr.widths), dtype=np.float64)
                     if left_pyr is not None else 1.2 ** np.arange(8, dtype=np.float64))
    n = len(left.u)
    if n == 0:
        return StereoMatches(*(np.zeros(0, dtype=t) for t in (np.int64, np.int64, np.float64,
                                                              np.float64, np.float64, np.int64)))
    mode = _lib.FT_STEREO_PHASE1 | _lib.FT_STEREO_REJECT
    mode |= _lib.FT_STEREO_REFINE if left_pyr is not None else _lib.FT_STEREO_FROM_CAND
    res, _, _ = _run_stereo(mode, left, right, cam, cfg, scale_pow, int(cam.height), left_pyr,
                            right_pyr)
    return res


# ---------------------------------------------------------------------------
# fisheye

def triangulate_rays(origin_a, dir_a, origin_b, dir_b):
    """Midpoint of the shortest segment between two rays, None when
    parallel (reference stereo.py:191-197, including its solve at :207-216)."""
    pt, _, _, _ = _closest_ray_points(origin_a, dir_a, origin_b, dir_b)
    return pt


def _closest_ray_points(oa, da, ob, db):
    # Host-side restatement of reference stereo.py:200-220, kept term for term
    # (including the sign of t at :216, which the reference tracker's output
    # depends on).
    da = np.asarray(da, dtype=np.float64)
    db = np.asarray(db, dtype=np.float64)
    oa = np.asarray(oa, dtype=np.float64)
    ob = np.asarray(ob, dtype=np.float64)
    if np.linalg.norm(np.cross(da, db)) < 1e-9:
        return None, None, None, None
    r = ob - oa
    a11, a12, a22 = da @ da, da @ db, db @ db
    b1, b2 = da @ r, db @ r
    den = a11 * a22 - a12 * a12
    s = (b1 * a22 - a12 * b2) / den
    t = (a11 * b2 - a12 * b1) / den
    pa = oa + s * da
    pb = ob + t * db
    gap = float(np.linalg.norm(pa - pb))
    return (pa + pb) / 2.0, gap, s, t


def fisheye_tri_params(cam, cfg: StereoMatchConfig, corrected: bool = False) -> _lib.FtFisheyeTri:
    """ft_fisheye_tri from a FisheyeCamera (cameras.py:100-157) and the config;
    the right->left transform is right_extrinsic.inverse() as the reference
    computes it (geometry.py:84-86, stereo.py:247)."""
    t = _lib.FtFisheyeTri()
    for k in ("fx", "fy", "cx", "cy", "k1", "k2", "k3", "k4"):
        setattr(t, k, float(getattr(cam, k)))
    rot_rl = np.asarray(cam.right_extrinsic.rotation, dtype=np.float64)
    tr_rl = np.asarray(cam.right_extrinsic.translation, dtype=np.float64)
    rot_lr = rot_rl.T
    tr_lr = -rot_lr @ tr_rl
    t.rot_rl[:] = [float(x) for x in rot_rl.reshape(9)]
    t.trans_rl[:] = [float(x) for x in tr_rl]
    t.rot_lr[:] = [float(x) for x in np.ascontiguousarray(rot_lr).reshape(9)]
    t.trans_lr[:] = [float(x) for x in tr_lr]
    t.ray_gap_ceiling = float(cfg.ray_gap_ceiling)
    t.corrected = 1 if corrected else 0
    return t


def _fisheye_device(left, right, cfg: StereoMatchConfig, tri):
    """One ft_session_fisheye call (ft_stereo_fisheye_bf when tri is None,
    else ft_stereo_fisheye) -> (idx, dist[, ok, points])."""
    from . import session as S
    ses = S.session()
    n = len(left.u)
    keep: list = []
    lf, rf = S.features(left, keep=keep), S.features(right, keep=keep)
    idx, dist = np.empty(n, np.int64), np.empty(n, np.int64)
    ok = np.empty(n, np.int32) if tri is not None else None
    pts = np.empty((n, 3)) if tri is not None else None
    with ses.lock:
        st = ses.lib.ft_session_fisheye(ses.handle, lf, rf, int(cfg.t_match), float(cfg.ratio),
                                        tri, idx.ctypes.data, dist.ctypes.data,
                                        ok.ctypes.data if ok is not None else None,
                                        pts.ctypes.data if pts is not None else None)
    _lib.check(st, "ft_session_fisheye")
    if tri is None:
        return idx, dist
    return idx, dist, ok, pts


def fisheye_bruteforce(left, right, cfg: StereoMatchConfig) -> tuple[np.ndarray, np.ndarray]:
    """kernels.py:434-464 over all left keypoints on the device: (idx, dist)."""
    return _fisheye_device(left, right, cfg, None)


def match_fisheye(left, right, cam, cfg: StereoMatchConfig, engine=None, corrected: bool = False
                  ) -> tuple[np.ndarray, np.ndarray, np.ndarray, np.ndarray]:
    """Brute-force fisheye matching plus ray-midpoint triangulation
    (reference stereo.py:223-273), both on the B200 in one launch
    (ft_stereo_fisheye).  corrected=False reproduces the reference's closest-
    point solve including the sign of t at stereo.py:216 (its tracker's
    behaviour); corrected=True uses the least-squares solution."""
    n = len(left.u)
    empty = (np.empty(0, dtype=np.int64), np.empty(0, dtype=np.int64), np.empty((0, 3)),
             np.empty(0, dtype=np.int64))
    if n == 0 or len(right.u) == 0:
        return empty
    idx, dist, ok, pts = _fisheye_device(left, right, cfg,
                                         fisheye_tri_params(cam, cfg, corrected))
    keep = np.nonzero(ok)[0]
    if len(keep) == 0:
        return empty
    return keep.astype(np.int64), idx[keep], pts[keep], dist[keep]


def compute_stereo_fisheye_matches(left, right, cam, cfg: StereoMatchConfig | None = None,
                                   corrected: bool = False) -> StereoMatches:
    """ORB-SLAM ComputeStereoFishEyeMatches: the reference tracker's fisheye
    ``_run_stereo`` branch (tracker.py:399-414) -> per-left StereoMatches."""
    cfg = cfg or StereoMatchConfig()
    lidx, ridx, points, dists = match_fisheye(left, right, cam, cfg, corrected=corrected)
    n = len(left.u)
    out = StereoMatches(right_idx=np.full(n, -1, dtype=np.int64),
                        distance=np.full(n, 10000, dtype=np.int64), disparity=np.zeros(n),
                        refined_u=np.zeros(n), depth=np.zeros(n), sad=np.zeros(n, dtype=np.int64))
    out.right_idx[lidx] = ridx
    out.distance[lidx] = dists
    out.depth[lidx] = points[:, 2] if len(points) else 0.0
    return out


def matches_to_csv_rows(matches: StereoMatches) -> list[str]:
    """'left_idx,right_idx,disparity,depth,distance' per matched pair
    (reference stereo.py:276-283)."""
    return [f"{i},{matches.right_idx[i]},{matches.disparity[i]:.6f},"
            f"{matches.depth[i]:.6f},{matches.distance[i]}"
            for i in np.nonzero(matches.right_idx >= 0)[0]]
