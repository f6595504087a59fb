"""Generate the golden fixtures under tests/golden/ by running the REFERENCE.

Test infrastructure only.  Runs in the build container, where the reference
package `trackfront` is importable from /root/reference/pkg/src; the GPU box
has no /root/reference, so the outputs are committed as compressed .npz files
and the tests read those.

    NUMBA_CACHE_DIR=/tmp/numba_cache PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_golden.py

Every fixture stores the exact inputs handed to the reference stage functions
and the reference outputs (numba CPU path, ExecutionEngine("seq")).  Recipes
follow SURVEY.md §8(d):

* cfg1  rendered 752x480 pinhole pair -> extract_features (ORB, 1200 kps, 8
        levels) -> match_pinhole_phase1 -> refine_match_phase2 -> reject_outliers
        (reference stereo.py:77-188, kernels.py:300-428)
* cfg2  feature-bundle frame (seed 3) + 5k-point local map (rng 7) ->
        phase1 + matches_from_candidates + reject_outliers, run_phase_a,
        resolve_conflicts, search_by_projection (plain / rotation-checked /
        skip-masked), search_local_points (projection.py:118-221,
        localmap.py:79-122)
* cfg3  TUM-VI-shaped fisheye pair (seed 5) -> bruteforce_match_kernel,
        match_fisheye (with the reference's triangulation), fisheye
        search_local_points on a 3050-point map (rng 9)
* small known-answer / edge cases: ties,
        duplicates, empty inputs, single candidates.
"""

from __future__ import annotations

import json
import math
import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
if REF_SRC not in sys.path:
    sys.path.insert(0, REF_SRC)

from trackfront import kernels  # noqa: E402
from trackfront.cameras import FisheyeCamera, PinholeCamera  # noqa: E402
from trackfront.descriptors import random_descriptors  # noqa: E402
from trackfront.engine import ExecutionEngine  # noqa: E402
from trackfront.extraction import ExtractionConfig, extract_features  # noqa: E402
from trackfront.geometry import Pose, so3_exp  # noqa: E402
from trackfront.localmap import LocalMap, search_local_points  # noqa: E402
from trackfront.mapping import (Frame, FrameGrid, MapPointSoA, NO_POINT)  # noqa: E402
from trackfront.projection import (ProjectionSearchConfig, resolve_conflicts,  # noqa: E402
                                   run_phase_a, search_by_projection)
from trackfront.stereo import (StereoMatchConfig, match_fisheye,  # noqa: E402
                               match_pinhole_phase1, matches_from_candidates,
                               refine_match_phase2, reject_outliers)
from trackfront.synthetic import (SyntheticSceneConfig, _octave_from_distance,  # noqa: E402
                                  default_pinhole, generate_synthetic)

ENGINE = ExecutionEngine("seq")


def feats_dict(prefix: str, f) -> dict:
    return {
        f"{prefix}_u": np.ascontiguousarray(f.u, dtype=np.float64),
        f"{prefix}_v": np.ascontiguousarray(f.v, dtype=np.float64),
        f"{prefix}_octave": np.ascontiguousarray(f.octave, dtype=np.int32),
        f"{prefix}_angle": np.ascontiguousarray(f.angle, dtype=np.float64),
        f"{prefix}_response": np.ascontiguousarray(f.response, dtype=np.float32),
        f"{prefix}_desc": np.ascontiguousarray(f.descriptors, dtype=np.uint64),
    }


def soa_dict(prefix: str, s: MapPointSoA) -> dict:
    return {
        f"{prefix}_positions": np.ascontiguousarray(s.positions),
        f"{prefix}_descriptors": np.ascontiguousarray(s.descriptors),
        f"{prefix}_normals": np.ascontiguousarray(s.normals),
        f"{prefix}_min_d": np.ascontiguousarray(s.min_distances),
        f"{prefix}_max_d": np.ascontiguousarray(s.max_distances),
        f"{prefix}_ids": np.ascontiguousarray(s.point_ids),
    }


def matches_dict(prefix: str, m) -> dict:
    return {
        f"{prefix}_right_idx": m.right_idx.copy(),
        f"{prefix}_distance": m.distance.copy(),
        f"{prefix}_disparity": m.disparity.copy(),
        f"{prefix}_refined_u": m.refined_u.copy(),
        f"{prefix}_depth": m.depth.copy(),
        f"{prefix}_sad": m.sad.copy(),
    }


def corr_dict(prefix: str, c) -> dict:
    return {
        f"{prefix}_point_idx": c.point_idx.copy(),
        f"{prefix}_keypoint_idx": c.keypoint_idx.copy(),
        f"{prefix}_distance": c.distance.copy(),
        f"{prefix}_octave": c.octave.copy(),
    }


def flip_bits(desc: np.ndarray, rng: np.random.Generator, nflip: int) -> np.ndarray:
    out = desc.copy()
    for i in range(len(out)):
        bits = rng.choice(256, size=nflip, replace=False)
        for b in bits:
            out[i, b >> 6] ^= np.uint64(1) << np.uint64(b & 63)
    return out


def build_local_map(seq, frame_idx: int, cam, total: int, rng, scfg) -> MapPointSoA:
    """All landmarks visible in the left view plus uniformly drawn others
    (SURVEY.md §8(d) cfg2 recipe)."""
    visible = seq.frames[frame_idx].landmark_ids_left
    others = np.setdiff1d(np.arange(len(seq.landmarks)), visible)
    extra = total - len(visible)
    if extra > 0:
        pick = rng.choice(others, size=min(extra, len(others)), replace=False)
        ids = np.sort(np.concatenate([visible, pick]))
    else:
        ids = np.sort(visible)
    pose_wc = seq.gt_poses[frame_idx]
    center = pose_wc.translation
    pos = seq.landmarks[ids]
    d = np.linalg.norm(pos - center, axis=1)
    normals = (pos - center) / d[:, None]
    octs = _octave_from_distance(d, scfg).astype(np.float64)
    max_d = d * (scfg.scale ** octs)
    min_d = max_d / (scfg.scale ** (scfg.levels - 1))
    desc = flip_bits(seq.landmark_desc[ids], rng, 8)
    return MapPointSoA(positions=pos.copy(), descriptors=desc, normals=normals,
                       min_distances=min_d, max_distances=max_d,
                       point_ids=ids.astype(np.int64))


def perturbed_pose(seq, frame_idx: int) -> Pose:
    gt = seq.pose_cw(frame_idx)
    rot = so3_exp(np.array([0.002, -0.001, 0.001])) @ gt.rotation
    return Pose(rot, gt.translation + np.array([0.01, 0.0, -0.01]))


def make_frame(fid, left, right, cam, pose, cell_px=48) -> Frame:
    grid = FrameGrid(left.u, left.v, cam.width, cam.height, cell_px)
    return Frame(fid, 0.0, left, right, np.full(len(left), -1.0),
                 np.full(len(left), NO_POINT, dtype=np.int64), pose, grid)


def pose_dict(prefix: str, p: Pose) -> dict:
    return {f"{prefix}_rot": p.rotation.copy(), f"{prefix}_trans": p.translation.copy()}


# ---------------------------------------------------------------------------

def gen_hamming() -> None:
    rng = np.random.default_rng(12345)
    n = 1024
    a = random_descriptors(rng, n)
    b = random_descriptors(rng, n)
    b[:64] = a[:64]            # distance 0
    b[64:128] = ~a[64:128]     # distance 256
    out = np.empty(n, dtype=np.int64)
    kernels.hamming_pairs_kernel(a, b, out, 0, n)
    np.savez_compressed(OUT / "hamming.npz", a=a, b=b, out=out)


def gen_cfg1() -> dict:
    scfg = SyntheticSceneConfig(landmark_count=8000, n_frames=2, trajectory="line")
    seq = generate_synthetic(scfg, seed=11)
    img_l, img_r = seq.render_pair(0)
    ecfg = ExtractionConfig()
    left, pyr_l = extract_features(img_l, ecfg, ENGINE)
    right, pyr_r = extract_features(img_r, ecfg, ENGINE)
    cam = seq.cam
    scfg_st = StereoMatchConfig()
    scale_pow = ecfg.scale_powers()
    idx, dist = match_pinhole_phase1(left, right, cam.height, scale_pow, scfg_st, ENGINE)
    m2 = refine_match_phase2(pyr_l, pyr_r, left, right, idx, dist, cam, scfg_st, ENGINE)
    pre = matches_dict("p2", m2)
    m3 = reject_outliers(m2, scfg_st)
    d = {}
    d.update(feats_dict("left", left))
    d.update(feats_dict("right", right))
    d.update(pyr_l_data=pyr_l.data.copy(), pyr_l_offsets=pyr_l.offsets.copy(),
             pyr_l_widths=pyr_l.widths.copy(), pyr_l_heights=pyr_l.heights.copy(),
             pyr_r_data=pyr_r.data.copy(), pyr_r_offsets=pyr_r.offsets.copy(),
             pyr_r_widths=pyr_r.widths.copy(), pyr_r_heights=pyr_r.heights.copy(),
             scale_pow=scale_pow, p1_idx=idx.copy(), p1_dist=dist.copy())
    d.update(pre)
    d.update(matches_dict("final", m3))
    np.savez_compressed(OUT / "cfg1_stereo.npz", **d)
    return {"cfg1": {"n_left": len(left), "n_right": len(right),
                     "p1_candidates": int((idx >= 0).sum()),
                     "final_matches": int((m3.right_idx >= 0).sum())}}


def gen_cfg2() -> dict:
    scfg = SyntheticSceneConfig(landmark_count=12000, n_frames=2, trajectory="line",
                                keypoint_noise_px=0.5)
    seq = generate_synthetic(scfg, seed=3)
    cam = seq.cam
    fr = seq.frames[0]
    left, right = fr.left, fr.right
    scfg_st = StereoMatchConfig()
    scale_pow = scfg.scale ** np.arange(scfg.levels, dtype=np.float64)
    idx, dist = match_pinhole_phase1(left, right, cam.height, scale_pow, scfg_st, ENGINE)
    m = matches_from_candidates(idx, dist, left, right, cam, scfg_st)
    pre = matches_dict("fc", m)
    m = reject_outliers(m, scfg_st)
    rng = np.random.default_rng(7)
    soa = build_local_map(seq, 0, cam, 5000, rng, scfg)
    pose = perturbed_pose(seq, 0)
    pcfg = ProjectionSearchConfig()
    frame = make_frame(0, left, right, cam, pose)
    kp, kd, ko = run_phase_a(soa, frame, pose, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    kp, kd, ko = kp.copy(), kd.copy(), ko.copy()
    corr = resolve_conflicts(kp, kd, ko)
    # rotation-checked, prev-frame style search (window 15, u_offset +1)
    ref_angles = np.random.default_rng(17).uniform(0.0, 2 * math.pi, len(soa))
    # bias: most points keep their true angle so the histogram is peaked
    lm_angle = seq.landmark_angle[soa.point_ids]
    keep = np.random.default_rng(18).uniform(size=len(soa)) < 0.8
    ref_angles = np.where(keep, lm_angle, ref_angles)
    corr_rot = search_by_projection(soa, frame, pose, cam, pcfg, scfg.scale, scfg.levels,
                                    ENGINE, ref_angles=ref_angles, rotation_check=True,
                                    window_px=pcfg.window_prev_px, u_offset=1.0)
    # skip-masked variant
    skip = (np.random.default_rng(19).uniform(size=len(soa)) < 0.3).astype(np.uint8)
    corr_skip = search_by_projection(soa, frame, pose, cam, pcfg, scfg.scale, scfg.levels,
                                     ENGINE, skip_mask=skip)
    # search_local_points on a fresh frame
    local = LocalMap((0,), soa.point_ids.copy(), soa)
    frame_a = make_frame(0, left, right, cam, pose)
    count_a = search_local_points(local, frame_a, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    # ... and on a frame with pre-filled slots (skip mask + "only if empty")
    frame_b = make_frame(0, left, right, cam, pose)
    prng = np.random.default_rng(23)
    pre_k = prng.choice(len(left), size=200, replace=False)
    pre_ids = prng.choice(soa.point_ids, size=200, replace=False)
    frame_b.slots[pre_k] = pre_ids
    slots_b_in = frame_b.slots.copy()
    count_b = search_local_points(local, frame_b, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    d = {}
    d.update(feats_dict("left", left))
    d.update(feats_dict("right", right))
    d.update(soa_dict("map", soa))
    d.update(pose_dict("pose", pose))
    d.update(scale_pow=scale_pow, p1_idx=idx.copy(), p1_dist=dist.copy())
    d.update(pre)
    d.update(matches_dict("final", m))
    d.update(pa_kp=kp, pa_dist=kd, pa_oct=ko, ref_angles=ref_angles, skip=skip)
    d.update(corr_dict("corr", corr))
    d.update(corr_dict("corr_rot", corr_rot))
    d.update(corr_dict("corr_skip", corr_skip))
    d.update(slots_a=frame_a.slots.copy(), count_a=np.int64(count_a),
             slots_b_in=slots_b_in, slots_b=frame_b.slots.copy(), count_b=np.int64(count_b),
             grid_start=frame.grid.start.copy(), grid_indices=frame.grid.indices.copy())
    np.savez_compressed(OUT / "cfg2_frame_map.npz", **d)
    return {"cfg2": {"n_left": len(left), "n_right": len(right), "map": len(soa),
                     "claims": int((kp >= 0).sum()), "corr": len(corr),
                     "corr_rot": len(corr_rot), "corr_skip": len(corr_skip),
                     "count_a": int(count_a), "count_b": int(count_b),
                     "stereo_matches": int((m.right_idx >= 0).sum())}}


def fisheye_cam() -> FisheyeCamera:
    return FisheyeCamera(fx=190.0, fy=190.0, cx=256.0, cy=256.0,
                         k1=0.003, k2=-0.002, k3=0.001, k4=-0.0005,
                         width=512, height=512,
                         right_extrinsic=Pose(np.eye(3), np.array([-0.1, 0.0, 0.0])))


def gen_cfg3() -> dict:
    cam = fisheye_cam()
    scfg = SyntheticSceneConfig(landmark_count=3050, n_frames=2, trajectory="line",
                                keypoint_noise_px=0.3)
    seq = generate_synthetic(scfg, seed=5, cam=cam)
    fr = seq.frames[0]
    left, right = fr.left, fr.right
    scfg_st = StereoMatchConfig()
    idx = np.empty(len(left), dtype=np.int64)
    dist = np.empty(len(left), dtype=np.int64)
    kernels.bruteforce_match_kernel(left.descriptors, right.descriptors, scfg_st.t_match,
                                    scfg_st.ratio, 0, len(left), idx, dist)
    lidx, ridx, pts, dists = match_fisheye(left, right, cam, scfg_st, ENGINE)
    rng = np.random.default_rng(9)
    soa = build_local_map(seq, 0, cam, 3050, rng, scfg)
    pose = perturbed_pose(seq, 0)
    pcfg = ProjectionSearchConfig()
    frame = make_frame(0, left, right, cam, pose)
    kp, kd, ko = run_phase_a(soa, frame, pose, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    kp, kd, ko = kp.copy(), kd.copy(), ko.copy()
    corr = resolve_conflicts(kp, kd, ko)
    local = LocalMap((0,), soa.point_ids.copy(), soa)
    frame_a = make_frame(0, left, right, cam, pose)
    count_a = search_local_points(local, frame_a, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    d = {}
    d.update(feats_dict("left", left))
    d.update(feats_dict("right", right))
    d.update(soa_dict("map", soa))
    d.update(pose_dict("pose", pose))
    d.update(bf_idx=idx, bf_dist=dist, mf_lidx=lidx, mf_ridx=ridx, mf_pts=pts, mf_dists=dists)
    d.update(pa_kp=kp, pa_dist=kd, pa_oct=ko)
    d.update(corr_dict("corr", corr))
    d.update(slots_a=frame_a.slots.copy(), count_a=np.int64(count_a))
    np.savez_compressed(OUT / "cfg3_fisheye.npz", **d)
    return {"cfg3": {"n_left": len(left), "n_right": len(right), "map": len(soa),
                     "bf_accepted": int((idx >= 0).sum()), "mf_accepted": len(lidx),
                     "claims": int((kp >= 0).sum()), "corr": len(corr),
                     "count_a": int(count_a)}}


def gen_edge() -> dict:
    """Tie / multiplicity / duplicate cases run through the reference kernels."""
    rng = np.random.default_rng(99)
    out = {}
    # brute force with heavy duplication: right set has repeated descriptors
    base = random_descriptors(rng, 40)
    left = base[rng.integers(0, 40, size=300)]
    right = base[rng.integers(0, 40, size=257)]
    right[::7] = ~right[::7]
    idx = np.empty(len(left), dtype=np.int64)
    dist = np.empty(len(left), dtype=np.int64)
    kernels.bruteforce_match_kernel(left, right, 100, 0.8, 0, len(left), idx, dist)
    out.update(dup_left=left, dup_right=right, dup_idx=idx, dup_dist=dist)
    # single right candidate (second stays at 100000)
    one_r = base[:1]
    idx1 = np.empty(len(left), dtype=np.int64)
    dist1 = np.empty(len(left), dtype=np.int64)
    kernels.bruteforce_match_kernel(left, one_r, 100, 0.8, 0, len(left), idx1, dist1)
    out.update(one_right=one_r, one_idx=idx1, one_dist=dist1)
    # phase 1 with coarse rows, many equal distances (low-entropy descriptors)
    n = 500
    small = random_descriptors(rng, 6)
    lu = rng.uniform(50, 700, n)
    lv = np.round(rng.uniform(0, 479, n) * 2) / 2  # half-integer rows: rounding ties
    ru = lu - rng.uniform(-5, 60, n)
    rv = lv + rng.normal(0, 1.0, n)
    rv[::5] = lv[::5]
    loct = rng.integers(0, 8, n).astype(np.int32)
    roct = np.clip(loct + rng.integers(-2, 3, n), 0, 7).astype(np.int32)
    ld = small[rng.integers(0, 6, n)]
    rd = small[rng.integers(0, 6, n)]
    from trackfront.mapping import FeatureSet
    lf = FeatureSet(lu, lv, loct, np.zeros(n), np.zeros(n, np.float32), ld)
    rf = FeatureSet(ru, rv, roct, np.zeros(n), np.zeros(n, np.float32), rd)
    sp = 1.2 ** np.arange(8, dtype=np.float64)
    p_idx, p_dist = match_pinhole_phase1(lf, rf, 480, sp, StereoMatchConfig(), ENGINE)
    out.update(tie_lu=lu, tie_lv=lv, tie_ru=ru, tie_rv=rv, tie_loct=loct, tie_roct=roct,
               tie_ld=ld, tie_rd=rd, tie_idx=p_idx.copy(), tie_dist=p_dist.copy())
    # reject_outliers median on even / odd counts
    from trackfront.stereo import StereoMatches
    sads = []
    for cnt in (1, 2, 7, 8, 101, 1000):
        s = rng.integers(0, 5000, cnt).astype(np.int64)
        s[: max(1, cnt // 10)] *= 7
        k = np.arange(cnt)
        mm = StereoMatches(right_idx=k.copy(), distance=np.full(cnt, 5, np.int64),
                           disparity=np.full(cnt, 3.0), refined_u=np.full(cnt, 1.0),
                           depth=np.full(cnt, 2.0), sad=s.copy())
        mm.right_idx[::9] = -1
        rin = mm.right_idx.copy()
        reject_outliers(mm, StereoMatchConfig())
        out[f"med{cnt}_sad"] = s
        out[f"med{cnt}_rin"] = rin
        out[f"med{cnt}_rout"] = mm.right_idx.copy()
        out[f"med{cnt}_sadout"] = mm.sad.copy()
        sads.append(cnt)
    np.savez_compressed(OUT / "edge_cases.npz", **out)
    return {"edge": {"dup_accepted": int((idx >= 0).sum()), "tie_matched": int((p_idx >= 0).sum()),
                     "median_counts": sads}}


# Non-default configs (tests/test_gpu_parity.py STEREO_CFGS / PROJ_CFGS).
STEREO_SWEEP = [
    dict(t_match=40),
    dict(band_factor=1.0, half_window=3, half_slide=3),
    dict(band_factor=3.5, half_window=7, half_slide=8, outlier_multiplier=1.5),
    dict(min_disparity=2.0, max_disparity=60.0, outlier_multiplier=4.0),
    dict(t_match=256, half_window=1, half_slide=1, ratio=0.6),
]
PROJ_SWEEP = [
    dict(window_px=2.0, t_proj=50),
    dict(window_px=12.0, ratio=0.7, view_cos_min=0.9),
    dict(window_px=30.0, ratio=1.0, view_cos_min=-1.0, t_proj=256),
    dict(histogram_bins=12, histogram_keep=1),
]
SCALES = [(1.2, 8), (1.3, 6), (2.0, 4)]


def _load(name):
    with np.load(OUT / name) as z:
        return {k: z[k] for k in z.files}


def _feats(d, prefix):
    from trackfront.mapping import FeatureSet
    return FeatureSet(u=d[f"{prefix}_u"], v=d[f"{prefix}_v"], octave=d[f"{prefix}_octave"],
                      angle=d[f"{prefix}_angle"], response=d[f"{prefix}_response"],
                      descriptors=d[f"{prefix}_desc"])


def _soa(d, prefix="map"):
    return MapPointSoA(positions=d[f"{prefix}_positions"], descriptors=d[f"{prefix}_descriptors"],
                       normals=d[f"{prefix}_normals"], min_distances=d[f"{prefix}_min_d"],
                       max_distances=d[f"{prefix}_max_d"], point_ids=d[f"{prefix}_ids"])


def _pyr(d, side, scale=1.2):
    from trackfront.extraction import ImagePyramid
    p = f"pyr_{side}"
    return ImagePyramid(d[f"{p}_data"], d[f"{p}_offsets"], d[f"{p}_widths"],
                        d[f"{p}_heights"], scale)


def _clip_octaves(f, levels):
    f.octave = np.minimum(np.asarray(f.octave), levels - 1).astype(np.int32)
    return f


def gen_sweeps() -> dict:
    """The reference on non-default StereoMatchConfig / ProjectionSearchConfig
    values and pyramid scales, over the committed cfg1 / cfg2 / cfg3 inputs
    (no new inputs except the scale-1.3 / 2.0 pyramids)."""
    d1, d2, d3 = _load("cfg1_stereo.npz"), _load("cfg2_frame_map.npz"), _load("cfg3_fisheye.npz")
    out, summ = {}, {}
    cam = default_pinhole()
    l1, r1 = _feats(d1, "left"), _feats(d1, "right")
    pl, pr = _pyr(d1, "l"), _pyr(d1, "r")
    l2, r2 = _feats(d2, "left"), _feats(d2, "right")
    sp = d1["scale_pow"]
    for k, kw in enumerate(STEREO_SWEEP):
        cfg = StereoMatchConfig(**kw)
        # cfg1: phase 1 -> phase 2 -> reject (rendered ORB frame)
        idx, dist = match_pinhole_phase1(l1, r1, cam.height, sp, cfg, ENGINE)
        m = reject_outliers(refine_match_phase2(pl, pr, l1, r1, idx, dist, cam, cfg, ENGINE), cfg)
        out.update(matches_dict(f"s{k}_cfg1", m))
        # cfg2: phase 1 -> from candidates -> reject (feature bundle)
        idx2, dist2 = match_pinhole_phase1(l2, r2, cam.height, sp, cfg, ENGINE)
        m2 = reject_outliers(matches_from_candidates(idx2, dist2, l2, r2, cam, cfg), cfg)
        out.update(matches_dict(f"s{k}_cfg2", m2))
        # cfg3 descriptors: fisheye brute force with this t_match / ratio
        bi = np.empty(len(d3["left_u"]), dtype=np.int64)
        bd = np.empty(len(d3["left_u"]), dtype=np.int64)
        kernels.bruteforce_match_kernel(d3["left_desc"], d3["right_desc"], cfg.t_match, cfg.ratio,
                                        0, len(bi), bi, bd)
        out.update({f"s{k}_bf_idx": bi, f"s{k}_bf_dist": bd})
        summ[f"stereo{k}"] = [int((m.right_idx >= 0).sum()), int((m2.right_idx >= 0).sum()),
                              int((bi >= 0).sum())]
    soa = _soa(d2)
    pose = Pose(d2["pose_rot"], d2["pose_trans"])
    ref_angles = np.random.default_rng(7).uniform(0, 2 * math.pi, len(soa))
    out["proj_ref_angles"] = ref_angles
    for k, kw in enumerate(PROJ_SWEEP):
        pcfg = ProjectionSearchConfig(**kw)
        for j, (scale, levels) in enumerate(SCALES):
            # fewer levels: the bundle's octaves clipped into the pyramid
            l2 = _clip_octaves(_feats(d2, "left"), levels)
            frame = make_frame(0, l2, r2, cam, pose)
            kp, kd, ko = run_phase_a(soa, frame, pose, cam, pcfg, scale, levels, ENGINE)
            kp, kd, ko = kp.copy(), kd.copy(), ko.copy()
            c = search_by_projection(soa, frame, pose, cam, pcfg, scale, levels, ENGINE,
                                     ref_angles=ref_angles, rotation_check=True, u_offset=-1.0)
            local = LocalMap((0,), soa.point_ids.copy(), soa)
            fa = make_frame(0, l2, r2, cam, pose)
            n = search_local_points(local, fa, cam, pcfg, scale, levels, ENGINE)
            t = f"p{k}_{j}"
            out.update({f"{t}_kp": kp, f"{t}_dist": kd, f"{t}_oct": ko, f"{t}_slots": fa.slots.copy(),
                        f"{t}_count": np.int64(n)})
            out.update(corr_dict(f"{t}_corr", c))
            summ[t] = [int((kp >= 0).sum()), len(c), int(n)]
    np.savez_compressed(OUT / "sweeps.npz", **out)
    return {"sweeps": summ}


def gen_scales() -> dict:
    """cfg1's rendered pair through the reference ORB extraction at pyramid
    scale 1.3 / 6 levels and 2.0 / 4 levels, then phase 1 -> 2 -> reject."""
    scfg = SyntheticSceneConfig(landmark_count=8000, n_frames=2, trajectory="line")
    seq = generate_synthetic(scfg, seed=11)
    img_l, img_r = seq.render_pair(0)
    cam = seq.cam
    out, summ = {}, {}
    for j, (scale, levels) in enumerate(SCALES[1:], start=1):
        ecfg = ExtractionConfig(scale=scale, levels=levels)
        left, pyr_l = extract_features(img_l, ecfg, ENGINE)
        right, pyr_r = extract_features(img_r, ecfg, ENGINE)
        cfg = StereoMatchConfig()
        sp = ecfg.scale_powers()
        idx, dist = match_pinhole_phase1(left, right, cam.height, sp, cfg, ENGINE)
        m = reject_outliers(refine_match_phase2(pyr_l, pyr_r, left, right, idx, dist, cam, cfg,
                                                ENGINE), cfg)
        t = f"x{j}"
        out.update(feats_dict(f"{t}_left", left))
        out.update(feats_dict(f"{t}_right", right))
        for side, p in (("l", pyr_l), ("r", pyr_r)):
            out.update({f"{t}_pyr_{side}_data": p.data.copy(), f"{t}_pyr_{side}_offsets": p.offsets.copy(),
                        f"{t}_pyr_{side}_widths": p.widths.copy(),
                        f"{t}_pyr_{side}_heights": p.heights.copy()})
        out.update({f"{t}_scale_pow": sp, f"{t}_p1_idx": idx.copy(), f"{t}_p1_dist": dist.copy()})
        out.update(matches_dict(f"{t}_final", m))
        summ[f"scale{scale}"] = {"levels": levels, "n_left": len(left),
                                 "octaves": np.bincount(left.octave, minlength=levels).tolist(),
                                 "p1": int((idx >= 0).sum()), "final": int((m.right_idx >= 0).sum())}
    np.savez_compressed(OUT / "scales.npz", **out)
    return {"scales": summ}


def gen_cfg5() -> dict:
    """2073-keypoint frame (landmark_count 20000, seed 3),
    20000-point local map: stereo (phase 1 + from candidates + reject) and
    search_local_points with 10 % of the keypoints pre-slotted."""
    scfg = SyntheticSceneConfig(landmark_count=20000, n_frames=2, trajectory="line",
                                keypoint_noise_px=0.5)
    seq = generate_synthetic(scfg, seed=3)
    cam = seq.cam
    fr = seq.frames[0]
    left, right = fr.left, fr.right
    cfg = StereoMatchConfig()
    sp = scfg.scale ** np.arange(scfg.levels, dtype=np.float64)
    idx, dist = match_pinhole_phase1(left, right, cam.height, sp, cfg, ENGINE)
    m = reject_outliers(matches_from_candidates(idx, dist, left, right, cam, cfg), cfg)
    soa = build_local_map(seq, 0, cam, 20000, np.random.default_rng(13), scfg)
    pose = perturbed_pose(seq, 0)
    pcfg = ProjectionSearchConfig()
    frame = make_frame(0, left, right, cam, pose)
    kp, kd, ko = run_phase_a(soa, frame, pose, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    kp, kd, ko = kp.copy(), kd.copy(), ko.copy()
    local = LocalMap((0,), soa.point_ids.copy(), soa)
    fb = make_frame(0, left, right, cam, pose)
    prng = np.random.default_rng(29)
    k = prng.choice(len(left), size=len(left) // 10, replace=False)
    fb.slots[k] = prng.choice(soa.point_ids, size=len(k), replace=False)
    slots_in = fb.slots.copy()
    n = search_local_points(local, fb, cam, pcfg, scfg.scale, scfg.levels, ENGINE)
    d = {}
    d.update(feats_dict("left", left))
    d.update(feats_dict("right", right))
    d.update(soa_dict("map", soa))
    d.update(pose_dict("pose", pose))
    d.update(scale_pow=sp, p1_idx=idx.copy(), p1_dist=dist.copy(), pa_kp=kp, pa_dist=kd,
             pa_oct=ko, slots_in=slots_in, slots=fb.slots.copy(), count=np.int64(n))
    d.update(matches_dict("final", m))
    np.savez_compressed(OUT / "cfg5_high_load.npz", **d)
    return {"cfg5": {"n_left": len(left), "n_right": len(right), "map": len(soa),
                     "visible_claims": int((kp >= 0).sum()), "count": int(n),
                     "stereo_matches": int((m.right_idx >= 0).sum())}}


def gen_prev() -> dict:
    """The reference's own search_prev_frame (projection.py:224-253) on cfg2:
    the previous frame's slots from its search_local_points, a world map of
    reference MapPoints, the current pose moved forward (u_offset +1), back
    (-1) and not at all (0); plus SPEC.md:352-353 static and empty cases."""
    from trackfront.mapping import MapPoint, WorldMap
    from trackfront.projection import search_prev_frame
    d2 = _load("cfg2_frame_map.npz")
    cam = default_pinhole()
    l2, r2 = _feats(d2, "left"), _feats(d2, "right")
    soa = _soa(d2)
    pose = Pose(d2["pose_rot"], d2["pose_trans"])
    world = WorldMap()
    for i, pid in enumerate(soa.point_ids):
        world.add_point(MapPoint(point_id=int(pid), position=soa.positions[i].copy(),
                                 descriptor=soa.descriptors[i].copy(),
                                 normal=soa.normals[i].copy(),
                                 min_distance=float(soa.min_distances[i]),
                                 max_distance=float(soa.max_distances[i])))
    pcfg = ProjectionSearchConfig()
    out, summ = {}, {}
    prev = make_frame(0, l2, r2, cam, pose)
    prev.slots[...] = d2["slots_a"]
    moves = {"fwd": np.array([0.002, -0.001, 0.004]), "back": np.array([-0.001, 0.002, -0.005]),
             "static": np.zeros(3)}
    for name, dt in moves.items():
        cur_pose = Pose(pose.rotation, pose.translation + dt)
        cur = make_frame(1, l2, r2, cam, cur_pose)
        corr, pids = search_prev_frame(prev, cur, cur_pose, world, cam, pcfg, 1.2, 8, ENGINE)
        out.update(corr_dict(f"{name}", corr))
        out[f"{name}_pids"] = np.asarray(pids).copy()
        out[f"{name}_trans"] = cur_pose.translation.copy()
        summ[name] = len(corr)
    # SPEC.md:352 static case: every slotted point re-matches its own keypoint
    st_k = out["static_keypoint_idx"]
    st_p = out["static_pids"][out["static_point_idx"]]
    summ["static_self_matches"] = int((prev.slots[st_k] == st_p).sum())
    empty = make_frame(0, l2, r2, cam, pose)
    corr, pids = search_prev_frame(empty, make_frame(1, l2, r2, cam, pose), pose, world, cam,
                                   pcfg, 1.2, 8, ENGINE)
    summ["empty"] = [len(corr), len(pids)]
    out["prev_slots"] = prev.slots.copy()
    np.savez_compressed(OUT / "prev_frame.npz", **out)
    return {"prev_frame": summ}


def digest(*arrays) -> np.ndarray:
    """sha256 over the raw bytes of the arrays (dtype + shape included), as
    32 uint8 -- a bit-exact check of outputs too large to commit."""
    import hashlib
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(a)
        h.update(str(a.dtype.str).encode())
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return np.frombuffer(h.digest(), dtype=np.uint8).copy()


def gen_cfg4(trajectory: str) -> dict:
    """BASELINE configs[3] / SURVEY §8(d) cfg4: the reference StereoTracker
    over a 100-frame feature-bundle sequence (tracker.py:225-393), every call
    of the hot-path stage functions captured (inputs, outputs).

    Compact form: keypoint descriptors / angles are the landmarks' (asserted
    below), so frames store landmark ids + u, v, octave; map points are the
    world's (immutable once created, ids 0..N-1), so a local map is a bitmask
    over the world table; outputs too large to commit are sha256 digests
    (golden_io.digest) next to compact copies of the indices."""
    import time
    import trackfront.tracker as T
    from trackfront.tracker import FrameInput, StereoTracker, TrackerConfig
    scfg = SyntheticSceneConfig(landmark_count=12000, n_frames=100, trajectory=trajectory,
                                keypoint_noise_px=0.5)
    seq = generate_synthetic(scfg, seed=4)
    n_lm = len(seq.landmarks)
    rec: dict[int, dict] = {}
    cur = {"f": -1}
    orig = {k: getattr(T, k) for k in ("match_pinhole_phase1", "matches_from_candidates",
                                        "reject_outliers", "search_prev_frame",
                                        "search_local_points", "update_local_map")}

    def slot(name):
        return rec.setdefault(cur["f"], {}).setdefault(name, {})

    def w_phase1(left, right, height, scale_pow, cfg, engine=None, **kw):
        idx, dist = orig["match_pinhole_phase1"](left, right, height, scale_pow, cfg, engine, **kw)
        slot("stereo").update(p1=digest(idx, dist))
        return idx, dist

    def w_fc(idx, dist, left, right, cam, cfg):
        m = orig["matches_from_candidates"](idx, dist, left, right, cam, cfg)
        slot("stereo").update(fc=digest(m.right_idx, m.distance, m.disparity, m.refined_u,
                                        m.depth, m.sad))
        return m

    def w_rej(m, cfg):
        out = orig["reject_outliers"](m, cfg)
        slot("stereo").update(final=digest(out.right_idx, out.distance, out.disparity,
                                           out.refined_u, out.depth, out.sad),
                              right_idx=out.right_idx.astype(np.int16),
                              distance=out.distance.astype(np.int16))
        return out

    def w_prev(prev, curf, pose, world, cam, cfg, scale, levels, engine=None, soa_out=None,
               pool=None):
        slots_in = prev.slots.copy()
        corr, pids = orig["search_prev_frame"](prev, curf, pose, world, cam, cfg, scale, levels,
                                               engine, soa_out=soa_out, pool=pool)
        slot("prev").update(prev_frame=prev.frame_id, prev_slots=slots_in.astype(np.int32),
                            prev_pose=np.concatenate([prev.pose.rotation.ravel(),
                                                      prev.pose.translation]),
                            pose=np.concatenate([pose.rotation.ravel(), pose.translation]),
                            n_corr=np.int64(len(corr)),
                            corr_digest=digest(corr.point_idx, corr.keypoint_idx, corr.distance,
                                               corr.octave),
                            pids=digest(pids))
        return corr, pids

    def w_local(local, frame, cam, cfg, scale, levels, engine=None, world=None, pool=None):
        before = frame.slots.copy()
        n = orig["search_local_points"](local, frame, cam, cfg, scale, levels, engine,
                                        world=world, pool=pool)
        mask = np.zeros(n_lm * 4, dtype=bool)  # world ids < landmarks x keyframes
        mask[np.asarray(local.point_ids, dtype=np.int64)] = True
        slot("local").update(slots_in=before.astype(np.int32), local_ids=local.point_ids.copy(),
                             pose=np.concatenate([frame.pose.rotation.ravel(),
                                                  frame.pose.translation]),
                             slots_out=digest(frame.slots),
                             count=np.int64(n))
        return n

    def w_update(frame, world, pool=None):
        slots_in = frame.slots.copy()
        local = orig["update_local_map"](frame, world, pool)
        soa = local.soa
        slot("update").update(slots_in=slots_in.astype(np.int32),
                              n_keyframes=np.int64(len(world.keyframes)),
                              n_points=np.int64(len(world.points)),
                              kf_ids=np.asarray(local.keyframe_ids, dtype=np.int32),
                              ids_digest=digest(np.asarray(local.point_ids, np.int64)),
                              soa_digest=digest(soa.positions, soa.descriptors, soa.normals,
                                                soa.min_distances, soa.max_distances,
                                                soa.point_ids))
        return local

    for k, fn in (("match_pinhole_phase1", w_phase1), ("matches_from_candidates", w_fc),
                  ("reject_outliers", w_rej), ("search_prev_frame", w_prev),
                  ("search_local_points", w_local), ("update_local_map", w_update)):
        setattr(T, k, fn)
    try:
        tr = StereoTracker(seq.cam, tracker=TrackerConfig(max_local_points=40000),
                           engine=ENGINE, warmup=False)
        statuses = []
        for i in range(len(seq)):
            cur["f"] = i
            res = tr.track_frame(FrameInput(timestamp=float(seq.timestamps[i]),
                                            features=seq.frames[i], imu=seq.imu_slice(i)))
            statuses.append(res.status)
    finally:
        for k, fn in orig.items():
            setattr(T, k, fn)
    # world table (ids 0..N-1, immutable after creation)
    n_pts = len(tr.world.points)
    assert sorted(tr.world.points) == list(range(n_pts))
    pts = [tr.world.points[i] for i in range(n_pts)]
    d = {"world_positions": np.array([p.position for p in pts]),
         "world_descriptors": np.array([p.descriptor for p in pts], dtype=np.uint64),
         "world_normals": np.array([p.normal for p in pts]),
         "world_min_d": np.array([p.min_distance for p in pts]),
         "world_max_d": np.array([p.max_distance for p in pts]),
         "landmark_desc": seq.landmark_desc.copy(), "landmark_angle": seq.landmark_angle.copy(),
         "n_frames": np.int64(len(seq)), "status": np.array(statuses)}
    # keyframe observation lists (KeyFrame.observed_point_ids, mapping.py:142-145),
    # immutable once the keyframe exists: kf k's ids at kf_obs[kf_off[k]:kf_off[k+1]]
    kfs = [tr.world.keyframes[k] for k in sorted(tr.world.keyframes)]
    assert [kf.kf_id for kf in kfs] == list(range(len(kfs)))
    obs = [np.asarray(kf.observed_point_ids(), dtype=np.int32) for kf in kfs]
    d["kf_off"] = np.concatenate([[0], np.cumsum([len(o) for o in obs])]).astype(np.int64)
    d["kf_obs"] = np.concatenate(obs).astype(np.int32) if obs else np.zeros(0, np.int32)
    d["kf_frame"] = np.array([kf.frame_id for kf in kfs], dtype=np.int32)
    lens = []
    for i, fr in enumerate(seq.frames):
        for side, f, ids in (("l", fr.left, fr.landmark_ids_left),
                             ("r", fr.right, fr.landmark_ids_right)):
            assert (f.descriptors == seq.landmark_desc[ids]).all()
            assert (f.angle == seq.landmark_angle[ids]).all()
            assert (f.response == 100.0).all()
            d[f"f{i}_{side}_ids"] = ids.astype(np.uint16)
            d[f"f{i}_{side}_uv"] = np.stack([f.u, f.v])
            d[f"f{i}_{side}_octave"] = f.octave.astype(np.int8)
        r = rec.get(i, {})
        for stage, fields in r.items():
            for k, v in fields.items():
                if stage == "update" and k == "slots_in":
                    continue  # == local_slots_in (same frame.slots, tracker.py:345-357)
                if stage == "local" and k == "local_ids":
                    m = np.zeros(n_pts, dtype=bool)
                    m[v] = True
                    d[f"f{i}_local_mask"] = np.packbits(m)
                    continue
                d[f"f{i}_{stage}_{k}"] = v
        lens.append(len(fr.left))
    np.savez_compressed(OUT / f"cfg4_{trajectory}.npz", **d)
    micros = {s: [rp.micros.get(s, 0) for rp in tr.reports[1:]] for s in
              ("stereo_match", "initial_pose", "update_local_map", "search_local_points",
               "total")}
    return {f"cfg4_{trajectory}": {
        "frames": len(seq), "status_counts": {s: statuses.count(s) for s in set(statuses)},
        "world_points": n_pts, "keyframes": len(kfs),
        "kps_per_frame_median": int(np.median(lens)),
        "local_map_median": int(np.median([len(r["local"]["local_ids"]) for r in rec.values()
                                           if "local" in r])),
        "stage_us_median_seq_engine": {k: float(np.median(v)) for k, v in micros.items()}}}


def main() -> None:
    kernels.warmup()
    summary = {}
    only = sys.argv[1:]
    if only:
        old = json.loads((OUT / "summary.json").read_text())
        summary.update(old)
        for name in only:
            summary.update(globals()[f"gen_{name}"]() if "_" not in name
                           else globals()[f"gen_{name.split('_')[0]}"](name.split("_", 1)[1]))
        (OUT / "summary.json").write_text(json.dumps(summary, indent=1))
        print(json.dumps({k: summary[k] for k in summary if any(k.startswith(o) for o in only)},
                         indent=1))
        return
    gen_hamming()
    summary.update(gen_edge())
    summary.update(gen_cfg2())
    summary.update(gen_cfg3())
    summary.update(gen_cfg1())
    summary.update(gen_cfg4("line"))
    summary.update(gen_cfg4("circle"))
    summary.update(gen_sweeps())
    summary.update(gen_scales())
    summary.update(gen_cfg5())
    summary.update(gen_prev())
    summary["generator"] = "tests/golden/make_golden.py (reference trackfront, seq engine)"
    (OUT / "summary.json").write_text(json.dumps(summary, indent=1))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
