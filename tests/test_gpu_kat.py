"""The reference SPEC's known-answer examples (listed in
SURVEY.md 8(c)) run through the B200 path; the stereo / fisheye ones also
through the CPU oracle, so those KATs pin both.  Small hand-built inputs.
The SAD-triple parabola, the 4.5-px interpolated shift
 and the exact ray intersection are in
test_spec_kat.py; search_prev_frame's static / empty cases
in test_golden_sweeps.py."""

import numpy as np
import pytest

import golden_io as G
import paper_2509_10757_b200 as ft
from paper_2509_10757_b200.types import (FeatureSet, Frame, FrameGrid, LocalMap, MapPointSoA,
                                         Pose, ProjectionSearchConfig, StereoMatchConfig)

pytestmark = pytest.mark.gpu
SCALE_POW = 1.2 ** np.arange(8.0)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def rand_desc(n, seed):
    return np.random.default_rng(seed).integers(0, 2 ** 63, size=(n, 4), dtype=np.int64).view(
        np.uint64)


def fs(u, v, desc, octave=None):
    n = len(u)
    return FeatureSet(u=np.asarray(u, np.float64), v=np.asarray(v, np.float64),
                      octave=np.zeros(n, np.int32) if octave is None else np.asarray(octave, np.int32),
                      angle=np.zeros(n), response=np.ones(n, np.float32), descriptors=desc)


def frame_of(left, cam, pose):
    grid = FrameGrid(left.u, left.v, cam.width, cam.height, 48)
    return Frame(0, 0.0, left, left, np.full(len(left.u), -1.0),
                 np.full(len(left.u), -1, dtype=np.int64), pose, grid)


def test_kat_phase1_singleton_and_band(oracle):
    """a same-row singleton with identical descriptors matches
    at distance 0; a right keypoint 3 band widths away matches nothing."""
    cfg = StereoMatchConfig()
    d = rand_desc(1, 1)
    left = fs([400.0], [200.0], d)
    for impl in (ft.match_pinhole_phase1, oracle.match_pinhole_phase1):
        idx, dist = impl(left, fs([390.0], [200.0], d), 480, SCALE_POW, cfg)
        assert idx.tolist() == [0] and dist.tolist() == [0]
        far = 200.0 + 3 * cfg.band_factor * SCALE_POW[0]
        idx, dist = impl(left, fs([390.0], [far], d), 480, SCALE_POW, cfg)
        assert idx.tolist() == [-1] and dist.tolist() == [10000]


def test_kat_phase2_integer_shift(oracle):
    """the right image is the left shifted by exactly 4 pixels
    -> disparity 4.0 with delta = 0 (a texture mirror-symmetric about the
    keypoint column makes the SADs at -1 / +1 equal, so the parabola's vertex
    is the integer minimum)."""
    from types import SimpleNamespace
    from paper_2509_10757_b200.pyramid import build_pyramid
    cam, cfg = G.pinhole(), StereoMatchConfig()
    h, w, xc, vy = 480, 752, 400, 240
    rng = np.random.default_rng(5)
    col = rng.integers(0, 256, size=(h, w // 2 + 8))
    xs = np.abs(np.arange(w) - xc)  # mirror symmetric about column xc
    left_img = col[:, np.minimum(xs, col.shape[1] - 1)].astype(np.uint8)
    right_img = np.zeros_like(left_img)
    right_img[:, :w - 4] = left_img[:, 4:]  # right(x) = left(x + 4)
    pcfg = SimpleNamespace(levels=8, scale=1.2, patch_size=31)
    pl, pr = build_pyramid(left_img, pcfg), build_pyramid(right_img, pcfg)
    d = rand_desc(1, 2)
    left, right = fs([float(xc)], [float(vy)], d), fs([float(xc - 4)], [float(vy)], d)
    idx = np.array([0], np.int64)
    dist = np.array([0], np.int64)
    for impl in (ft.refine_match_phase2, oracle.refine_match_phase2):
        m = impl(pl, pr, left, right, idx, dist, cam, cfg)
        assert m.right_idx.tolist() == [0]
        assert m.disparity.tolist() == [4.0] and m.refined_u.tolist() == [float(xc - 4)]
        assert m.sad.tolist() == [0]


@pytest.mark.parametrize("case", ["uniform", "one_outlier"])
def test_kat_reject_outliers(oracle, case):
    """equal scores keep every match; one score at 10x the
    median with m_out = 2 drops exactly that match."""
    cfg = StereoMatchConfig(outlier_multiplier=2.0)
    sad = np.full(9, 50, np.int64)
    if case == "one_outlier":
        sad[4] = 500
    for impl in (ft.reject_outliers, oracle.reject_outliers):
        m = ft.StereoMatches(right_idx=np.arange(9, dtype=np.int64),
                             distance=np.full(9, 5, np.int64), disparity=np.full(9, 3.0),
                             refined_u=np.full(9, 1.0), depth=np.full(9, 2.0), sad=sad.copy())
        impl(m, cfg)
        want = np.arange(9)
        if case == "one_outlier":
            want[4] = -1
        np.testing.assert_array_equal(m.right_idx, want)


def test_kat_fisheye_identity_and_ambiguity(oracle):
    """identical descriptor lists (distinct per index) match
    i <-> i; two right keypoints at the same best distance fail the ratio
    test."""
    from paper_2509_10757_b200.stereo import fisheye_bruteforce
    cfg = StereoMatchConfig()
    d = rand_desc(64, 3)
    f = fs(np.zeros(64), np.zeros(64), d)
    idx, dist = fisheye_bruteforce(f, f, cfg)
    np.testing.assert_array_equal(idx, np.arange(64))
    np.testing.assert_array_equal(dist, 0)
    oidx, odist = oracle.bruteforce(d, d, cfg.t_match, cfg.ratio)
    np.testing.assert_array_equal(oidx, idx)
    np.testing.assert_array_equal(odist, dist)
    # ambiguity: the left descriptor 5 bits away from two identical right ones
    # (at distance 0 the reference's `best <= ratio * second` holds: 0 <= 0)
    q = d[:1].copy()
    q[0, 0] ^= np.uint64(0b11111)
    dup = fs(np.zeros(2), np.zeros(2), np.repeat(d[:1], 2, axis=0))
    idx, dist = fisheye_bruteforce(fs([0.0], [0.0], q), dup, cfg)
    assert idx.tolist() == [-1] and dist.tolist() == [5]  # rejected, dist = best (kernels.py)
    oidx, odist = oracle.bruteforce(q, dup.descriptors, cfg.t_match, cfg.ratio)
    assert oidx.tolist() == [-1] and odist.tolist() == [5]


def _self_consistent_scene(n=200, seed=4):
    """Keypoints spread over the image, points back-projected from them at
    depth 4 m with identity pose, each carrying its keypoint's descriptor."""
    cam = G.pinhole()
    rng = np.random.default_rng(seed)
    u = rng.uniform(60, cam.width - 60, n)
    v = rng.uniform(60, cam.height - 60, n)
    z = 4.0
    pos = np.stack([(u - cam.cx) / cam.fx * z, (v - cam.cy) / cam.fy * z, np.full(n, z)], 1)
    desc = rand_desc(n, seed + 1)
    dist_c = np.linalg.norm(pos, axis=1)
    soa = MapPointSoA(positions=pos, descriptors=desc, normals=pos / dist_c[:, None],
                      min_distances=dist_c / 1.2 ** 7 / 1.01, max_distances=dist_c * 1.001,
                      point_ids=np.arange(1000, 1000 + n, dtype=np.int64))
    pose = Pose(np.eye(3), np.zeros(3))
    return cam, fs(u, v, desc), soa, pose


def test_kat_projection_self_consistency(oracle):
    """points back-projected from the frame's own keypoints (own
    depth, identity pose, own descriptor) match their keypoints at distance 0."""
    cam, left, soa, pose = _self_consistent_scene()
    cfg = ProjectionSearchConfig()
    c = ft.search_by_projection(soa, frame_of(left, cam, pose), pose, cam, cfg, 1.2, 8)
    np.testing.assert_array_equal(c.point_idx, np.arange(len(left.u)))
    np.testing.assert_array_equal(c.keypoint_idx, np.arange(len(left.u)))
    np.testing.assert_array_equal(c.distance, 0)


def test_kat_projection_conflict_lower_point_wins(oracle):
    """two points with identical descriptors claiming one
    keypoint -> exactly one correspondence, the lower point index."""
    cam, left, soa, pose = _self_consistent_scene(n=40)
    k = 7  # duplicate point 7 as the LAST point (same position and descriptor)
    dup = MapPointSoA(positions=np.vstack([soa.positions, soa.positions[k:k + 1]]),
                      descriptors=np.vstack([soa.descriptors, soa.descriptors[k:k + 1]]),
                      normals=np.vstack([soa.normals, soa.normals[k:k + 1]]),
                      min_distances=np.append(soa.min_distances, soa.min_distances[k]),
                      max_distances=np.append(soa.max_distances, soa.max_distances[k]),
                      point_ids=np.append(soa.point_ids, 99999))
    c = ft.search_by_projection(dup, frame_of(left, cam, pose), pose, cam,
                                ProjectionSearchConfig(), 1.2, 8)
    claim = c.point_idx[c.keypoint_idx == k]
    assert claim.tolist() == [k]
    assert len(dup.point_ids) - 1 not in c.point_idx.tolist()


def test_kat_search_local_points_exclusion_and_empty(oracle):
    """a LocalMap of points already slotted in the frame adds
    no association; an empty LocalMap adds none."""
    cam, left, soa, pose = _self_consistent_scene(n=60)
    cfg = ProjectionSearchConfig()
    local = LocalMap(keyframe_ids=(0,), point_ids=soa.point_ids.copy(), soa=soa)
    fr = frame_of(left, cam, pose)
    fr.slots[:] = soa.point_ids  # every point already slotted at its keypoint
    before = fr.slots.copy()
    ft.search_local_points(local, fr, cam, cfg, 1.2, 8)
    np.testing.assert_array_equal(fr.slots, before)
    empty = LocalMap(keyframe_ids=(), point_ids=np.empty(0, np.int64),
                     soa=MapPointSoA(np.empty((0, 3)), np.empty((0, 4), np.uint64),
                                     np.empty((0, 3)), np.empty(0), np.empty(0),
                                     np.empty(0, np.int64)))
    fr2 = frame_of(left, cam, pose)
    assert ft.search_local_points(empty, fr2, cam, cfg, 1.2, 8) == 0
    assert (fr2.slots == -1).all()
