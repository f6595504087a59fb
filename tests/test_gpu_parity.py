"""GPU parity: the B200 drop-in (through the C ABI) against the reference's
golden outputs and the CPU oracle on the same inputs.  Bit-exact for indices,
distances, SADs and slots; disparity / refined_u / depth are compared exactly
too (they are computed in fp64 with the reference's evaluation order), with
the north-star tolerance (1e-4 px) asserted as the contract."""

import numpy as np
import pytest

import golden_io as G
import paper_2509_10757_b200 as ft
from paper_2509_10757_b200.types import Frame, FrameGrid, ProjectionSearchConfig, StereoMatchConfig

pytestmark = pytest.mark.gpu

FIELDS = ("right_idx", "distance", "disparity", "refined_u", "depth", "sad")
CORR = ("point_idx", "keypoint_idx", "distance", "octave")
PX_TOL = 1e-4  # north star: stereo depth / uR within 1e-4 px


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def assert_matches(m, d, prefix):
    for f in ("right_idx", "distance", "sad"):
        np.testing.assert_array_equal(getattr(m, f), d[f"{prefix}_{f}"], err_msg=f)
    for f in ("disparity", "refined_u", "depth"):
        np.testing.assert_allclose(getattr(m, f), d[f"{prefix}_{f}"], rtol=0, atol=PX_TOL,
                                   err_msg=f)
        np.testing.assert_array_equal(getattr(m, f), d[f"{prefix}_{f}"], err_msg=f + " (bitwise)")


def assert_corr(c, d, prefix):
    for f in CORR:
        np.testing.assert_array_equal(getattr(c, f), d[f"{prefix}_{f}"], err_msg=f)


def make_frame(left, right, cam, pose):
    grid = FrameGrid(left.u, left.v, cam.width, cam.height, 48)
    return Frame(0, 0.0, left, right, np.full(len(left.u), -1.0),
                 np.full(len(left.u), -1, dtype=np.int64), pose, grid)


def test_hamming_pairs_capi():
    import torch
    from paper_2509_10757_b200 import _lib
    d = G.load("hamming.npz")
    L = _lib.load()
    a = torch.from_numpy(d["a"].view(np.int64)).cuda()
    b = torch.from_numpy(d["b"].view(np.int64)).cuda()
    out = torch.empty(len(d["a"]), dtype=torch.int64, device="cuda")
    _lib.check(L.ft_hamming_pairs(a.data_ptr(), b.data_ptr(), len(d["a"]), out.data_ptr(),
                                  torch.cuda.current_stream().cuda_stream), "hamming")
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy(), d["out"])


def test_cfg1_phase1_phase2_reject():
    d = G.load("cfg1_stereo.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cam, cfg = G.pinhole(), StereoMatchConfig()
    idx, dist = ft.match_pinhole_phase1(left, right, cam.height, d["scale_pow"], cfg)
    np.testing.assert_array_equal(idx, d["p1_idx"])
    np.testing.assert_array_equal(dist, d["p1_dist"])
    pl, pr = G.pyramid(d, "l"), G.pyramid(d, "r")
    m = ft.refine_match_phase2(pl, pr, left, right, idx, dist, cam, cfg)
    assert_matches(m, d, "p2")
    ft.reject_outliers(m, cfg)
    assert_matches(m, d, "final")
    # fused single launch (tracker _run_stereo pinhole branch)
    f = ft.compute_stereo_matches(left, right, cam, cfg, d["scale_pow"], pl, pr)
    assert_matches(f, d, "final")


def test_cfg2_stereo_from_candidates():
    d = G.load("cfg2_frame_map.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cam, cfg = G.pinhole(), StereoMatchConfig()
    idx, dist = ft.match_pinhole_phase1(left, right, cam.height, d["scale_pow"], cfg)
    np.testing.assert_array_equal(idx, d["p1_idx"])
    m = ft.matches_from_candidates(idx, dist, left, right, cam, cfg)
    assert_matches(m, d, "fc")
    f = ft.compute_stereo_matches(left, right, cam, cfg, d["scale_pow"])
    assert_matches(f, d, "final")


def test_cfg2_projection_all_variants():
    d = G.load("cfg2_frame_map.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cam, cfg = G.pinhole(), ProjectionSearchConfig()
    pts, pose = G.soa(d), G.pose(d)
    frame = make_frame(left, right, cam, pose)
    kp, kd, ko = ft.run_phase_a(pts, frame, pose, cam, cfg, 1.2, 8)
    np.testing.assert_array_equal(kp, d["pa_kp"])
    np.testing.assert_array_equal(kd, d["pa_dist"])
    np.testing.assert_array_equal(ko, d["pa_oct"])
    assert_corr(ft.resolve_conflicts(kp, kd, ko), d, "corr")
    assert_corr(ft.search_by_projection(pts, frame, pose, cam, cfg, 1.2, 8), d, "corr")
    c = ft.search_by_projection(pts, frame, pose, cam, cfg, 1.2, 8, ref_angles=d["ref_angles"],
                                rotation_check=True, window_px=cfg.window_prev_px, u_offset=1.0)
    assert_corr(c, d, "corr_rot")
    c = ft.search_by_projection(pts, frame, pose, cam, cfg, 1.2, 8, skip_mask=d["skip"])
    assert_corr(c, d, "corr_skip")
    # standalone phase C on the golden phase-B output
    base = ft.search_by_projection(pts, frame, pose, cam, cfg, 1.2, 8,
                                   window_px=cfg.window_prev_px, u_offset=1.0)
    c2 = ft.rotation_consistency_filter(base, d["ref_angles"], left.angle, cfg)
    assert_corr(c2, d, "corr_rot")


def test_cfg2_search_local_points():
    d = G.load("cfg2_frame_map.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cam, cfg = G.pinhole(), ProjectionSearchConfig()
    local, pose = G.local_map(d), G.pose(d)
    fa = make_frame(left, right, cam, pose)
    n = ft.search_local_points(local, fa, cam, cfg, 1.2, 8)
    assert n == int(d["count_a"])
    np.testing.assert_array_equal(fa.slots, d["slots_a"])
    fb = make_frame(left, right, cam, pose)
    fb.slots[...] = d["slots_b_in"]
    n = ft.search_local_points(local, fb, cam, cfg, 1.2, 8)
    assert n == int(d["count_b"])
    np.testing.assert_array_equal(fb.slots, d["slots_b"])


def test_cfg3_fisheye():
    d = G.load("cfg3_fisheye.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cfg = StereoMatchConfig()
    from paper_2509_10757_b200.stereo import fisheye_bruteforce
    idx, dist = fisheye_bruteforce(left, right, cfg)
    np.testing.assert_array_equal(idx, d["bf_idx"])
    np.testing.assert_array_equal(dist, d["bf_dist"])
    cam = G.fisheye()
    lidx, ridx, pts3, dists = ft.match_fisheye(left, right, cam, cfg)
    np.testing.assert_array_equal(lidx, d["mf_lidx"])
    np.testing.assert_array_equal(ridx, d["mf_ridx"])
    # device unproject / closest points (CUDA sin, cos, hypot, sqrt) vs the
    # reference's numpy + glibc: accepted sets exact, points within 1e-12 rel
    np.testing.assert_allclose(pts3, d["mf_pts"], rtol=1e-12, atol=1e-15)
    np.testing.assert_array_equal(dists, d["mf_dists"])
    pcfg = ProjectionSearchConfig()
    pts, pose = G.soa(d), G.pose(d)
    frame = make_frame(left, right, cam, pose)
    kp, kd, ko = ft.run_phase_a(pts, frame, pose, cam, pcfg, 1.2, 8)
    np.testing.assert_array_equal(kp, d["pa_kp"])
    np.testing.assert_array_equal(kd, d["pa_dist"])
    np.testing.assert_array_equal(ko, d["pa_oct"])
    fa = make_frame(left, right, cam, pose)
    n = ft.search_local_points(G.local_map(d), fa, cam, pcfg, 1.2, 8)
    assert n == int(d["count_a"])
    np.testing.assert_array_equal(fa.slots, d["slots_a"])


def test_edge_cases():
    d = G.load("edge_cases.npz")
    from types import SimpleNamespace as NS
    from paper_2509_10757_b200.stereo import fisheye_bruteforce
    cfg = StereoMatchConfig()

    def F(desc, u=None, v=None, o=None):
        n = len(desc)
        return NS(u=np.zeros(n) if u is None else u, v=np.zeros(n) if v is None else v,
                  octave=np.zeros(n, np.int32) if o is None else o, descriptors=desc)

    idx, dist = fisheye_bruteforce(F(d["dup_left"]), F(d["dup_right"]), cfg)
    np.testing.assert_array_equal(idx, d["dup_idx"])
    np.testing.assert_array_equal(dist, d["dup_dist"])
    idx, dist = fisheye_bruteforce(F(d["dup_left"]), F(d["one_right"]), cfg)
    np.testing.assert_array_equal(idx, d["one_idx"])
    np.testing.assert_array_equal(dist, d["one_dist"])
    lf = F(d["tie_ld"], d["tie_lu"], d["tie_lv"], d["tie_loct"])
    rf = F(d["tie_rd"], d["tie_ru"], d["tie_rv"], d["tie_roct"])
    idx, dist = ft.match_pinhole_phase1(lf, rf, 480, 1.2 ** np.arange(8.0), cfg)
    np.testing.assert_array_equal(idx, d["tie_idx"])
    np.testing.assert_array_equal(dist, d["tie_dist"])
    for cnt in (1, 2, 7, 8, 101, 1000):
        m = ft.StereoMatches(right_idx=d[f"med{cnt}_rin"].copy(),
                             distance=np.full(cnt, 5, np.int64), disparity=np.full(cnt, 3.0),
                             refined_u=np.full(cnt, 1.0), depth=np.full(cnt, 2.0),
                             sad=d[f"med{cnt}_sad"].copy())
        ft.reject_outliers(m, cfg)
        np.testing.assert_array_equal(m.right_idx, d[f"med{cnt}_rout"])
        np.testing.assert_array_equal(m.sad, d[f"med{cnt}_sadout"])


def test_empty_inputs():
    e = ft.FeatureSet.empty()
    cfg = StereoMatchConfig()
    idx, dist = ft.match_pinhole_phase1(e, e, 480, np.ones(8), cfg)
    assert len(idx) == 0
    assert ft.match_fisheye(e, e, G.fisheye(), cfg)[0].shape == (0,)
    assert len(ft.resolve_conflicts(np.empty(0, np.int64), np.empty(0, np.int64),
                                    np.empty(0, np.int64))) == 0
    # left keypoints but no right keypoints
    d = G.load("cfg2_frame_map.npz")
    left = G.feats(d, "left")
    idx, dist = ft.match_pinhole_phase1(left, e, 480, d["scale_pow"], cfg)
    assert (idx == -1).all() and (dist == 10000).all()


def _oracle_local_search(O, w, pcfg, slots):
    grid = O.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
    return O.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                 w.left.octave, w.left.descriptors, grid, slots, w.pose, w.cam,
                                 pcfg, 1.2, 8)


@pytest.mark.parametrize("seed,n_lm,m_pts,images", [(11, 12000, 5000, True),
                                                    (12, 20000, 20000, False),
                                                    (13, 20000, 20000, True),
                                                    (14, 4000, 1000, True)])
def test_random_pinhole_vs_oracle(oracle, seed, n_lm, m_pts, images):
    from synthetic import make_workload
    w = make_workload(seed=seed, n_landmarks=n_lm, map_points=m_pts, images=images)
    cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
    ref = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam, cfg,
                                w.scale_pow)
    got = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left,
                                    w.pyr_right)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f)
    slots = np.full(len(w.left.u), -1, np.int64)
    # pre-slot a few keypoints with map ids to exercise skip + "only if empty"
    rng = np.random.default_rng(seed)
    k = rng.choice(len(slots), size=len(slots) // 10, replace=False)
    slots[k] = rng.choice(w.local.point_ids, size=len(k), replace=False)
    frame = w.frame()
    frame.slots[...] = slots
    n_ref = _oracle_local_search(oracle, w, pcfg, slots)
    n = ft.search_local_points(w.local, frame, w.cam, pcfg, 1.2, 8)
    assert n == n_ref
    np.testing.assert_array_equal(frame.slots, slots)


@pytest.mark.parametrize("seed", [21, 22])
def test_random_fisheye_vs_oracle(oracle, seed):
    from synthetic import make_workload
    from paper_2509_10757_b200.stereo import fisheye_bruteforce
    w = make_workload(seed=seed, n_landmarks=5000, map_points=5000, fisheye=True, noise_px=0.3)
    cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
    idx, dist = fisheye_bruteforce(w.left, w.right, cfg)
    ridx, rdist = oracle.bruteforce(w.left.descriptors, w.right.descriptors, cfg.t_match,
                                    cfg.ratio, 4)
    np.testing.assert_array_equal(idx, ridx)
    np.testing.assert_array_equal(dist, rdist)
    frame = w.frame()
    kp, kd, ko = ft.run_phase_a(w.local.soa, frame, w.pose, w.cam, pcfg, 1.2, 8)
    grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
    rkp, rkd, rko = oracle.run_phase_a(w.local.soa, w.left.u, w.left.v, w.left.octave,
                                       w.left.descriptors, grid, w.pose, w.cam, pcfg, 1.2, 8)
    np.testing.assert_array_equal(kp, rkp)
    np.testing.assert_array_equal(kd, rkd)
    np.testing.assert_array_equal(ko, rko)


def test_projection_fp64_audit_many_points(oracle):
    """Transcendental audit (SURVEY §7 hard part 1): 1e6 random fisheye and
    pinhole map points near frustum edges, device vs oracle phase A."""
    from synthetic import make_workload
    for fish in (False, True):
        w = make_workload(seed=31, n_landmarks=6000, map_points=2000, fisheye=fish)
        rng = np.random.default_rng(5)
        m = 200_000
        pts = ft.MapPointSoA(
            positions=rng.uniform(-6, 6, size=(m, 3)) + np.array([4.0, 0, 0]),
            descriptors=w.local.soa.descriptors[rng.integers(0, 2000, m)],
            normals=np.tile(np.array([[1.0, 0, 0]]), (m, 1)),
            min_distances=np.full(m, 0.1), max_distances=rng.uniform(2, 12, m),
            point_ids=np.arange(m, dtype=np.int64))
        pcfg = ProjectionSearchConfig(view_cos_min=-1.0)
        frame = w.frame()
        kp, kd, ko = ft.run_phase_a(pts, frame, w.pose, w.cam, pcfg, 1.2, 8)
        grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
        rkp, rkd, rko = oracle.run_phase_a(pts, w.left.u, w.left.v, w.left.octave,
                                           w.left.descriptors, grid, w.pose, w.cam, pcfg, 1.2, 8,
                                           nthreads=8)
        np.testing.assert_array_equal(kp, rkp)
        np.testing.assert_array_equal(ko, rko)
        np.testing.assert_array_equal(kd, rkd)


def test_pack_kernels_match_host_packing():
    """ft_pack_keypoints / ft_pack_points (device SoA -> records) equal the
    host-side packing the runtime does."""
    import torch
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.runtime import fill_kp_records, fill_point_records
    d = G.load("cfg2_frame_map.npz")
    left, pts = G.feats(d, "left"), G.soa(d)
    n, m = len(left.u), len(pts.point_ids)
    L = _lib.load()
    cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    s = torch.cuda.current_stream().cuda_stream
    cnt = cu(np.array([n], np.int32))
    u, v, o, ang = cu(left.u), cu(left.v), cu(left.octave.astype(np.int32)), cu(left.angle)
    desc = cu(left.descriptors.view(np.int64))
    out = torch.zeros(n * 64, dtype=torch.uint8, device="cuda")
    _lib.check(L.ft_pack_keypoints(1, u.data_ptr(), v.data_ptr(), o.data_ptr(), ang.data_ptr(),
                                   desc.data_ptr(), cnt.data_ptr(), n, out.data_ptr(), s), "pack")
    ref = np.zeros(n, _lib.KP_RECORD)
    fill_kp_records(ref, left, with_angle=True)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(out.cpu().numpy().view(_lib.KP_RECORD), ref)
    cntp = cu(np.array([m], np.int32))
    args = [cu(pts.positions), cu(pts.normals), cu(pts.min_distances), cu(pts.max_distances),
            cu(pts.descriptors.view(np.int64)), cu(pts.point_ids)]
    outp = torch.zeros(m * 112, dtype=torch.uint8, device="cuda")
    _lib.check(L.ft_pack_points(1, *[t.data_ptr() for t in args], cntp.data_ptr(), m,
                                outp.data_ptr(), s), "pack points")
    refp = np.zeros(m, _lib.POINT_RECORD)
    fill_point_records(refp, pts)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(outp.cpu().numpy().view(_lib.POINT_RECORD), refp)


def test_device_pyramid_matches_reference_pyramids():
    """ft_build_pyramids rebuilds the reference's cfg1 pyramids (levels 1..7)
    bit-exactly from level 0 (the raw image)."""
    from types import SimpleNamespace
    from paper_2509_10757_b200.pyramid import build_pyramid
    d = G.load("cfg1_stereo.npz")
    for side in ("l", "r"):
        ref = G.pyramid(d, side)
        h, w = int(ref.heights[0]), int(ref.widths[0])
        img = ref.data[:h * w].reshape(h, w)
        got = build_pyramid(img, SimpleNamespace(levels=8, scale=1.2, patch_size=31))
        np.testing.assert_array_equal(got.offsets, ref.offsets)
        for lvl in range(8):
            np.testing.assert_array_equal(got.level(lvl), ref.level(lvl), err_msg=f"{side} level {lvl}")


@pytest.mark.parametrize("shape,levels,n_images", [((480, 752), 8, 1), ((480, 752), 8, 7),
                                                   ((512, 512), 8, 3), ((217, 333), 5, 2),
                                                   ((480, 752), 8, 300)])
def test_device_pyramid_batched_vs_oracle(oracle, shape, levels, n_images):
    """ft_build_pyramids over n_images raw images in one call (chunked
    cooperative waves past one resident wave) vs the C oracle, bit-exact."""
    import torch
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.runtime import make_workspace, pyramid_struct
    from types import SimpleNamespace
    rng = np.random.default_rng(shape[0] * 7 + n_images)
    h, w = shape
    n_ref = min(n_images, 4)
    imgs = rng.integers(0, 256, size=(n_images, h, w), dtype=np.uint8)
    # smooth-ish content too (flat areas and gradients hit the .5 rounding cases)
    yy, xx = np.mgrid[0:h, 0:w]
    imgs[0] = ((xx * 3 + yy * 5) // 7 % 256).astype(np.uint8)
    refs = [oracle.build_pyramid(imgs[i], levels, 1.2) for i in range(n_ref)]
    _, offsets, ws, hs = refs[0]
    total = int(offsets[-1])
    lib = _lib.load()
    stream = torch.cuda.Stream()
    pyr = torch.zeros(n_images * total, dtype=torch.uint8, device="cuda")
    src = torch.from_numpy(imgs.reshape(-1)).cuda()
    ws_ = make_workspace(lib, torch.device("cuda"), stream, (n_images + 1) // 2, 1, 1)
    geo = SimpleNamespace(offsets=offsets, widths=ws, heights=hs)
    st = lib.ft_build_pyramids(n_images, pyramid_struct(geo, pyr.data_ptr(), total),
                               src.data_ptr(), h * w, ws_, stream.cuda_stream)
    _lib.check(st, "ft_build_pyramids")
    stream.synchronize()
    got = pyr.cpu().numpy().reshape(n_images, total)
    for i in range(n_ref):
        np.testing.assert_array_equal(got[i], refs[i][0], err_msg=f"image {i}")
    for i in range(n_ref, n_images, 37):  # spot-check the later chunks
        np.testing.assert_array_equal(got[i], oracle.build_pyramid(imgs[i], levels, 1.2)[0],
                                      err_msg=f"image {i}")


@pytest.mark.parametrize("corrected", [False, True])
def test_fisheye_triangulation_vs_oracle(oracle, corrected):
    """ft_stereo_fisheye (brute force + unproject + closest points + checks in
    one launch) vs the oracle's restatement of stereo.py:245-273, in the
    reference's mode (its t sign, stereo.py:216) and the corrected
    least-squares mode (1397 triangulated pairs on cfg3)."""
    d = G.load("cfg3_fisheye.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cfg, cam = StereoMatchConfig(), G.fisheye()
    got = ft.match_fisheye(left, right, cam, cfg, corrected=corrected)
    ref = oracle.fisheye_triangulate(left, right, d["bf_idx"], d["bf_dist"], cam,
                                     cfg.ray_gap_ceiling, corrected)
    for a, b, name in zip(got, ref, ("left_ids", "right_ids", "points", "dists")):
        if name == "points":
            np.testing.assert_allclose(a, b, rtol=1e-9, atol=1e-12, err_msg=name)
        else:
            np.testing.assert_array_equal(a, b, err_msg=name)
    if corrected:
        assert len(got[0]) > 1000
        m = ft.compute_stereo_fisheye_matches(left, right, cam, cfg, corrected=True)
        np.testing.assert_allclose(m.depth[got[0]], got[2][:, 2], rtol=0, atol=0)


def _world_from_soa(soa):
    """Minimal host world map (reference mapping.py MapPoint fields used by
    decompose_map_points) keyed by point id."""
    from types import SimpleNamespace
    pts = {}
    for i, pid in enumerate(soa.point_ids):
        pts[int(pid)] = SimpleNamespace(point_id=int(pid), position=soa.positions[i],
                                        descriptor=soa.descriptors[i], normal=soa.normals[i],
                                        min_distance=float(soa.min_distances[i]),
                                        max_distance=float(soa.max_distances[i]))
    return SimpleNamespace(points=pts)


@pytest.mark.parametrize("use_table", [False, True])
def test_search_prev_frame(oracle, use_table):
    """projection.py:224-253 on cfg2: the previous frame's slotted points
    (from SearchLocalPoints) searched in the current frame with the rotation
    check, the 15-px window and the +-1 px offset from the relative forward
    translation; host-decomposed SoA, or resident MapTable slots."""
    import math
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.types import Pose
    d = G.load("cfg2_frame_map.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    cam, cfg = G.pinhole(), ProjectionSearchConfig()
    local, pose = G.local_map(d), G.pose(d)
    prev = make_frame(left, right, cam, pose)
    prev.slots[...] = d["slots_a"]
    world = _world_from_soa(local.soa)
    cur_pose = Pose(pose.rotation, pose.translation + np.array([0.002, -0.001, 0.004]))
    cur = make_frame(left, right, cam, cur_pose)
    table = MapTable(capacity=8192) if use_table else None
    corr, pids = ft.search_prev_frame(prev, cur, cur_pose, world, cam, cfg, 1.2, 8, table=table)
    # oracle composition (reference projection.py:231-253)
    slot_idx = np.nonzero(prev.slots != -1)[0]
    ids = prev.slots[slot_idx]
    order = {int(p): i for i, p in enumerate(local.soa.point_ids)}
    rows = np.array([order[int(p)] for p in ids])
    sub = type(local.soa)(positions=local.soa.positions[rows],
                          descriptors=local.soa.descriptors[rows], normals=local.soa.normals[rows],
                          min_distances=local.soa.min_distances[rows],
                          max_distances=local.soa.max_distances[rows], point_ids=ids)
    rel = cur_pose.matrix() @ np.linalg.inv(prev.pose.matrix())
    fwd = float(rel[2, 3])
    u_off = math.copysign(cfg.prev_u_offset_px, fwd) if abs(fwd) > 1e-9 else 0.0
    grid = oracle.frame_grid(left.u, left.v, cam.width, cam.height, 48) + (48,)
    ref = oracle.search_by_projection(sub, left.u, left.v, left.octave, left.descriptors,
                                      left.angle, grid, cur_pose, cam, cfg, 1.2, 8,
                                      ref_angles=left.angle[slot_idx],
                                      rotation_check=cfg.rotation_check_prev,
                                      window_px=cfg.window_prev_px, u_offset=u_off)
    np.testing.assert_array_equal(pids, ids)
    assert len(ref.point_idx) > 100
    for f in ("point_idx", "keypoint_idx", "distance", "octave"):
        np.testing.assert_array_equal(getattr(corr, f), getattr(ref, f), err_msg=f)
    if use_table:  # a second call finds every point resident: no upload
        before = table.bytes_uploaded
        ft.search_prev_frame(prev, cur, cur_pose, world, cam, cfg, 1.2, 8, table=table)
        assert table.bytes_uploaded == before


STEREO_CFGS = [
    dict(t_match=40),
    dict(band_factor=1.0, half_window=3, half_slide=3),
    dict(band_factor=3.5, half_window=7, half_slide=8, outlier_multiplier=1.5),
    dict(min_disparity=2.0, max_disparity=60.0, outlier_multiplier=4.0),
    dict(t_match=256, half_window=1, half_slide=1, ratio=0.6),
]


@pytest.mark.parametrize("kw", STEREO_CFGS)
def test_stereo_config_sweep_vs_oracle(oracle, kw):
    """Non-default StereoMatchConfig values (thresholds, band, window /
    slide sizes incl. the 1x1 and 15x15 extremes, disparity range,
    outlier multiplier) through phase 1 -> phase 2 -> reject and the fisheye
    ratio test, bit-exact with the oracle."""
    from synthetic import make_workload
    w = make_workload(seed=31, n_landmarks=12000, map_points=2000, images=True)
    cfg = StereoMatchConfig(**kw)
    ref = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam, cfg,
                                w.scale_pow)
    got = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left,
                                    w.pyr_right)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f"{kw} {f}")
    from paper_2509_10757_b200.stereo import fisheye_bruteforce
    idx, dist = fisheye_bruteforce(w.left, w.right, cfg)
    ridx, rdist = oracle.bruteforce(w.left.descriptors, w.right.descriptors, cfg.t_match,
                                    cfg.ratio, 4)
    np.testing.assert_array_equal(idx, ridx)
    np.testing.assert_array_equal(dist, rdist)


PROJ_CFGS = [
    dict(window_px=2.0, t_proj=50),
    dict(window_px=12.0, ratio=0.7, view_cos_min=0.9),
    dict(window_px=30.0, ratio=1.0, view_cos_min=-1.0, t_proj=256),
    dict(histogram_bins=12, histogram_keep=1),
]


@pytest.mark.parametrize("kw", PROJ_CFGS)
@pytest.mark.parametrize("scale,levels", [(1.2, 8), (1.3, 6), (2.0, 4)])
def test_projection_config_sweep_vs_oracle(oracle, kw, scale, levels):
    """Non-default ProjectionSearchConfig values and pyramid scale / level
    counts (level prediction uses 1 / log(scale)) through phase A, resolve,
    rotation filter and SearchLocalPoints, bit-exact with the oracle."""
    from synthetic import make_workload
    w = make_workload(seed=41, n_landmarks=12000, map_points=5000)
    pcfg = ProjectionSearchConfig(**kw)
    frame = w.frame()
    grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
    kp, kd, ko = ft.run_phase_a(w.local.soa, frame, w.pose, w.cam, pcfg, scale, levels)
    rkp, rkd, rko = oracle.run_phase_a(w.local.soa, w.left.u, w.left.v, w.left.octave,
                                       w.left.descriptors, grid, w.pose, w.cam, pcfg, scale,
                                       levels)
    np.testing.assert_array_equal(kp, rkp)
    np.testing.assert_array_equal(kd, rkd)
    np.testing.assert_array_equal(ko, rko)
    rng = np.random.default_rng(7)
    ref_ang = rng.uniform(0, 2 * np.pi, len(w.local.point_ids))
    c = ft.search_by_projection(w.local.soa, frame, w.pose, w.cam, pcfg, scale, levels,
                                ref_angles=ref_ang, rotation_check=True, u_offset=-1.0)
    rc = oracle.search_by_projection(w.local.soa, w.left.u, w.left.v, w.left.octave,
                                     w.left.descriptors, w.left.angle, grid, w.pose, w.cam, pcfg,
                                     scale, levels, ref_angles=ref_ang, rotation_check=True,
                                     u_offset=-1.0)
    for f in ("point_idx", "keypoint_idx", "distance", "octave"):
        np.testing.assert_array_equal(getattr(c, f), getattr(rc, f), err_msg=f)
    slots = np.full(len(w.left.u), -1, np.int64)
    n_ref = oracle.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                       w.left.octave, w.left.descriptors, grid, slots, w.pose,
                                       w.cam, pcfg, scale, levels)
    f2 = w.frame()
    n = ft.search_local_points(w.local, f2, w.cam, pcfg, scale, levels)
    assert n == n_ref
    np.testing.assert_array_equal(f2.slots, slots)


def test_rejection_median_large_sads(oracle):
    """Median rejection when accepted SADs exceed the histograms' fine range
    (>= 4096): a right pyramid of uncorrelated noise makes every SAD large,
    so the gather + radix-select path runs; bit-exact with the oracle."""
    from copy import deepcopy
    from synthetic import make_workload
    w = make_workload(seed=51, n_landmarks=12000, map_points=1000, images=True)
    pr = deepcopy(w.pyr_right)
    rng = np.random.default_rng(3)
    pr.data = rng.integers(0, 256, size=pr.data.shape, dtype=np.uint8)
    cfg = StereoMatchConfig()
    ref = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, pr, w.cam, cfg, w.scale_pow)
    idx, dist = oracle.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)
    pre = oracle.refine_match_phase2(w.pyr_left, pr, w.left, w.right, idx, dist, w.cam, cfg)
    assert pre.sad[pre.right_idx >= 0].max() >= 4096
    # the median itself lies above the group histogram's fine range: the
    # gather + radix-select path decides (ft_track.cu stereo_frame)
    assert np.median(pre.sad[pre.right_idx >= 0]) >= 4096
    got = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left, pr)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f)


@pytest.mark.parametrize("tail", [False, True])
@pytest.mark.parametrize("amp", [60, 70, 75])
def test_rejection_median_near_histogram_edge(oracle, amp, tail, monkeypatch):
    """Medians around the group histograms' fine range (4096): right-image
    noise of +-amp puts the median SAD at ~3.6k / ~4.0k (hundreds of SADs in
    the overflow bin, median still resolved by the histograms) / above 4096
    (gather fallback); every case bit-exact with the oracle, with the group
    barrier path and with the dedicated tail block (persistent plans' mode)."""
    from copy import deepcopy
    if tail:
        monkeypatch.setenv("FT_TAIL_LAUNCH", "1")
    from synthetic import make_workload
    w = make_workload(seed=51, n_landmarks=12000, map_points=1000, images=True)
    pr = deepcopy(w.pyr_right)
    rng = np.random.default_rng(3)
    noise = rng.integers(-amp, amp + 1, size=pr.data.shape)
    pr.data = np.clip(pr.data.astype(np.int32) + noise, 0, 255).astype(np.uint8)
    cfg = StereoMatchConfig()
    ref = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, pr, w.cam, cfg, w.scale_pow)
    got = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left, pr)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f)


@pytest.mark.parametrize("seed", [31, 32])
def test_pipelined_patch_edges_vs_oracle(oracle, seed):
    """The block-batched SAD pass stages patch rows as 16-B chunks, falling back
    to byte loads where a chunk would reach outside its level (first / last
    rows and columns of a level, the end of the last level).  Keypoints placed
    on every level right at the patch borders, through the fused call (the
    block-batched passes; the session's pyramid base is not 16-B aligned), must
    equal the oracle."""
    from synthetic import make_workload
    from paper_2509_10757_b200.types import FeatureSet
    w = make_workload(seed=seed, n_landmarks=2000, map_points=500, images=True)
    pyr, scale_pow = w.pyr_left, w.scale_pow
    rng = np.random.default_rng(seed)
    lu, lv, lo, ru, rv, ro, desc_l, desc_r = [], [], [], [], [], [], [], []
    for o in range(len(pyr.widths)):
        wd, ht, s = int(pyr.widths[o]), int(pyr.heights[o]), float(scale_pow[o])
        for x in (5, 6, 7, 15, 16, 17, wd - 18, wd - 17, wd - 8, wd - 7, wd - 6):
            for y in (5, 6, ht // 2, ht - 7, ht - 6):
                d = rng.integers(0, 2**63, 4, dtype=np.uint64)
                disp = 2.0 + rng.integers(0, 6)  # level-o pixels
                lu.append(x * s + rng.uniform(-0.3, 0.3) * s)
                lv.append(y * s)
                lo.append(o)
                ru.append((x - disp) * s)
                rv.append(y * s)
                ro.append(o)
                desc_l.append(d)
                d2 = d.copy()
                d2[0] ^= np.uint64(1 << int(rng.integers(0, 8)))  # a few bits apart
                desc_r.append(d2)

    def fs(u, v, o, d):
        n = len(u)
        return FeatureSet(np.array(u), np.array(v), np.array(o, np.int32), np.zeros(n),
                          np.zeros(n, np.float32), np.array(d, np.uint64).reshape(n, 4))
    left, right = fs(lu, lv, lo, desc_l), fs(ru, rv, ro, desc_r)
    cfg = StereoMatchConfig()
    ref = oracle.stereo_pinhole(left, right, w.pyr_left, w.pyr_right, w.cam, cfg, scale_pow)
    got = ft.compute_stereo_matches(left, right, w.cam, cfg, scale_pow, w.pyr_left, w.pyr_right)
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(got, f), getattr(ref, f), err_msg=f)
    assert (ref.right_idx >= 0).sum() > 20  # the edge patches were refined, not all rejected
