"""Reference goldens beyond the default configs (tests/golden/make_golden.py:
gen_sweeps, gen_scales, gen_cfg5, gen_prev), each checked through the CPU
oracle (every round, no GPU) and through the B200 drop-in (``-m gpu``):

* sweeps.npz   5 non-default StereoMatchConfig values on the cfg1 rendered
               ORB frame (phase 1 -> 2 -> reject), the cfg2 bundle (phase 1 ->
               from candidates -> reject) and the cfg3 fisheye descriptors
               (brute force); 4 non-default ProjectionSearchConfig values x
               pyramid scale 1.2 / 1.3 / 2.0 (8 / 6 / 4 levels) on cfg2 (phase
               A, rotation-checked search_by_projection, search_local_points)
* scales.npz   cfg1's images through ORB extraction at scale 1.3 / 2.0
               (reference pyramids), phase 1 -> 2 -> reject
* cfg5_high_load.npz  2073 keypoints + a 20000-point local map
* prev_frame.npz      the reference's own search_prev_frame (forward /
               backward / static motion) and its SPEC.md:352-353 cases
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import golden_io as G
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig

FIELDS = ("right_idx", "distance", "disparity", "refined_u", "depth", "sad")
CORR = ("point_idx", "keypoint_idx", "distance", "octave")
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


def _eq(a, b, what):
    np.testing.assert_array_equal(np.asarray(a), np.asarray(b), err_msg=what)


def assert_matches(m, d, prefix):
    for f in FIELDS:
        _eq(getattr(m, f), d[f"{prefix}_{f}"], f"{prefix} {f}")


def assert_corr(c, d, prefix):
    for f in CORR:
        _eq(getattr(c, f), d[f"{prefix}_{f}"], f"{prefix} {f}")


def _grid(O, left, cam):
    return O.frame_grid(left.u, left.v, cam.width, cam.height, 48) + (48,)


class OracleImpl:
    """The stage compositions through the C oracle (oracle/oracle.py)."""

    def __init__(self, O):
        self.O = O

    def stereo_refine(self, left, right, pl, pr, cam, cfg, sp):
        return self.O.stereo_pinhole(left, right, pl, pr, cam, cfg, sp)

    def stereo_fc(self, left, right, cam, cfg, sp):
        return self.O.stereo_pinhole(left, right, None, None, cam, cfg, sp)

    def bruteforce(self, ld, rd, cfg):
        return self.O.bruteforce(ld, rd, cfg.t_match, cfg.ratio)

    def phase_a(self, soa, left, pose, cam, pcfg, scale, levels):
        return self.O.run_phase_a(soa, left.u, left.v, left.octave, left.descriptors,
                                  _grid(self.O, left, cam), pose, cam, pcfg, scale, levels)

    def sbp_rot(self, soa, left, pose, cam, pcfg, scale, levels, ref_angles, u_offset):
        return self.O.search_by_projection(soa, left.u, left.v, left.octave, left.descriptors,
                                           left.angle, _grid(self.O, left, cam), pose, cam, pcfg,
                                           scale, levels, ref_angles=ref_angles,
                                           rotation_check=True, u_offset=u_offset)

    def slp(self, soa, left, right, slots, pose, cam, pcfg, scale, levels):
        s = np.asarray(slots, np.int64).copy()
        n = self.O.search_local_points(soa.point_ids, soa, left.u, left.v, left.octave,
                                       left.descriptors, _grid(self.O, left, cam), s, pose, cam,
                                       pcfg, scale, levels)
        return n, s

    def prev(self, prev_slots, prev_pose, left, right, pose, soa_by_id, cam, pcfg):
        """projection.py:231-253 composed from the oracle's search."""
        slot_idx = np.nonzero(prev_slots != -1)[0]
        pids = prev_slots[slot_idx]
        if len(slot_idx) == 0:
            return None, pids
        rel = pose.matrix() @ np.linalg.inv(prev_pose.matrix())
        fwd = float(rel[2, 3])
        u_off = math.copysign(pcfg.prev_u_offset_px, fwd) if abs(fwd) > 1e-9 else 0.0
        c = self.O.search_by_projection(soa_by_id(pids), left.u, left.v, left.octave,
                                        left.descriptors, left.angle, _grid(self.O, left, cam),
                                        pose, cam, pcfg, 1.2, 8,
                                        ref_angles=left.angle[slot_idx],
                                        rotation_check=pcfg.rotation_check_prev,
                                        window_px=pcfg.window_prev_px, u_offset=u_off)
        return c, pids


class DeviceImpl:
    """The same stages through the B200 drop-in (C ABI)."""

    def __init__(self):
        import paper_2509_10757_b200 as ft
        self.ft = ft

    def stereo_refine(self, left, right, pl, pr, cam, cfg, sp):
        ft = self.ft
        # the tracker's three calls (tracker.py:418-427) ...
        idx, dist = ft.match_pinhole_phase1(left, right, cam.height, sp, cfg)
        m = ft.reject_outliers(ft.refine_match_phase2(pl, pr, left, right, idx, dist, cam, cfg),
                               cfg)
        # ... and the fused ComputeStereoMatches agree
        f = ft.compute_stereo_matches(left, right, cam, cfg, sp, pl, pr)
        for k in FIELDS:
            _eq(getattr(f, k), getattr(m, k), f"fused {k}")
        return m

    def stereo_fc(self, left, right, cam, cfg, sp):
        ft = self.ft
        idx, dist = ft.match_pinhole_phase1(left, right, cam.height, sp, cfg)
        m = ft.reject_outliers(ft.matches_from_candidates(idx, dist, left, right, cam, cfg), cfg)
        f = ft.compute_stereo_matches(left, right, cam, cfg, sp)
        for k in FIELDS:
            _eq(getattr(f, k), getattr(m, k), f"fused {k}")
        return m

    def bruteforce(self, ld, rd, cfg):
        from types import SimpleNamespace
        from paper_2509_10757_b200.stereo import fisheye_bruteforce
        z = lambda n: np.zeros(n)  # noqa: E731
        lf = SimpleNamespace(u=z(len(ld)), v=z(len(ld)), octave=np.zeros(len(ld), np.int32),
                             descriptors=ld)
        rf = SimpleNamespace(u=z(len(rd)), v=z(len(rd)), octave=np.zeros(len(rd), np.int32),
                             descriptors=rd)
        return fisheye_bruteforce(lf, rf, cfg)

    def _frame(self, left, right, pose, cam, slots=None):
        from paper_2509_10757_b200.types import Frame, FrameGrid
        g = FrameGrid(left.u, left.v, cam.width, cam.height, 48)
        n = len(left.u)
        s = np.full(n, -1, np.int64) if slots is None else np.asarray(slots, np.int64).copy()
        return Frame(0, 0.0, left, right, np.full(n, -1.0), s, pose, g)

    def phase_a(self, soa, left, pose, cam, pcfg, scale, levels):
        return self.ft.run_phase_a(soa, self._frame(left, left, pose, cam), pose, cam, pcfg,
                                   scale, levels)

    def sbp_rot(self, soa, left, pose, cam, pcfg, scale, levels, ref_angles, u_offset):
        return self.ft.search_by_projection(soa, self._frame(left, left, pose, cam), pose, cam,
                                            pcfg, scale, levels, ref_angles=ref_angles,
                                            rotation_check=True, u_offset=u_offset)

    def slp(self, soa, left, right, slots, pose, cam, pcfg, scale, levels):
        from paper_2509_10757_b200.types import LocalMap
        f = self._frame(left, right, pose, cam, slots)
        n = self.ft.search_local_points(LocalMap((0,), soa.point_ids.copy(), soa), f, cam, pcfg,
                                        scale, levels)
        return n, f.slots

    def prev(self, prev_slots, prev_pose, left, right, pose, soa_by_id, cam, pcfg):
        world = _World(soa_by_id)
        prev = self._frame(left, right, prev_pose, cam, prev_slots)
        cur = self._frame(left, right, pose, cam)
        return self.ft.search_prev_frame(prev, cur, pose, world, cam, pcfg, 1.2, 8)


class _World:
    def __init__(self, soa_by_id):
        from types import SimpleNamespace
        full = soa_by_id(None)
        self.points = {int(p): SimpleNamespace(point_id=int(p), position=full.positions[i],
                                               descriptor=full.descriptors[i],
                                               normal=full.normals[i],
                                               min_distance=float(full.min_distances[i]),
                                               max_distance=float(full.max_distances[i]))
                       for i, p in enumerate(full.point_ids)}


@pytest.fixture(params=["oracle", pytest.param("device", marks=pytest.mark.gpu)])
def impl(request):
    if request.param == "oracle":
        from oracle import oracle as O
        O.lib()
        return OracleImpl(O)
    return DeviceImpl()


# ---------------------------------------------------------------------------

@pytest.mark.parametrize("k", range(len(STEREO_SWEEP)))
def test_stereo_sweep(impl, k):
    d, d1, d2, d3 = (G.load("sweeps.npz"), G.load("cfg1_stereo.npz"), G.load("cfg2_frame_map.npz"),
                     G.load("cfg3_fisheye.npz"))
    cfg, cam = StereoMatchConfig(**STEREO_SWEEP[k]), G.pinhole()
    m = impl.stereo_refine(G.feats(d1, "left"), G.feats(d1, "right"), G.pyramid(d1, "l"),
                           G.pyramid(d1, "r"), cam, cfg, d1["scale_pow"])
    assert_matches(m, d, f"s{k}_cfg1")
    m2 = impl.stereo_fc(G.feats(d2, "left"), G.feats(d2, "right"), cam, cfg, d2["scale_pow"])
    assert_matches(m2, d, f"s{k}_cfg2")
    bi, bd = impl.bruteforce(d3["left_desc"], d3["right_desc"], cfg)
    _eq(bi, d[f"s{k}_bf_idx"], "bf idx")
    _eq(bd, d[f"s{k}_bf_dist"], "bf dist")


def _clip(f, levels):
    f.octave = np.minimum(np.asarray(f.octave), levels - 1).astype(np.int32)
    return f


@pytest.mark.parametrize("j", range(len(SCALES)))
@pytest.mark.parametrize("k", range(len(PROJ_SWEEP)))
def test_projection_sweep(impl, k, j):
    d, d2 = G.load("sweeps.npz"), G.load("cfg2_frame_map.npz")
    scale, levels = SCALES[j]
    pcfg, cam = ProjectionSearchConfig(**PROJ_SWEEP[k]), G.pinhole()
    left, right = _clip(G.feats(d2, "left"), levels), G.feats(d2, "right")
    soa, pose = G.soa(d2), G.pose(d2)
    t = f"p{k}_{j}"
    kp, kd, ko = impl.phase_a(soa, left, pose, cam, pcfg, scale, levels)
    _eq(kp, d[f"{t}_kp"], "kp")
    _eq(kd, d[f"{t}_dist"], "dist")
    _eq(ko, d[f"{t}_oct"], "oct")
    c = impl.sbp_rot(soa, left, pose, cam, pcfg, scale, levels, d["proj_ref_angles"], -1.0)
    assert_corr(c, d, f"{t}_corr")
    n, slots = impl.slp(soa, left, right, np.full(len(left.u), -1), pose, cam, pcfg, scale,
                        levels)
    assert n == int(d[f"{t}_count"])
    _eq(slots, d[f"{t}_slots"], "slots")


@pytest.mark.parametrize("j", [1, 2])
def test_scale_extraction_stereo(impl, j):
    d = G.load("scales.npz")
    t = f"x{j}"
    scale = SCALES[j][0]
    sub = {k[len(t) + 1:]: v for k, v in d.items() if k.startswith(t + "_")}
    m = impl.stereo_refine(G.feats(sub, "left"), G.feats(sub, "right"),
                           G.pyramid(sub, "l", scale), G.pyramid(sub, "r", scale), G.pinhole(),
                           StereoMatchConfig(), sub["scale_pow"])
    assert_matches(m, sub, "final")


def test_cfg5_high_load(impl):
    d = G.load("cfg5_high_load.npz")
    cam, cfg, pcfg = G.pinhole(), StereoMatchConfig(), ProjectionSearchConfig()
    left, right, soa, pose = G.feats(d, "left"), G.feats(d, "right"), G.soa(d), G.pose(d)
    assert len(left.u) > 2000 and len(soa.point_ids) == 20000
    m = impl.stereo_fc(left, right, cam, cfg, d["scale_pow"])
    assert_matches(m, d, "final")
    kp, kd, ko = impl.phase_a(soa, left, pose, cam, pcfg, 1.2, 8)
    _eq(kp, d["pa_kp"], "kp")
    _eq(kd, d["pa_dist"], "dist")
    _eq(ko, d["pa_oct"], "oct")
    n, slots = impl.slp(soa, left, right, d["slots_in"], pose, cam, pcfg, 1.2, 8)
    assert n == int(d["count"])
    _eq(slots, d["slots"], "slots")


@pytest.mark.parametrize("motion", ["fwd", "back", "static"])
def test_search_prev_frame_reference(impl, motion):
    """The reference's own search_prev_frame outputs; static motion is
    SPEC.md:352 (every slotted point re-matches its own keypoint)."""
    from paper_2509_10757_b200.types import Pose
    d, d2 = G.load("prev_frame.npz"), G.load("cfg2_frame_map.npz")
    cam, pcfg = G.pinhole(), ProjectionSearchConfig()
    left, right, soa, pose = G.feats(d2, "left"), G.feats(d2, "right"), G.soa(d2), G.pose(d2)
    row = {int(p): i for i, p in enumerate(soa.point_ids)}

    def soa_by_id(ids):
        if ids is None:
            return soa
        r = np.array([row[int(p)] for p in ids], dtype=np.int64)
        return type(soa)(positions=soa.positions[r], descriptors=soa.descriptors[r],
                         normals=soa.normals[r], min_distances=soa.min_distances[r],
                         max_distances=soa.max_distances[r], point_ids=np.asarray(ids, np.int64))

    cur_pose = Pose(pose.rotation, d[f"{motion}_trans"])
    c, pids = impl.prev(d["prev_slots"], pose, left, right, cur_pose, soa_by_id, cam, pcfg)
    assert_corr(c, d, motion)
    _eq(pids, d[f"{motion}_pids"], "pids")
    if motion == "static":
        assert (d["prev_slots"][c.keypoint_idx] == np.asarray(pids)[c.point_idx]).all()
        assert len(c.point_idx) == int((d["prev_slots"] != -1).sum())


def test_search_prev_frame_empty(impl):
    """a previous frame with zero map points -> empty result."""
    d2 = G.load("cfg2_frame_map.npz")
    left, right, soa, pose = G.feats(d2, "left"), G.feats(d2, "right"), G.soa(d2), G.pose(d2)
    c, pids = impl.prev(np.full(len(left.u), -1, np.int64), pose, left, right, pose,
                        lambda ids: soa, G.pinhole(), ProjectionSearchConfig())
    assert (c is None or len(c.point_idx) == 0) and len(pids) == 0
