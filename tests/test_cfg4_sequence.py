"""cfg4 (BASELINE configs[3]): the reference StereoTracker over 100-frame
feature-bundle sequences (line, circle), replayed stage by stage.

tests/golden/make_golden.py:gen_cfg4 ran the reference tracker
(tracker.py:225-393) and captured every call of the hot-path stage functions
it makes per frame:

    _run_stereo (tracker.py:415-427): match_pinhole_phase1 ->
        matches_from_candidates -> reject_outliers
    initial pose (tracker.py:311-314): search_prev_frame
    local map (tracker.py:354-357): search_local_points

with their inputs (frames, the previous frame's slots, predicted / refined
poses, the local map as a set of world points) and sha256 digests of their
outputs.  Here the same calls are replayed through the CPU oracle (CPU, every
round), through the drop-in functions the tracker calls under install(), and
through the resident per-frame pipeline (FramePipeline / AsyncRunner: stereo
and the local-map search in one launch, map points resident in a MapTable).
Every output must be bit-identical to the reference's.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import golden_io as G
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig

TRAJ = ("line", "circle")
SCALE, LEVELS = 1.2, 8
SCALE_POW = SCALE ** np.arange(LEVELS, dtype=np.float64)


@pytest.fixture(scope="module", params=TRAJ)
def seq(request):
    return G.Cfg4(request.param)


def _mdig(m):
    return G.digest(np.asarray(m.right_idx, np.int64), np.asarray(m.distance, np.int64),
                    np.asarray(m.disparity, np.float64), np.asarray(m.refined_u, np.float64),
                    np.asarray(m.depth, np.float64), np.asarray(m.sad, np.int64))


def _cdig(c):
    return G.digest(*(np.asarray(getattr(c, k), np.int64)
                      for k in ("point_idx", "keypoint_idx", "distance", "octave")))


def _frames(seq):
    return [i for i in range(seq.n_frames) if seq.has(i, "stereo_final")]


def _check(got, want, what):
    assert np.array_equal(got, want), what


# ---------------------------------------------------------------------------
# CPU: the oracle reproduces the reference tracker's stage calls

def test_cfg4_fixture_shape(seq):
    st = list(seq.d["status"])
    assert st[0] == "initialized" and st[1:] == ["ok"] * (seq.n_frames - 1)
    assert len(_frames(seq)) == seq.n_frames
    assert all(seq.has(i, "local_count") and seq.has(i, "prev_corr_digest")
               for i in range(1, seq.n_frames))


def test_cfg4_oracle_replay(oracle, seq):
    O = oracle
    cfg, pcfg, cam = StereoMatchConfig(), ProjectionSearchConfig(), seq.cam
    for i in _frames(seq):
        left, right = seq.feats(i, "l"), seq.feats(i, "r")
        idx, dist = O.match_pinhole_phase1(left, right, 480, SCALE_POW, cfg)
        _check(G.digest(np.asarray(idx, np.int64), np.asarray(dist, np.int64)),
               seq.get(i, "stereo_p1"), f"frame {i} phase 1")
        m = O.matches_from_candidates(idx, dist, left, right, cam, cfg)
        _check(_mdig(m), seq.get(i, "stereo_fc"), f"frame {i} from_candidates")
        m = O.reject_outliers(m, cfg)
        _check(_mdig(m), seq.get(i, "stereo_final"), f"frame {i} reject")
        if i == 0:
            continue
        grid = O.frame_grid(left.u, left.v, cam.width, cam.height, 48) + (48,)
        # search_prev_frame (projection.py:224-253)
        prev_slots = seq.get(i, "prev_prev_slots").astype(np.int64)
        pf = int(seq.get(i, "prev_prev_frame"))
        prev_left = seq.feats(pf, "l")
        slot_idx = np.nonzero(prev_slots != -1)[0]
        pids = prev_slots[slot_idx]
        pose = seq.pose(i, "prev_pose")
        prev_pose = seq.pose(i, "prev_prev_pose")
        rel = pose.matrix() @ np.linalg.inv(prev_pose.matrix())
        fwd = float(rel[2, 3])
        u_off = math.copysign(pcfg.prev_u_offset_px, fwd) if abs(fwd) > 1e-9 else 0.0
        corr = O.search_by_projection(seq.world_soa(pids), left.u, left.v, left.octave,
                                      left.descriptors, left.angle, grid, pose, cam, pcfg,
                                      SCALE, LEVELS, ref_angles=prev_left.angle[slot_idx],
                                      rotation_check=pcfg.rotation_check_prev,
                                      window_px=pcfg.window_prev_px, u_offset=u_off)
        _check(_cdig(corr), seq.get(i, "prev_corr_digest"), f"frame {i} search_prev_frame")
        _check(G.digest(pids), seq.get(i, "prev_pids"), f"frame {i} prev pids")
        # search_local_points (localmap.py:79-122)
        ids = seq.local_ids(i)
        slots = seq.get(i, "local_slots_in").astype(np.int64)
        n = O.search_local_points(ids, seq.world_soa(ids), left.u, left.v, left.octave,
                                  left.descriptors, grid, slots, seq.pose(i, "local_pose"), cam,
                                  pcfg, SCALE, LEVELS)
        assert n == int(seq.get(i, "local_count")), f"frame {i} count"
        _check(G.digest(slots), seq.get(i, "local_slots_out"), f"frame {i} slots")


# ---------------------------------------------------------------------------
# B200: the drop-in stage functions (the calls the tracker makes under install())

@pytest.mark.gpu
def test_cfg4_dropin_replay(seq):
    import paper_2509_10757_b200 as ft
    cfg, pcfg, cam = StereoMatchConfig(), ProjectionSearchConfig(), seq.cam
    world = seq.world()
    cap = 4096  # the tracker's prev_soa_* pool buffers (tracker.py:196-201)
    soa_out = ft.MapPointSoA(positions=np.empty((cap, 3)), descriptors=np.empty((cap, 4), np.uint64),
                             normals=np.empty((cap, 3)), min_distances=np.empty(cap),
                             max_distances=np.empty(cap), point_ids=np.empty(cap, np.int64))
    for i in _frames(seq):
        left, right = seq.feats(i, "l"), seq.feats(i, "r")
        # tracker._run_stereo (tracker.py:418-427), pool-style out buffers
        oi, od = np.empty(len(left.u), np.int64), np.empty(len(left.u), np.int64)
        idx, dist = ft.match_pinhole_phase1(left, right, 480, SCALE_POW, cfg, out_idx=oi,
                                            out_dist=od)
        assert idx is oi and dist is od
        _check(G.digest(idx, dist), seq.get(i, "stereo_p1"), f"frame {i} phase 1")
        m = ft.matches_from_candidates(idx, dist, left, right, cam, cfg)
        _check(_mdig(m), seq.get(i, "stereo_fc"), f"frame {i} from_candidates")
        out = ft.reject_outliers(m, cfg)
        assert out is m
        _check(_mdig(m), seq.get(i, "stereo_final"), f"frame {i} reject")
        # the fused ORB-SLAM ComputeStereoMatches: one launch, same result
        fused = ft.compute_stereo_matches(left, right, cam, cfg, SCALE_POW)
        _check(_mdig(fused), seq.get(i, "stereo_final"), f"frame {i} fused stereo")
        if i == 0:
            continue
        pf = int(seq.get(i, "prev_prev_frame"))
        prev = seq.frame(pf, seq.pose(i, "prev_prev_pose"), seq.get(i, "prev_prev_slots"))
        pose = seq.pose(i, "prev_pose")
        cur = seq.frame(i, pose)
        corr, pids = ft.search_prev_frame(prev, cur, pose, world, cam, pcfg, SCALE, LEVELS,
                                          soa_out=soa_out)
        _check(_cdig(corr), seq.get(i, "prev_corr_digest"), f"frame {i} search_prev_frame")
        _check(G.digest(np.asarray(pids, np.int64)), seq.get(i, "prev_pids"), f"frame {i} pids")
        # the tracker's pooled soa_out is filled in place (tracker.py:304-314)
        k = len(pids)
        assert np.shares_memory(pids, soa_out.point_ids)
        _check(soa_out.positions[:k], seq.world_soa(pids).positions, f"frame {i} soa_out")
        frame = seq.frame(i, seq.pose(i, "local_pose"), seq.get(i, "local_slots_in"))
        n = ft.search_local_points(seq.local_map(i), frame, cam, pcfg, SCALE, LEVELS)
        assert n == int(seq.get(i, "local_count")), f"frame {i} count"
        _check(G.digest(frame.slots), seq.get(i, "local_slots_out"), f"frame {i} slots")


@pytest.mark.gpu
def test_cfg4_prev_frame_resident_table(seq):
    """search_prev_frame with the resident MapTable: only points missing from
    the table are decomposed and uploaded (the map delta), results identical."""
    import paper_2509_10757_b200 as ft
    from paper_2509_10757_b200.maptable import MapTable
    pcfg, cam = ProjectionSearchConfig(), seq.cam
    world, table = seq.world(), MapTable(capacity=32768)
    uploaded = []
    for i in range(1, seq.n_frames):
        pf = int(seq.get(i, "prev_prev_frame"))
        prev = seq.frame(pf, seq.pose(i, "prev_prev_pose"), seq.get(i, "prev_prev_slots"))
        pose = seq.pose(i, "prev_pose")
        before = table.bytes_uploaded
        corr, pids = ft.search_prev_frame(prev, seq.frame(i, pose), pose, world, cam, pcfg,
                                          SCALE, LEVELS, table=table)
        uploaded.append(table.bytes_uploaded - before)
        _check(_cdig(corr), seq.get(i, "prev_corr_digest"), f"frame {i} search_prev_frame")
    # after the first frame only new map points cross PCIe
    assert sum(uploaded[1:]) < 0.5 * uploaded[0] * (seq.n_frames - 2)


# ---------------------------------------------------------------------------
# B200: the resident per-frame pipeline (stereo + SearchLocalPoints, one launch)

def _pipeline_inputs(seq, i):
    return (seq.feats(i, "l"), seq.feats(i, "r"), seq.local_map(i), seq.pose(i, "local_pose"),
            seq.get(i, "local_slots_in").astype(np.int64))


@pytest.mark.gpu
def test_cfg4_pipeline_replay(seq):
    """FramePipeline (one graph-captured cooperative launch per frame, map
    points resident in a MapTable, frames ship 4-B table slots)."""
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.pipeline import FramePipeline
    table = MapTable(capacity=32768)
    pipe = FramePipeline(seq.cam, n_streams=1, cap_kp=2048, cap_points=8192, map_table=table)
    for i in range(1, seq.n_frames):
        left, right, local, pose, slots = _pipeline_inputs(seq, i)
        pipe.load_frame(0, left, right, local, pose, slots=slots)
        pipe.replay()
        pipe.synchronize()
        r = pipe.result(0, len(left.u))
        _check(_mdig(r.matches), seq.get(i, "stereo_final"), f"frame {i} stereo")
        _check(G.digest(r.slots), seq.get(i, "local_slots_out"), f"frame {i} slots")
        assert r.n_slots == int(seq.get(i, "local_count")), f"frame {i} count"


@pytest.mark.gpu
@pytest.mark.parametrize("persistent", [False, True])
def test_cfg4_async_runner_replay(seq, persistent):
    """AsyncRunner: the sequence's frames submitted back to back (copies of
    step k+1 overlap the compute of step k; persistent=True: one long-lived
    track kernel), every step checked."""
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    table = MapTable(capacity=32768)
    pipes = [FramePipeline(seq.cam, n_streams=1, cap_kp=2048, cap_points=8192, map_table=table)
             for _ in range(4)]
    staged = []
    for i in range(1, seq.n_frames):
        p = pipes[0]
        left, right, local, pose, slots = _pipeline_inputs(seq, i)
        p.load_frame(0, left, right, local, pose, slots=slots)
        staged.append(p.staged_inputs())
    runner = AsyncRunner(pipes, persistent=persistent)
    try:
        for k, inp in enumerate(staged):
            runner.submit(k, inp)
            if k >= 2:
                _check_step(seq, runner, k - 2)
        for k in range(max(0, len(staged) - 2), len(staged)):
            _check_step(seq, runner, k)
    finally:
        runner.close()


def _check_step(seq, runner, k):
    i = k + 1
    p = runner.wait(k)
    r = p.result(0, len(seq.feats(i, "l").u))
    _check(_mdig(r.matches), seq.get(i, "stereo_final"), f"frame {i} stereo")
    _check(G.digest(r.slots), seq.get(i, "local_slots_out"), f"frame {i} slots")
    assert r.n_slots == int(seq.get(i, "local_count")), f"frame {i} count"


class _Pool:
    """The reference BufferPool's acquire (buffers.py:38-52): views of
    pre-reserved storage."""

    def __init__(self):
        self.buf = {}

    def acquire(self, name, shape, dtype):
        b = self.buf.get(name)
        if b is None:
            b = self.buf[name] = np.empty(4096, dtype)
        return b[:shape[0]]


@pytest.mark.gpu
def test_cfg4_install_fused_run_stereo(seq):
    """install()'s replacement of StereoTracker._run_stereo (one fused launch)
    on every frame: the reference's StereoMatches and its side effect, the
    phase-1 candidates in the pool's stereo_idx / stereo_dist buffers."""
    from types import SimpleNamespace
    from paper_2509_10757_b200.install import _fused_run_stereo
    tracker = SimpleNamespace(cam=seq.cam, stereo=StereoMatchConfig(), pool=_Pool(),
                              extraction=SimpleNamespace(scale_powers=lambda: SCALE_POW.copy()))
    for i in _frames(seq):
        left, right = seq.feats(i, "l"), seq.feats(i, "r")
        m = _fused_run_stereo(tracker, left, right, None, None)
        _check(_mdig(m), seq.get(i, "stereo_final"), f"frame {i} stereo")
        n = len(left.u)
        _check(G.digest(tracker.pool.buf["stereo_idx"][:n], tracker.pool.buf["stereo_dist"][:n]),
               seq.get(i, "stereo_p1"), f"frame {i} pool candidates")


def test_cfg4_oracle_update_local_map(oracle, seq):
    """localmap.py:42-76 (the reference keeps it on the host):
    the oracle's set restatement over the keyframe observation lists gives the
    reference tracker's keyframes and ascending point ids on every frame."""
    for i in range(1, seq.n_frames):
        kfs, ids = oracle.update_local_map(seq.get(i, "local_slots_in"), seq.d["kf_obs"],
                                           seq.d["kf_off"], int(seq.get(i, "update_n_keyframes")))
        _check(kfs.astype(np.int32), seq.get(i, "update_kf_ids"), f"frame {i} keyframes")
        _check(G.digest(ids), seq.get(i, "update_ids_digest"), f"frame {i} point ids")
        _check(ids, seq.local_ids(i), f"frame {i} ids == the searched local map")


@pytest.mark.gpu
def test_cfg4_update_local_map_device(seq):
    """update_local_map on the device (reference
    localmap.py:42-76) over the growing world of the reference run: keyframe
    ids and ascending point ids equal the reference's on every frame; the
    resident local map feeds search_local_points in place (slots equal the
    reference's); its lazily gathered SoA equals the reference's SoA; only
    new keyframes / points cross PCIe."""
    import paper_2509_10757_b200 as ft
    pcfg, cam = ProjectionSearchConfig(), seq.cam
    world = seq.growing_world()
    shipped = []
    from paper_2509_10757_b200.worldmap import world_table
    for i in range(1, seq.n_frames):
        world.advance(int(seq.get(i, "update_n_keyframes")), int(seq.get(i, "update_n_points")))
        frame = seq.frame(i, seq.pose(i, "local_pose"), seq.get(i, "local_slots_in"))
        before = world_table(world).bytes_uploaded if i > 1 else 0
        local = ft.update_local_map(frame, world)
        shipped.append(world_table(world).bytes_uploaded - before)
        _check(np.asarray(local.keyframe_ids, np.int32), seq.get(i, "update_kf_ids"),
               f"frame {i} keyframes")
        _check(G.digest(np.asarray(local.point_ids, np.int64)), seq.get(i, "update_ids_digest"),
               f"frame {i} point ids")
        n = ft.search_local_points(local, frame, cam, pcfg, SCALE, LEVELS)
        assert n == int(seq.get(i, "local_count")), f"frame {i} count"
        _check(G.digest(frame.slots), seq.get(i, "local_slots_out"), f"frame {i} slots")
        if i % 17 == 1:  # the lazily gathered SoA (decompose_map_points order)
            s = local.soa
            _check(G.digest(s.positions, s.descriptors, s.normals, s.min_distances,
                            s.max_distances, s.point_ids), seq.get(i, "update_soa_digest"),
                   f"frame {i} soa")
    # the world is mirrored once: per frame only the keyframes / points added since
    assert max(shipped[1:]) < 0.5 * world_table(world).bytes_uploaded


@pytest.mark.gpu
def test_cfg4_prev_frame_resident_world(seq):
    """install(resident_world=True): search_prev_frame reads the previous
    frame's points from the world mirror update_local_map keeps in HBM;
    correspondences and point ids equal the reference's on every frame."""
    import paper_2509_10757_b200 as ft
    from paper_2509_10757_b200 import projection as P
    pcfg, cam = ProjectionSearchConfig(), seq.cam
    world = seq.growing_world()
    P._RESIDENT_WORLD = True
    try:
        for i in range(1, seq.n_frames):
            world.advance(int(seq.get(i, "update_n_keyframes")),
                          int(seq.get(i, "update_n_points")))
            pf = int(seq.get(i, "prev_prev_frame"))
            prev = seq.frame(pf, seq.pose(i, "prev_prev_pose"), seq.get(i, "prev_prev_slots"))
            pose = seq.pose(i, "prev_pose")
            corr, pids = ft.search_prev_frame(prev, seq.frame(i, pose), pose, world, cam, pcfg,
                                              SCALE, LEVELS)
            _check(_cdig(corr), seq.get(i, "prev_corr_digest"), f"frame {i} search_prev_frame")
            _check(G.digest(np.asarray(pids, np.int64)), seq.get(i, "prev_pids"), f"frame {i}")
    finally:
        P._RESIDENT_WORLD = False
