"""GPU parity of the resident, graph-captured FramePipeline (ft_track_frames):
several independent frame streams per launch, repeated graph replays (the
barrier / epoch counters must carry across launches), and enough streams to
force multiple frame waves per group slot."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

FIELDS = ("right_idx", "distance", "disparity", "refined_u", "depth", "sad")


@pytest.fixture(scope="module")
def workloads():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from synthetic import make_workload
    return [make_workload(seed=100 + i, n_landmarks=12000, map_points=5000, images=True,
                          offset=0.05 * i, id_base=100_000 * i) for i in range(4)]


@pytest.fixture(scope="module")
def expected(workloads, oracle):
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    out = []
    for i, w in enumerate(workloads):
        m = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam,
                                  StereoMatchConfig(), w.scale_pow)
        rng = np.random.default_rng(i)
        slots_in = np.full(len(w.left.u), -1, np.int64)
        k = rng.choice(len(slots_in), size=60, replace=False)
        slots_in[k] = rng.choice(w.local.point_ids, size=60, replace=False)
        slots = slots_in.copy()
        grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
        n = oracle.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                       w.left.octave, w.left.descriptors, grid, slots, w.pose,
                                       w.cam, ProjectionSearchConfig(), 1.2, 8)
        out.append((m, slots_in, slots, n))
    return out


def _run(workloads, expected, n_streams, replays, raw=False, table=None, build_levels=None):
    from paper_2509_10757_b200.pipeline import FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    cap_pts = max(len(w.local.point_ids) for w in workloads)
    pipe = FramePipeline(w0.cam, n_streams=n_streams, cap_kp=(cap_kp + 31) // 32 * 32,
                         cap_points=(cap_pts + 255) // 256 * 256, pyramid_geometry=w0.pyr_left,
                         raw_images=raw, map_table=table, build_levels=build_levels)
    for s in range(n_streams):
        w = workloads[s % len(workloads)]
        pipe.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                        slots=expected[s % len(workloads)][1])
    for r in range(replays):
        pipe.replay(copies=True)
        pipe.synchronize()
        for s in range(n_streams):
            w = workloads[s % len(workloads)]
            m, _, slots, n = expected[s % len(workloads)]
            res = pipe.result(s, len(w.left.u))
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                              err_msg=f"stream {s} replay {r} {f}")
            np.testing.assert_array_equal(res.slots, slots, err_msg=f"stream {s} replay {r}")
            assert res.n_slots == n
            assert res.n_matched == int((m.right_idx >= 0).sum())


def test_single_stream_replays(workloads, expected):
    _run(workloads, expected, 1, 5)


def test_four_streams(workloads, expected):
    _run(workloads, expected, 4, 3)


def test_many_streams_multiple_waves(workloads, expected):
    _run(workloads, expected, 200, 2)


def test_raw_images_pipeline(workloads, expected):
    """Frames ship level-0 images; the device builds the pyramids."""
    _run(workloads, expected, 1, 3, raw=True)
    _run(workloads, expected, 8, 2, raw=True)


def test_hybrid_pyramid_levels(workloads, expected):
    """Raw level 0 + shipped upper levels: the device builds levels
    1..build_levels only (truncated geometry) and the upper levels are
    copied into place; results equal the oracle's."""
    for b in (1, 2, 3, 5):
        _run(workloads, expected, 2, 2, raw=True, build_levels=b)


def test_raw_images_many_streams(workloads, expected):
    """More images than one cooperative wave holds: the pyramid build runs in
    chunks with different blocks-per-image, sharing the barrier counters."""
    _run(workloads, expected, 64, 2, raw=True)
    _run(workloads, expected, 300, 1, raw=True)


def test_synthetic_pyramids_equal_device_build(workloads):
    """The workload generator's numpy pyramid equals the bit-exact device
    build (so raw-image runs compare against the same oracle inputs)."""
    from types import SimpleNamespace
    from paper_2509_10757_b200.pyramid import build_pyramid
    w = workloads[0]
    h, wd = int(w.pyr_left.heights[0]), int(w.pyr_left.widths[0])
    got = build_pyramid(w.pyr_left.data[:h * wd].reshape(h, wd),
                        SimpleNamespace(levels=8, scale=1.2, patch_size=31))
    np.testing.assert_array_equal(got.data, w.pyr_left.data)


def test_resident_map_table(workloads, expected):
    """Frames ship table slots; ft_gather_points rebuilds each frame's local
    map from the resident table (same order -> same tie-breaks)."""
    from paper_2509_10757_b200.maptable import MapTable
    table = MapTable(capacity=64 * 1024)
    _run(workloads, expected, 4, 2, table=table)
    first = table.bytes_uploaded
    assert first > 0
    _run(workloads, expected, 8, 2, table=table)  # all points resident: no delta
    assert table.bytes_uploaded == first


def test_map_table_slots_and_update(workloads):
    import torch
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.maptable import MapTable
    w = workloads[0]
    t = MapTable(capacity=16384)
    t.upsert(w.local.point_ids, w.local.soa)
    s = t.slots(w.local.point_ids)
    assert len(set(s.tolist())) == len(s)
    rec = t.table.cpu().numpy().view(_lib.POINT_RECORD)
    np.testing.assert_array_equal(rec["id"][s], w.local.point_ids)
    np.testing.assert_array_equal(rec["pos"][s], w.local.soa.positions)
    # overwrite one point (a map update) and read it back through the gather
    soa2 = type(w.local.soa)(**{k: np.array(getattr(w.local.soa, k)) for k in
                                ("positions", "descriptors", "normals", "min_distances",
                                 "max_distances", "point_ids")})
    soa2.positions[3] += 1.0
    t.upsert(w.local.point_ids[3:4], _Rows(soa2, [3]))
    s2 = t.slots(w.local.point_ids)
    # copy-on-write: the rewritten point moved, nothing else did
    assert s2[3] != s[3] and (np.delete(s2, 3) == np.delete(s, 3)).all()
    L = _lib.load()

    def gather(slots):
        out = torch.zeros(len(slots) * 112, dtype=torch.uint8, device="cuda")
        idx = torch.from_numpy(slots).cuda()
        cnt = torch.tensor([len(slots)], dtype=torch.int32, device="cuda")
        st = torch.zeros(1, dtype=torch.int32, device="cuda")
        _lib.check(L.ft_gather_points(1, t.ptr, t.capacity, idx.data_ptr(), cnt.data_ptr(),
                                      len(slots), out.data_ptr(), st.data_ptr(), None), "gather")
        torch.cuda.synchronize()
        assert int(st.item()) == 0
        return out.cpu().numpy().view(_lib.POINT_RECORD)

    got = gather(s2)
    np.testing.assert_array_equal(got["pos"][3], soa2.positions[3])
    np.testing.assert_array_equal(got["pos"][4], w.local.soa.positions[4])
    # a step that took its slot list before the update still reads the old record
    old = gather(s)
    np.testing.assert_array_equal(old["pos"][3], w.local.soa.positions[3])
    # retired slots are recycled only after reclaim()
    size = t.size
    assert t.reclaim() == 1
    t.upsert(w.local.point_ids[4:5], _Rows(soa2, [4]))
    assert t.size == size and t.slots(w.local.point_ids[4:5])[0] == s[3]
    with pytest.raises(KeyError):
        t.slots(np.array([10 ** 12]))


class _Rows:
    def __init__(self, soa, rows):
        for k in ("positions", "descriptors", "normals", "min_distances", "max_distances",
                  "point_ids"):
            setattr(self, k, np.asarray(getattr(soa, k))[rows])


def test_async_runner_overlapped_steps(workloads, expected):
    """AsyncRunner: H2D of step k+1 / compute of k / D2H of k-1 overlapped on
    two pipelines; every step's results equal the oracle's."""
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    table = MapTable(capacity=32 * 1024)
    pipes = [FramePipeline(w0.cam, n_streams=2, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left, map_table=table)
             for _ in range(2)]
    staged = []
    for k in range(4):  # step k: streams carry workloads k and k+1
        p = pipes[k % 2]
        for s in range(2):
            w = workloads[(k + s) % 4]
            p.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                         slots=expected[(k + s) % 4][1])
        staged.append(p.staged_inputs())
    runner = AsyncRunner(pipes)
    n_steps = 10
    for k in range(n_steps):
        if k >= 2:
            _check_step(runner.wait(k - 2), workloads, expected, k - 2)
        runner.submit(k, staged[k % 4])
    for k in (n_steps - 2, n_steps - 1):
        _check_step(runner.wait(k), workloads, expected, k)


def _check_step(pipe, workloads, expected, k):
    for s in range(2):
        w = workloads[(k % 4 + s) % 4]
        m, _, slots, n = expected[(k % 4 + s) % 4]
        res = pipe.result(s, len(w.left.u))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                          err_msg=f"step {k} stream {s} {f}")
        np.testing.assert_array_equal(res.slots, slots, err_msg=f"step {k} stream {s}")
        assert res.n_slots == n


@pytest.mark.parametrize("use_table", [False, True])
def test_fisheye_pipeline(oracle, use_table):
    """FisheyePipeline (cfg3 shape): ft_stereo_fisheye + fisheye
    SearchLocalPoints per stream, vs the oracle's brute force, triangulation
    (reference mode) and search_local_points with the KB projection."""
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.pipeline import FisheyePipeline
    from synthetic import make_workload
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    ws = [make_workload(seed=500 + i, n_landmarks=4800, map_points=3050, fisheye=True,
                        offset=0.05 * i, id_base=100_000 * i) for i in range(3)]
    cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
    table = MapTable(capacity=16384) if use_table else None
    pipe = FisheyePipeline(ws[0].cam, n_streams=3, cap_kp=2048, cap_points=4096,
                           map_table=table)
    for s, w in enumerate(ws):
        pipe.load_frame(s, w.left, w.right, w.local, w.pose)
    for rep in range(2):
        pipe.replay(copies=True)
        pipe.synchronize()
        for s, w in enumerate(ws):
            r = pipe.result(s, len(w.left.u))
            idx, dist = oracle.bruteforce(w.left.descriptors, w.right.descriptors, cfg.t_match,
                                          cfg.ratio)
            np.testing.assert_array_equal(r["right_idx"], idx)
            np.testing.assert_array_equal(r["distance"], dist)
            lidx, _, pts, _ = oracle.fisheye_triangulate(w.left, w.right, idx, dist, w.cam,
                                                         cfg.ray_gap_ceiling)
            np.testing.assert_array_equal(np.nonzero(r["ok"])[0], lidx)
            np.testing.assert_allclose(r["points"][lidx], pts.reshape(-1, 3), rtol=1e-9,
                                       atol=1e-12)
            slots = np.full(len(w.left.u), -1, np.int64)
            grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
            n = oracle.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                           w.left.octave, w.left.descriptors, grid, slots,
                                           w.pose, w.cam, pcfg, 1.2, 8)
            np.testing.assert_array_equal(r["slots"], slots, err_msg=f"stream {s}")
            assert r["n_slots"] == n


def test_high_load_batched(oracle):
    """cfg5 shape (~2000 kps / image, 20k-point local maps) at 64 streams per
    launch: the map role must split each frame's 20k points over several
    blocks (per-block shared arrays), results equal the oracle's."""
    from paper_2509_10757_b200.pipeline import FramePipeline
    from synthetic import make_workload
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    ws = [make_workload(seed=900 + i, n_landmarks=20000, map_points=20000, images=True,
                        offset=0.05 * i) for i in range(2)]
    cap = (max(max(len(w.left.u), len(w.right.u)) for w in ws) + 31) // 32 * 32
    pipe = FramePipeline(ws[0].cam, n_streams=64, cap_kp=cap, cap_points=20480,
                         pyramid_geometry=ws[0].pyr_left)
    for s in range(64):
        w = ws[s % 2]
        pipe.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    pipe.replay(copies=True)
    pipe.synchronize()
    for i, w in enumerate(ws):
        m = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam,
                                  StereoMatchConfig(), w.scale_pow)
        slots = np.full(len(w.left.u), -1, np.int64)
        grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
        n = oracle.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                       w.left.octave, w.left.descriptors, grid, slots, w.pose,
                                       w.cam, ProjectionSearchConfig(), 1.2, 8)
        for s in (i, i + 62):
            r = pipe.result(s, len(w.left.u))
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(r.matches, f), getattr(m, f),
                                              err_msg=f"stream {s} {f}")
            np.testing.assert_array_equal(r.slots, slots, err_msg=f"stream {s}")
            assert r.n_slots == n


def test_level_range_shipping(workloads, expected):
    """Single-stream ship mode lays the pyramids out as [right 0..L-1 | small
    inputs | left L-1..0]: shipping only input_range() (levels >= the lowest
    left octave) through AsyncRunner gives the oracle's results, even with
    the unshipped levels of the device buffers holding garbage."""
    import torch
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(2)]
    assert pipes[0].level_ranges
    ring = pipes[0].staging_ring(4)
    ranges = []
    for k, w in enumerate(workloads):
        pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                            slots=expected[k][1])
        pipes[0].stage_into(ring[k])
        ranges.append(pipes[0].input_range())
        lo, hi = ranges[-1]
        assert hi - lo < pipes[0].in_end  # octaves 5-7: lower levels not shipped
    for p in pipes:
        p.dev.fill_(0xAB)  # unshipped levels hold garbage
        p.capture()
    runner = AsyncRunner(pipes)
    for k in range(8):
        if k >= 2:
            _check_one(runner.wait(k - 2), workloads, expected, (k - 2) % 4)
        runner.submit(k, ring[k % 4], ranges[k % 4])
    for k in (6, 7):
        _check_one(runner.wait(k), workloads, expected, k % 4)


def _check_one(pipe, workloads, expected, i):
    w = workloads[i]
    m, _, slots, n = expected[i]
    res = pipe.result(0, len(w.left.u))
    for f in FIELDS:
        np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f), err_msg=f)
    np.testing.assert_array_equal(res.slots, slots)
    assert res.n_slots == n


@pytest.mark.parametrize("packed", [True, False])
def test_multi_stream_level_ranges(workloads, expected, packed):
    """S > 1 ship mode: per step only the small inputs and each stream's
    needed pyramid levels cross PCIe -- packed into one region and placed by
    ft_copy_ranges (packed) or as S + 1 separate ranges -- with every other
    byte of the device inputs holding garbage; results equal the oracle's."""
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    S = 5
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=S, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left,
                           packed_upload=packed) for _ in range(3)]
    assert pipes[0].packed == packed
    ring = pipes[0].staging_ring(4)
    ranges = []
    for k in range(4):
        for s in range(S):
            w = workloads[(k + s) % 4]
            pipes[0].load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                                slots=expected[(k + s) % 4][1])
        pipes[0].stage_into(ring[k])
        ranges.append(pipes[0].input_ranges())
        assert len(ranges[-1]) == (1 if packed else S + 1)
        assert sum(hi - lo for lo, hi in ranges[-1]) < pipes[0].h2d_bytes()
    for p in pipes:
        p.dev.fill_(0xAB)
        p.capture()
    runner = AsyncRunner(pipes)

    def check(pipe, k):
        for s in range(S):
            i = (k % 4 + s) % 4
            w = workloads[i]
            m, _, slots, n = expected[i]
            res = pipe.result(s, len(w.left.u))
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                              err_msg=f"step {k} stream {s} {f}")
            np.testing.assert_array_equal(res.slots, slots, err_msg=f"step {k} stream {s}")
            assert res.n_slots == n

    for k in range(9):
        if k >= 3:
            check(runner.wait(k - 3), k - 3)
        runner.submit(k, ring[k % 4], ranges[k % 4])
    for k in (6, 7, 8):
        check(runner.wait(k), k)
    runner.close()


def test_copy_ranges_alignments():
    """ft_copy_ranges at every source/destination alignment and odd length
    (vector body + byte head/tail, and the byte path for mismatched
    residues); zero-length segments are no-ops."""
    import ctypes
    import torch
    from paper_2509_10757_b200 import _lib
    lib = _lib.load()
    base = torch.zeros(1 << 20, dtype=torch.uint8, device="cuda")
    src = torch.randint(0, 256, (200_000,), dtype=torch.uint8, device="cuda")
    base[:200_000] = src
    desc, want, dst = [], [], 300_000
    for so, n in ((0, 1), (3, 17), (16, 4096), (5, 12345), (7, 0), (1, 70_001)):
        d = dst + (so % 16 if n % 2 else (so + 3) % 16)
        desc.append((so, d, n))
        want.append((d, src[so:so + n].clone()))
        dst = d + n + 64
    dd = torch.tensor(desc, dtype=torch.int64, device="cuda").reshape(-1)
    _lib.check(lib.ft_copy_ranges(base.data_ptr(), dd.data_ptr(), len(desc),
                                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)),
               "ft_copy_ranges")
    torch.cuda.synchronize()
    for d, v in want:
        assert torch.equal(base[d:d + len(v)], v)
    assert lib.ft_copy_ranges(None, dd.data_ptr(), 1, None) == -1


@pytest.mark.timeout(180)
@pytest.mark.parametrize("n_streams,use_table", [(1, False), (2, False), (1, True)])
def test_persistent_runner(workloads, expected, n_streams, use_table):
    """Persistent runner: one long-lived track kernel serves 3 slots, steps
    handed over by device flags (no launch per step); every step's results
    equal the oracle's, including with level-range shipping (S = 1) and
    garbage in the unshipped bytes."""
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    S = n_streams
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    table = None
    if use_table:  # map points read in place from the resident table
        from paper_2509_10757_b200.maptable import MapTable
        table = MapTable(capacity=32 * 1024)
    pipes = [FramePipeline(w0.cam, n_streams=S, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left,
                           packed_upload=False, map_table=table) for _ in range(3)]
    ring = pipes[0].staging_ring(4)
    ranges = []
    for k in range(4):
        for s in range(S):
            w = workloads[(k + s) % 4]
            pipes[0].load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                                slots=expected[(k + s) % 4][1])
        pipes[0].stage_into(ring[k])
        ranges.append(pipes[0].input_ranges())
    for p in pipes:
        p.dev.fill_(0xAB)
    try:
        runner = AsyncRunner(pipes, persistent=True)
    except _lib.FtError as exc:
        # a grid that would hold (nearly) every SM is refused up front
        assert "status -2" in str(exc) and S > 1
        pipes[0].replay(copies=False)
        pipes[0].synchronize()
        return

    def check(pipe, k):
        for s in range(S):
            i = (k % 4 + s) % 4
            w = workloads[i]
            m, _, slots, n = expected[i]
            res = pipe.result(s, len(w.left.u))
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                              err_msg=f"step {k} stream {s} {f}")
            np.testing.assert_array_equal(res.slots, slots, err_msg=f"step {k} stream {s}")
            assert res.n_slots == n

    try:
        n_steps = 40
        for k in range(n_steps):
            if k >= 3:
                check(runner.wait(k - 3), k - 3)
            runner.submit(k, ring[k % 4], ranges[k % 4])
        for k in range(n_steps - 3, n_steps):
            check(runner.wait(k), k)
    finally:
        runner.close()
    # the kernel has ended: ordinary launches run again on the same pipelines
    pipes[0].replay(copies=False)
    pipes[0].synchronize()


@pytest.mark.timeout(180)
@pytest.mark.parametrize("groups", [2, 4])
def test_persistent_runner_groups(workloads, expected, groups):
    """Persistent runner with step groups: 4 slots, `groups` steps computed at
    once on disjoint SMs; every step equals the oracle."""
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(4)]
    ring = pipes[0].staging_ring(4)
    ranges = []
    for k in range(4):
        w = workloads[k]
        pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                            slots=expected[k][1])
        pipes[0].stage_into(ring[k])
        ranges.append(pipes[0].input_ranges())
    for p in pipes:
        p.dev.fill_(0xAB)
    runner = AsyncRunner(pipes, persistent=True, groups=groups)

    def check(pipe, k):
        w = workloads[k % 4]
        m, _, slots, n = expected[k % 4]
        res = pipe.result(0, len(w.left.u))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                          err_msg=f"step {k} {f}")
        np.testing.assert_array_equal(res.slots, slots, err_msg=f"step {k}")
        assert res.n_slots == n

    try:
        n_steps = 41
        for k in range(n_steps):
            if k >= 4:
                check(runner.wait(k - 4), k - 4)
            runner.submit(k, ring[k % 4], ranges[k % 4])
        for k in range(n_steps - 4, n_steps):
            check(runner.wait(k), k)
    finally:
        runner.close()
    with pytest.raises(ValueError):
        AsyncRunner(pipes[:3], persistent=True, groups=2)


@pytest.mark.timeout(180)
@pytest.mark.parametrize("arena,m,groups", [(True, 2, 1), (True, 4, 2), (True, 4, 1),
                                            (False, 2, 1)])
def test_persistent_runner_batched_submit(workloads, expected, arena, m, groups):
    """submit_batch: m consecutive steps per call.  With the slots in one
    DeviceArena each range is one strided 2D copy for all m steps
    (ft_runner_submit_batch); without it, step-by-step copies.  Every step
    equals the oracle either way (each step is still its own frame)."""
    from paper_2509_10757_b200.pipeline import AsyncRunner, DeviceArena, FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    ar = DeviceArena(4) if arena else None
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left, arena=ar)
             for _ in range(4)]
    if arena:
        pitch = pipes[1].dev.data_ptr() - pipes[0].dev.data_ptr()
        assert pitch > 0 and all(p.dev.data_ptr() == pipes[0].dev.data_ptr() + j * pitch
                                 for j, p in enumerate(pipes))
    ring = pipes[0].staging_ring(4)
    for k in range(4):
        w = workloads[k]
        pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                            slots=expected[k][1])
        pipes[0].stage_into(ring[k])
    full = [(0, pipes[0].in_end)]  # one range for every step of a batch
    for p in pipes:
        p.dev.fill_(0xAB)
    runner = AsyncRunner(pipes, persistent=True, groups=groups)

    def check(pipe, k):
        w = workloads[k % 4]
        mt, _, slots, n = expected[k % 4]
        res = pipe.result(0, len(w.left.u))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(res.matches, f), getattr(mt, f),
                                          err_msg=f"step {k} {f}")
        np.testing.assert_array_equal(res.slots, slots, err_msg=f"step {k}")
        assert res.n_slots == n

    try:
        n_steps, k = 40, 0
        while k < n_steps:
            for j in range(k - 4, k + m - 4):  # results about to be overwritten
                if j >= 0:
                    check(runner.wait(j), j)
            runner.submit_batch(k, ring[k % 4:k % 4 + m], full)
            k += m
        for j in range(n_steps - 4, n_steps):
            check(runner.wait(j), j)
    finally:
        runner.close()


@pytest.mark.timeout(180)
def test_tail_blocks_per_launch(workloads, expected, monkeypatch):
    """The dedicated stereo-tail / map-resolve blocks (persistent plans' mode)
    forced on ordinary launches: same results as the group-barrier path."""
    monkeypatch.setenv("FT_TAIL_LAUNCH", "1")
    _run(workloads, expected, 1, 3)
    _run(workloads, expected, 3, 2)
    from paper_2509_10757_b200.maptable import MapTable
    _run(workloads, expected, 1, 2, table=MapTable(capacity=32 * 1024))


@pytest.mark.timeout(180)
@pytest.mark.parametrize("groups", [1, 2, 4])
def test_resident_ring(workloads, expected, groups):
    """ft_track_frames_ring: 11 steps over 4 resident pipelines in one
    persistent launch (each pipeline runs 2-3 times), with 1 / 2 / 4 step
    groups (that many frames in flight on disjoint SMs); every pipeline's
    final outputs equal the oracle's."""
    import torch
    from paper_2509_10757_b200.pipeline import FramePipeline, run_ring
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(4)]
    for i, (p, w) in enumerate(zip(pipes, workloads)):
        p.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                     slots=expected[i][1])
        p.dev[:p.in_end].copy_(p.host[:p.in_end])
        p.dev[p.out_begin:p.out_end].fill_(0x5A)  # nothing stale can pass
    torch.cuda.synchronize()
    run_ring(pipes, 11, groups=groups)
    pipes[0].synchronize()
    for i, (p, w) in enumerate(zip(pipes, workloads)):
        p.copy_outputs()
        m, _, slots, n = expected[i]
        res = p.result(0, len(w.left.u))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f), err_msg=f)
        np.testing.assert_array_equal(res.slots, slots)
        assert res.n_slots == n
    run_ring(pipes, 0, groups=groups)  # no-op
    with pytest.raises(ValueError):
        run_ring(pipes[:3], 4, groups=2)  # slots must be a multiple of the groups


@pytest.mark.timeout(300)
def test_persistent_high_load(oracle):
    """cfg5 shape (~2000 kps, 20k-point maps) through the persistent runner: the
    plan's geometry leaves SMs for the tail blocks (every SM would be needed
    otherwise), results equal the oracle's."""
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    from synthetic import make_workload
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    ws = [make_workload(seed=910 + i, n_landmarks=20000, map_points=20000, images=True,
                        offset=0.05 * i, id_base=1_000_000 * (i + 1)) for i in range(2)]
    cap = (max(max(len(w.left.u), len(w.right.u)) for w in ws) + 31) // 32 * 32
    table = MapTable(capacity=2 * 20480 + 1024)
    pipes = [FramePipeline(ws[0].cam, n_streams=1, cap_kp=cap, cap_points=20480,
                           pyramid_geometry=ws[0].pyr_left, map_table=table)
             for _ in range(4)]
    ring = pipes[0].staging_ring(2)
    for k, w in enumerate(ws):
        pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
        pipes[0].stage_into(ring[k])
    want = []
    for w in ws:
        m = oracle.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam,
                                  StereoMatchConfig(), w.scale_pow)
        slots = np.full(len(w.left.u), -1, np.int64)
        grid = oracle.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
        n = oracle.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                       w.left.octave, w.left.descriptors, grid, slots, w.pose,
                                       w.cam, ProjectionSearchConfig(), 1.2, 8)
        want.append((m, slots, n))
    runner = AsyncRunner(pipes, persistent=True)
    try:
        for k in range(10):
            if k >= 4:
                pipe = runner.wait(k - 4)
                m, slots, n = want[(k - 4) % 2]
                r = pipe.result(0, len(ws[(k - 4) % 2].left.u))
                for f in FIELDS:
                    np.testing.assert_array_equal(getattr(r.matches, f), getattr(m, f),
                                                  err_msg=f"step {k - 4} {f}")
                np.testing.assert_array_equal(r.slots, slots)
                assert r.n_slots == n
            runner.submit(k, ring[k % 2])
        for k in range(6, 10):
            runner.wait(k)
    finally:
        runner.close()


@pytest.mark.timeout(180)
def test_runner_auto_mode(workloads, expected):
    """persistent="auto": the persistent kernel where the step is one track
    launch, graph launches otherwise (raw images); both give the oracle's
    results."""
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    for raw, want in ((False, True), (True, False)):
        pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                               cap_points=5120, pyramid_geometry=w0.pyr_left, raw_images=raw)
                 for _ in range(2)]
        staged = []
        for k in range(2):
            w = workloads[k]
            pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                                slots=expected[k][1])
            staged.append(pipes[0].staged_inputs())
        runner = AsyncRunner(pipes, persistent="auto")
        try:
            assert runner.persistent == want
            for k in range(4):
                if k >= 2:
                    _check_one(runner.wait(k - 2), workloads, expected, (k - 2) % 2)
                runner.submit(k, staged[k % 2])
            for k in (2, 3):
                _check_one(runner.wait(k), workloads, expected, k % 2)
        finally:
            runner.close()


@pytest.mark.timeout(180)
@pytest.mark.timeout(180)
def test_resident_ring_20_groups(workloads, expected):
    """ft_track_frames_ring at the bench's step-group pick: 20 groups of 7
    blocks (4 stereo + 3 map each) over 20 resident pipelines, 45 steps
    (every pipeline runs 2-3 times): every pipeline's outputs equal the
    oracle's."""
    import torch
    from paper_2509_10757_b200.pipeline import FramePipeline, run_ring
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(20)]
    for i, p in enumerate(pipes):
        w = workloads[i % 4]
        p.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                     slots=expected[i % 4][1])
        p.dev[:p.in_end].copy_(p.host[:p.in_end])
        p.dev[p.out_begin:p.out_end].fill_(0x5A)
    torch.cuda.synchronize()
    run_ring(pipes, 45, groups=20)
    pipes[0].synchronize()
    for i, p in enumerate(pipes):
        w = workloads[i % 4]
        p.copy_outputs()
        m, _, slots, n = expected[i % 4]
        res = p.result(0, len(w.left.u))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f), err_msg=f)
        np.testing.assert_array_equal(res.slots, slots)
        assert res.n_slots == n


@pytest.mark.timeout(240)
def test_resident_ring_35_groups_multi_batch(workloads, expected):
    """ft_track_frames_ring at 35 step groups: 4 blocks per group, so a frame
    has ONE stereo block holding every left keypoint -- the block-batched
    stereo passes then run several 384-keypoint batches (records re-staged
    per batch on mbar[1]).  Every pipeline's outputs equal the oracle's."""
    import torch
    from paper_2509_10757_b200.pipeline import FramePipeline, run_ring
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    assert max(len(w.left.u) for w in workloads) > 384  # more than one batch per block
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(35)]
    for i, p in enumerate(pipes):
        w = workloads[i % 4]
        p.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                     slots=expected[i % 4][1])
        p.dev[:p.in_end].copy_(p.host[:p.in_end])
        p.dev[p.out_begin:p.out_end].fill_(0x5A)
    torch.cuda.synchronize()
    run_ring(pipes, 70, groups=35)
    pipes[0].synchronize()
    for i, p in enumerate(pipes):
        w = workloads[i % 4]
        p.copy_outputs()
        m, _, slots, n = expected[i % 4]
        res = p.result(0, len(w.left.u))
        for f in FIELDS:
            np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f), err_msg=f)
        np.testing.assert_array_equal(res.slots, slots)
        assert res.n_slots == n


def test_resident_ring_multi_stream(workloads, expected):
    """ft_track_frames_ring over 3 pipelines of 2 streams each (2 frames per
    step: group barriers inside the persistent kernel, no tail blocks):
    every pipeline's outputs equal the oracle's."""
    import torch
    from paper_2509_10757_b200.pipeline import FramePipeline, run_ring
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=2, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left, packed_upload=False)
             for _ in range(3)]
    for i, p in enumerate(pipes):
        for s in range(2):
            j = (i + s) % 4
            w = workloads[j]
            p.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                         slots=expected[j][1])
        p.dev[:p.in_end].copy_(p.host[:p.in_end])
    torch.cuda.synchronize()
    run_ring(pipes, 7)
    pipes[0].synchronize()
    for i, p in enumerate(pipes):
        p.copy_outputs()
        for s in range(2):
            j = (i + s) % 4
            w = workloads[j]
            m, _, slots, n = expected[j]
            res = p.result(s, len(w.left.u))
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                              err_msg=f"pipe {i} stream {s} {f}")
            np.testing.assert_array_equal(res.slots, slots)
            assert res.n_slots == n


@pytest.mark.timeout(120)
def test_persistent_runner_guard(workloads, expected):
    """While a persistent runner holds the GPU's SMs, calls that would need a
    cooperative track launch raise instead of hanging; after close() they run."""
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline, run_ring
    import paper_2509_10757_b200 as ft
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(2)]
    w = workloads[0]
    pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    r = AsyncRunner(pipes, persistent=True)
    try:
        with pytest.raises(_lib.FtError):
            ft.compute_stereo_matches(w.left, w.right, w.cam)
        with pytest.raises(_lib.FtError):
            pipes[1].replay()
        with pytest.raises(_lib.FtError):
            run_ring(pipes, 2)
        with pytest.raises(_lib.FtError):
            AsyncRunner(pipes, persistent=True)
        r.submit(0)
        r.wait(0)
    finally:
        r.close()
    m = ft.compute_stereo_matches(w.left, w.right, w.cam, scale_pow=w.scale_pow,
                                  left_pyr=w.pyr_left, right_pyr=w.pyr_right)
    np.testing.assert_array_equal(m.right_idx, expected[0][0].right_idx)


@pytest.mark.timeout(120)
def test_persistent_runner_idle_gaps(workloads, expected):
    """Real-time cadence: steps submitted with idle gaps (the pump sleeps on
    its condition variable once nothing is in flight) still complete, in
    order, with the oracle's results, and promptly after each submit."""
    import time
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    w0 = workloads[0]
    cap_kp = max(max(len(w.left.u), len(w.right.u)) for w in workloads)
    pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=(cap_kp + 31) // 32 * 32,
                           cap_points=5120, pyramid_geometry=w0.pyr_left) for _ in range(2)]
    ring = pipes[0].staging_ring(2)
    ranges = []
    for k in range(2):
        w = workloads[k]
        pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right,
                            slots=expected[k][1])
        pipes[0].stage_into(ring[k])
        ranges.append(pipes[0].input_ranges())
    runner = AsyncRunner(pipes, persistent=True)
    try:
        for k in range(6):
            time.sleep(0.01)  # 10 ms with nothing in flight: the pump is asleep
            t0 = time.perf_counter()
            runner.submit(k, ring[k % 2], ranges[k % 2])
            res = runner.wait(k).result(0, len(workloads[k % 2].left.u))
            assert time.perf_counter() - t0 < 0.5
            m, _, slots, n = expected[k % 2]
            for f in FIELDS:
                np.testing.assert_array_equal(getattr(res.matches, f), getattr(m, f),
                                              err_msg=f"step {k} {f}")
            np.testing.assert_array_equal(res.slots, slots)
    finally:
        runner.close()
