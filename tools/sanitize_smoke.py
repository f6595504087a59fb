"""Smoke-sized launches of every kernel for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): the fused track kernel (per launch, with
tail blocks, multi-stream), a 2-step resident ring (1 and 2 step groups), the
persistent runner (3 steps), the fisheye brute force + triangulation, the
pyramid build, copy_ranges, gather / scatter and the host-array session.
Every output is checked against the oracle so a sanitizer run also proves
the results."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2509_10757_b200 as ft  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2509_10757_b200.maptable import MapTable  # noqa: E402
from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline, run_ring  # noqa: E402
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig  # noqa: E402
from synthetic import make_workload  # noqa: E402

only = set(sys.argv[1:])


def want(name):
    return not only or name in only


cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
ws = [make_workload(seed=900 + i, n_landmarks=3000, map_points=800, images=True,
                    offset=0.05 * i, id_base=10_000 * (i + 1)) for i in range(2)]
ck = int(max(max(len(w.left.u), len(w.right.u)) for w in ws) + 31) // 32 * 32
cp = 1024
done = []
if want("session"):
    w = ws[0]
    m = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left,
                                  w.pyr_right)
    ref = O.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam, cfg, w.scale_pow)
    assert all(np.array_equal(getattr(m, f), getattr(ref, f)) for f in
               ("right_idx", "distance", "disparity", "refined_u", "depth", "sad"))
    fr = w.frame()
    n = ft.search_local_points(w.local, fr, w.cam, pcfg, 1.2, 8)
    slots = np.full(len(w.left.u), -1, np.int64)
    grid = O.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
    assert n == O.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                      w.left.octave, w.left.descriptors, grid, slots, w.pose,
                                      w.cam, pcfg, 1.2, 8)
    assert np.array_equal(fr.slots, slots)
    done.append("session(stereo, project)")
if want("track"):
    for tail in (False, True):
        if tail:
            os.environ["FT_TAIL_LAUNCH"] = "1"
        p = FramePipeline(ws[0].cam, n_streams=2, cap_kp=ck, cap_points=cp,
                          pyramid_geometry=ws[0].pyr_left)
        for s, w in enumerate(ws):
            p.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
        p.run_eager()
        p.synchronize()
        os.environ.pop("FT_TAIL_LAUNCH", None)
    done.append("track_kernel (group barriers, tail blocks, 2 streams)")
if want("ring"):
    pipes = []
    for i in range(4):
        p = FramePipeline(ws[0].cam, n_streams=1, cap_kp=ck, cap_points=cp,
                          pyramid_geometry=ws[0].pyr_left)
        w = ws[i % 2]
        p.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
        p.dev[:p.in_end].copy_(p.host[:p.in_end])
        pipes.append(p)
    torch.cuda.synchronize()
    for G in (1, 2):
        run_ring(pipes, 4, groups=G)
        torch.cuda.synchronize()
        for i, p in enumerate(pipes):
            p.copy_outputs()
            bench.spot_check(p, ws[i % 2])
    done.append("track_persist_kernel ring (groups 1, 2)")
if want("runner"):
    table = MapTable(capacity=4096)
    pipes = [FramePipeline(ws[0].cam, n_streams=1, cap_kp=ck, cap_points=cp,
                           pyramid_geometry=ws[0].pyr_left, map_table=table) for _ in range(2)]
    ring = pipes[0].staging_ring(2)
    rng = []
    for k, w in enumerate(ws):
        pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
        pipes[0].stage_into(ring[k])
        rng.append(pipes[0].input_ranges())
    r = AsyncRunner(pipes, persistent=True)
    try:
        for k in range(3):
            if k >= 2:
                r.wait(k - 2)
            r.submit(k, ring[k % 2], rng[k % 2])
        for k in range(1, 3):
            bench.spot_check(r.wait(k), ws[k % 2])
    finally:
        r.close()
    done.append("persistent runner (3 steps, resident map table)")
if want("fisheye"):
    fw = make_workload(seed=905, n_landmarks=1500, map_points=500, fisheye=True)
    got = ft.match_fisheye(fw.left, fw.right, fw.cam, cfg, corrected=True)
    bi, bd = O.bruteforce(fw.left.descriptors, fw.right.descriptors, cfg.t_match, cfg.ratio)
    ref = O.fisheye_triangulate(fw.left, fw.right, bi, bd, fw.cam, cfg.ray_gap_ceiling, True)
    assert np.array_equal(got[0], ref[0])
    done.append("fisheye_bf_kernel + triangulation")
if want("pyramid"):
    from types import SimpleNamespace
    from paper_2509_10757_b200.pyramid import build_pyramid
    w = ws[0]
    h, wd = int(w.pyr_left.heights[0]), int(w.pyr_left.widths[0])
    img = w.pyr_left.data[:h * wd].reshape(h, wd)
    pyr = build_pyramid(img, SimpleNamespace(levels=8, scale=1.2, patch_size=31))
    assert np.array_equal(pyr.data, O.build_pyramid(img, 8, 1.2)[0])
    p = FramePipeline(w.cam, n_streams=2, cap_kp=ck, cap_points=cp,
                      pyramid_geometry=w.pyr_left, raw_images=True)
    for s, ww in enumerate(ws):
        p.load_frame(s, ww.left, ww.right, ww.local, ww.pose, ww.pyr_left, ww.pyr_right)
    p.run_eager()
    p.synchronize()
    done.append("pyramid_kernel (single + 2-stream raw-image pipeline)")
if want("copy"):
    p = FramePipeline(ws[0].cam, n_streams=3, cap_kp=ck, cap_points=cp,
                      pyramid_geometry=ws[0].pyr_left, packed_upload=True)
    for s in range(3):
        w = ws[s % 2]
        p.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    p.run_eager()
    p.synchronize()
    done.append("copy_ranges (packed 3-stream upload)")
print("sanitize smoke ok:", "; ".join(done))
