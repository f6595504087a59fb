"""Profile the reference-facing drop-in path (host side): cProfile over the
tracker-seam calls on cfg2 frames and the cfg4 sequence's stage calls."""
import cProfile
import pstats
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402

import paper_2509_10757_b200 as ft  # noqa: E402
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig  # noqa: E402
from synthetic import make_workload  # noqa: E402

cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
ws = [make_workload(seed=1000 + i, n_landmarks=12000, map_points=5000, images=True) for i in range(4)]


def seam(w):
    idx, dist = ft.match_pinhole_phase1(w.left, w.right, w.cam.height, w.scale_pow, cfg)
    m = ft.reject_outliers(ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right,
                                                  idx, dist, w.cam, cfg), cfg)
    return ft.search_local_points(w.local, w.frame(), w.cam, pcfg, 1.2, 8)


def timeit(name, fn, n=100):
    for k in range(5):
        fn(ws[k % 4])
    ts = []
    for k in range(n):
        t0 = time.perf_counter()
        fn(ws[k % 4])
        ts.append(time.perf_counter() - t0)
    print(f"{name}: median {1e6 * np.median(ts):.0f} us")


w = ws[0]
timeit("phase1", lambda w: ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg))
idx, dist = ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)
timeit("refine", lambda w: ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, idx,
                                                  dist, w.cam, cfg))
m = ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, idx, dist, w.cam, cfg)
timeit("reject", lambda w: ft.reject_outliers(m, cfg))
timeit("fused_stereo", lambda w: ft.compute_stereo_matches(w.left, w.right, w.cam, cfg,
                                                           w.scale_pow, w.pyr_left, w.pyr_right))
timeit("search_local_points", lambda w: ft.search_local_points(w.local, w.frame(), w.cam, pcfg,
                                                               1.2, 8))
timeit("seam", seam)
pr = cProfile.Profile()
pr.enable()
for k in range(100):
    seam(ws[k % 4])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)


def fused_frame(w):
    ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left, w.pyr_right)
    return ft.search_local_points(w.local, w.frame(), w.cam, pcfg, 1.2, 8)


timeit("fused_frame", fused_frame)
pr = cProfile.Profile()
pr.enable()
for k in range(200):
    fused_frame(ws[k % 4])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
