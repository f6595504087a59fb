"""Where a drop-in call's time goes: the native session call vs the Python
around it (cfg2 frame: phase 1 / refine / reject / fused stereo /
search_local_points), host timers."""
import sys
import time
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import paper_2509_10757_b200 as ft  # noqa: E402
from paper_2509_10757_b200 import session as S  # noqa: E402
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig  # noqa: E402
from synthetic import make_workload  # noqa: E402

T = defaultdict(float)
N = defaultdict(int)


class Wrapped:
    def __init__(self, lib):
        self._lib = lib

    def __getattr__(self, name):
        f = getattr(self._lib, name)
        if not name.startswith("ft_session_"):
            return f

        def g(*a):
            t0 = time.perf_counter()
            r = f(*a)
            T[name] += time.perf_counter() - t0
            N[name] += 1
            return r
        return g


ses = S.session()
ses.lib = Wrapped(ses.lib)
for n in ("features", "points", "pyramid", "stereo_params", "project_params", "matches_struct"):
    f0 = getattr(S, n)

    def mk(f0, n):
        def g(*a, **k):
            t0 = time.perf_counter()
            r = f0(*a, **k)
            T["py." + n] += time.perf_counter() - t0
            N["py." + n] += 1
            return r
        return g
    setattr(S, n, mk(f0, n))
cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
w = make_workload(seed=1000, n_landmarks=12000, map_points=5000, images=True)
idx, dist = ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)
m = ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, idx, dist, w.cam, cfg)
fr = w.frame()
for name, fn in (
        ("phase1", lambda: ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)),
        ("refine", lambda: ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, idx,
                                                  dist, w.cam, cfg)),
        ("reject", lambda: ft.reject_outliers(m, cfg)),
        ("fused", lambda: ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow,
                                                    w.pyr_left, w.pyr_right)),
        ("slp", lambda: ft.search_local_points(w.local, fr, w.cam, pcfg, 1.2, 8))):
    for _ in range(10):
        fn()
    T.clear()
    N.clear()
    t0 = time.perf_counter()
    n = 300
    for _ in range(n):
        fn()
    tot = time.perf_counter() - t0
    print(f"== {name}: {1e6 * tot / n:.0f} us per call")
    for k in sorted(T, key=T.get, reverse=True):
        print(f"   {k:24s} {1e6 * T[k] / n:8.1f} us/call  ({N[k] / n:.1f} per call)")
