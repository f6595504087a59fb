"""Native session phase times per call type (FT_SESSION_TIMING=1): pack /
issue / kernel / sync / unpack, on cfg2 frames and the cfg4 stage calls."""
import os
import sys
import time
from pathlib import Path

os.environ.setdefault("FT_SESSION_TIMING", "1")
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

import paper_2509_10757_b200 as ft  # noqa: E402
from paper_2509_10757_b200 import session as S  # noqa: E402
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig  # noqa: E402
from synthetic import make_workload  # noqa: E402

cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
w = make_workload(seed=1000, n_landmarks=12000, map_points=5000, images=True)
fr = w.frame()
ses = S.session()
idx, dist = ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)
m = ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, idx, dist, w.cam, cfg)
for name, fn in (
        ("phase1", lambda: ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)),
        ("refine", lambda: ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, idx,
                                                  dist, w.cam, cfg)),
        ("reject", lambda: ft.reject_outliers(m, cfg)),
        ("fused", lambda: ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow,
                                                    w.pyr_left, w.pyr_right)),
        ("fused_nopyr", lambda: ft.compute_stereo_matches(w.left, w.right, w.cam, cfg,
                                                          w.scale_pow)),
        ("slp", lambda: ft.search_local_points(w.local, fr, w.cam, pcfg, 1.2, 8))):
    for _ in range(10):
        fn()
    ses.stats(reset=True)
    n = 300
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    tot = 1e6 * (time.perf_counter() - t0) / n
    st = ses.stats(reset=True)
    c = max(1.0, st.pop("calls"))
    print(f"{name:12s} total {tot:6.1f} us | " + " ".join(f"{k} {v / c:6.1f}" for k, v in st.items()))
