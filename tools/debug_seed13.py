import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2509_10757_b200 as ft
from synthetic import make_workload
from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
from oracle import oracle as O
w = make_workload(seed=13, n_landmarks=20000, map_points=20000, images=True)
cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()
ref = O.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam, cfg, w.scale_pow)
got = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left, w.pyr_right)
for f in ("right_idx", "distance", "disparity", "refined_u", "depth", "sad"):
    a, b = getattr(got, f), getattr(ref, f)
    bad = np.nonzero(a != b)[0]
    print(f, "mismatches", len(bad), bad[:10], a[bad[:5]], b[bad[:5]])
print("n", len(w.left.u), len(w.right.u), "matched", (ref.right_idx >= 0).sum(), (got.right_idx >= 0).sum())
idx, dist = ft.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)
ridx, rdist = O.match_pinhole_phase1(w.left, w.right, 480, w.scale_pow, cfg)
print("phase1 mism", (idx != ridx).sum())
m2 = ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, ridx, rdist, w.cam, cfg)
r2 = O.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right, ridx, rdist, w.cam, cfg)
print("phase2 mism", (m2.right_idx != r2.right_idx).sum(), (m2.sad != r2.sad).sum())
