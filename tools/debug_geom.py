import os, sys
os.environ["FT_DEBUG_GEOMETRY"] = "1"
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import golden_io as G
import paper_2509_10757_b200 as ft
from paper_2509_10757_b200.types import StereoMatchConfig
import torch
print(torch.cuda.get_device_properties(0))
d = G.load("cfg1_stereo.npz")
left, right = G.feats(d, "left"), G.feats(d, "right")
cam, cfg = G.pinhole(), StereoMatchConfig()
idx, dist = ft.match_pinhole_phase1(left, right, cam.height, d["scale_pow"], cfg)
pl, pr = G.pyramid(d, "l"), G.pyramid(d, "r")
m = ft.refine_match_phase2(pl, pr, left, right, idx, dist, cam, cfg)
ft.reject_outliers(m, cfg)
f = ft.compute_stereo_matches(left, right, cam, cfg, d["scale_pow"], pl, pr)
print("ok")
