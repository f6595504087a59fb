"""A/B of the fisheye all-pairs kernel at 1, 2, 4 and 64 frames: the cluster
(DSMEM merge) latency path vs the split-K path (FT_FISHEYE_CLUSTER=0 in a
second process).  Prints bench.hamming_roofline's launch times / POPC fraction."""
import json
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10757_b200 import _lib  # noqa: E402

peak = bench.popc_peak(torch, _lib)
r = bench.hamming_roofline(torch, _lib, peak)
print(json.dumps({"cluster_env": os.environ.get("FT_FISHEYE_CLUSTER", "default"), **r}))
