"""Fixed cost of one ft_track_frames graph replay: the cfg2 pipeline shape
with an empty frame (0 keypoints, 0 map points) vs the real frame."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2509_10757_b200.pipeline import FramePipeline  # noqa: E402
from synthetic import make_workload  # noqa: E402
from paper_2509_10757_b200.types import FeatureSet, LocalMap, MapPointSoA  # noqa: E402

w = make_workload(seed=1000, n_landmarks=12000, map_points=5000, images=True)
pipe = FramePipeline(w.cam, n_streams=1, cap_kp=1280, cap_points=5120, pyramid_geometry=w.pyr_left)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timed(warm):
    ts = []
    for _ in range(30):
        with torch.cuda.stream(pipe.stream):
            pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end], non_blocking=True)
            if not warm:
                flush.fill_(1)
                flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.stream)
        pipe.replay(copies=False)
        b.record(pipe.stream)
        pipe.synchronize()
        ts.append(a.elapsed_time(b))
    return 1e3 * float(np.median(ts))


pipe.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
pipe.capture()
print(f"real frame : cold {timed(False):6.1f} us  warm {timed(True):6.1f} us")
e = FeatureSet(u=np.zeros(0), v=np.zeros(0), octave=np.zeros(0, np.int32), angle=np.zeros(0),
               response=np.zeros(0, np.float32), descriptors=np.zeros((0, 4), np.uint64))
em = LocalMap((0,), np.zeros(0, np.int64), MapPointSoA(np.zeros((0, 3)), np.zeros((0, 4), np.uint64),
                                                      np.zeros((0, 3)), np.zeros(0), np.zeros(0),
                                                      np.zeros(0, np.int64)))
pipe.load_frame(0, e, e, em, w.pose, w.pyr_left, w.pyr_right)
print(f"empty frame: cold {timed(False):6.1f} us  warm {timed(True):6.1f} us")

# in-kernel timeline of the empty frame (eager launch; FT_DEBUG_TIMELINE)
import os  # noqa: E402
if len(sys.argv) > 1:
    os.environ["FT_DEBUG_TIMELINE"] = sys.argv[1]
    for _ in range(3):
        pipe.launch_track(pipe.stream)
        pipe.synchronize()
    lines = open(os.environ["FT_DEBUG_TIMELINE"]).read().strip().split("\n")
    st = [i for i, l in enumerate(lines) if l.startswith("launch")]
    T = np.array([[int(x) for x in l.split()[1:]] for l in lines[st[-1] + 1:]], dtype=np.float64)
    t0 = T[:, 0][T[:, 0] > 0].min()
    last = T.max()
    print("empty frame in-kernel: first start -> last mark %.2f us; starts spread %.2f us"
          % ((last - t0) / 1e3, (T[:, 0][T[:, 0] > 0].max() - t0) / 1e3))
