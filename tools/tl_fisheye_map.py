"""Timeline (FT_DEBUG_TIMELINE) of the cfg3 fisheye map-only launch."""
import os
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2509_10757_b200 import _lib  # noqa: E402
from paper_2509_10757_b200.pipeline import FisheyePipeline  # noqa: E402
from synthetic import make_workload  # noqa: E402

path = os.environ["FT_DEBUG_TIMELINE"]
w = make_workload(seed=700, n_landmarks=4800, map_points=3050, fisheye=True)
pipe = FisheyePipeline(w.cam, n_streams=1, cap_kp=1536, cap_points=4096)
pipe.load_frame(0, w.left, w.right, w.local, w.pose)
with torch.cuda.stream(pipe.stream):
    pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end], non_blocking=True)
for _ in range(4):
    _lib.check(pipe.lib.ft_project_search(1, pipe.points, pipe.kl, pipe.pparams, pipe.pio,
                                          pipe.pmode, pipe.pout, pipe.ws,
                                          pipe.stream.cuda_stream), "proj")
    pipe.synchronize()
lines = open(path).read().strip().split("\n")
st = [i for i, l in enumerate(lines) if l.startswith("launch")]
T = np.array([[int(x) for x in l.split()[1:]] for l in lines[st[-1] + 1:]], dtype=np.float64)
t0 = T[:, 0][T[:, 0] > 0].min()
names = ["start", "staged+csr+hash", "projected", "searched", "barrier", "end", "table landed",
         "points landed"]
print(lines[st[-1]])
for k, n in enumerate(names):
    c = T[:, k]
    c = c[c > 0]
    if len(c):
        r = (c - t0) / 1e3
        print(f"  {n:18s} min {r.min():7.2f} med {np.median(r):7.2f} max {r.max():7.2f}")
