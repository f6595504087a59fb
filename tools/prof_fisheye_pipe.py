"""cfg3 FisheyePipeline step breakdown: fisheye stereo alone, local-map search
alone, and the two-branch graph, each CUDA-event timed after an L2 flush."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2509_10757_b200 import _lib  # noqa: E402
from paper_2509_10757_b200.pipeline import FisheyePipeline  # noqa: E402
from synthetic import make_workload  # noqa: E402

w = make_workload(seed=700, n_landmarks=4800, map_points=3050, fisheye=True)
pipe = FisheyePipeline(w.cam, n_streams=1, cap_kp=1536, cap_points=4096)
pipe.load_frame(0, w.left, w.right, w.local, w.pose)
pipe.capture()
pipe.replay(copies=True)
pipe.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = pipe.stream


def timed(fn, n=20, warm=False):
    ts = []
    for _ in range(n):
        with torch.cuda.stream(s):
            if not warm:
                flush.fill_(1)
                flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        fn()
        b.record(s)
        s.synchronize()
        ts.append(a.elapsed_time(b))
    return 1e3 * float(np.median(ts))


def bf():
    _lib.check(pipe.lib.ft_stereo_fisheye(1, pipe.kl, pipe.kr, 50, 0.8, pipe.tri, pipe._d("idx"),
                                          pipe._d("dist"), pipe._d("ok"), pipe._d("pts"), pipe.ws,
                                          s.cuda_stream), "bf")


def proj():
    _lib.check(pipe.lib.ft_project_search(1, pipe.points, pipe.kl, pipe.pparams, pipe.pio,
                                          pipe.pmode, pipe.pout, pipe.ws, s.cuda_stream), "proj")


def graph():
    with torch.cuda.stream(s):
        pipe.graph_compute.replay()


for name, fn in (("fisheye stereo", bf), ("map search", proj), ("graph (both)", graph)):
    print(f"{name:16s} cold {timed(fn):7.1f} us   warm {timed(fn, warm=True):7.1f} us")
