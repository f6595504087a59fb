"""Launch overheads in a CUDA graph: ft_bench_popc (normal launch, no smem)
with the track kernel's grid shape, vs an empty-frame ft_track_frames
(cooperative, 137 KB dynamic smem)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2509_10757_b200 import _lib  # noqa: E402

lib = _lib.load()
s = torch.cuda.Stream()
sink = torch.zeros(1, dtype=torch.int32, device="cuda")


def graph_time(fn, reps=200):
    fn()
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for _ in range(10):
            fn()
    with torch.cuda.stream(s):
        g.replay()
        s.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            g.replay()
        b.record(s)
        s.synchronize()
    return 1e3 * a.elapsed_time(b) / (reps * 10)


for blocks, threads in ((120, 512), (148, 512), (1, 32)):
    t = graph_time(lambda: lib.ft_bench_popc(blocks, threads, 1, sink.data_ptr(), s.cuda_stream))
    print(f"bench_popc {blocks}x{threads}: {t:.2f} us per launch (back to back in a graph)")

# empty-frame track kernel, back to back
from paper_2509_10757_b200.pipeline import FramePipeline  # noqa: E402
from synthetic import make_workload  # noqa: E402
from paper_2509_10757_b200.types import FeatureSet, LocalMap, MapPointSoA  # noqa: E402

w = make_workload(seed=1000, n_landmarks=12000, map_points=5000, images=True)
pipe = FramePipeline(w.cam, n_streams=1, cap_kp=1280, cap_points=5120, pyramid_geometry=w.pyr_left)
e = FeatureSet(u=np.zeros(0), v=np.zeros(0), octave=np.zeros(0, np.int32), angle=np.zeros(0),
               response=np.zeros(0, np.float32), descriptors=np.zeros((0, 4), np.uint64))
em = LocalMap((0,), np.zeros(0, np.int64), MapPointSoA(np.zeros((0, 3)), np.zeros((0, 4), np.uint64),
                                                      np.zeros((0, 3)), np.zeros(0), np.zeros(0),
                                                      np.zeros(0, np.int64)))
pipe.load_frame(0, e, e, em, w.pose, w.pyr_left, w.pyr_right)
with torch.cuda.stream(pipe.stream):
    pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end])
s = pipe.stream
t = graph_time(lambda: pipe.launch_track(pipe.stream), reps=50)
import os  # noqa: E402
print("track empty frame (cooperative): "
      f"{t:.2f} us per launch (back to back in a graph)")

# real cfg2 frame, back to back (no flush: the e2e steady state's compute)
pipe.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
with torch.cuda.stream(pipe.stream):
    pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end])
t = graph_time(lambda: pipe.launch_track(pipe.stream), reps=50)
print(f"track real frame (cooperative): {t:.2f} us per launch (back to back in a graph)")
