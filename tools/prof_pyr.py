"""Profile helper: ft_build_pyramids on N raw 752x480 images (graph-free,
eager), timed with CUDA events on the launching stream.  Used under ncu too.

    python tools/prof_pyr.py [N] [iters]
"""
import sys
from pathlib import Path
from types import SimpleNamespace

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2509_10757_b200 import _lib  # noqa: E402
from paper_2509_10757_b200.pyramid import pyramid_geometry  # noqa: E402
from paper_2509_10757_b200.runtime import make_workspace, pyramid_struct  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 2
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 20
h, w = 480, 752
geo = pyramid_geometry(w, h, 1.2, 8)
total = int(geo.offsets[-1])
lib = _lib.load()
stream = torch.cuda.Stream()
rng = np.random.default_rng(0)
imgs = torch.from_numpy(rng.integers(0, 256, size=(n, h * w), dtype=np.uint8)).cuda()
pyr = torch.zeros(n * ((total + 255) // 256 * 256), dtype=torch.uint8, device="cuda")
ws = make_workspace(lib, torch.device("cuda"), stream, (n + 1) // 2, 1, 1)
ps = pyramid_struct(geo, pyr.data_ptr(), (total + 255) // 256 * 256)
# capture once (host-side planning stays out of the timed region), replay timed
_lib.check(lib.ft_build_pyramids(n, ps, imgs.data_ptr(), h * w, ws, stream.cuda_stream), "pyr")
stream.synchronize()
graph = torch.cuda.CUDAGraph()
with torch.cuda.graph(graph, stream=stream):
    _lib.check(lib.ft_build_pyramids(n, ps, imgs.data_ptr(), h * w, ws, stream.cuda_stream), "pyr")
ts = []
with torch.cuda.stream(stream):
    for i in range(iters):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        graph.replay()
        b.record(stream)
        stream.synchronize()
        ts.append(a.elapsed_time(b))
print(f"n_images={n} median_ms={np.median(ts):.4f} min_ms={np.min(ts):.4f}")
