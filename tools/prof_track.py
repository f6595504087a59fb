"""Profile helper: the fused per-frame kernel (ft_track_frames) over S frame
streams per launch (cfg2 workload, pyramids resident), graph-captured,
CUDA-event timed with an L2 flush before every launch.

    python tools/prof_track.py [S] [iters] [--warm]
"""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2509_10757_b200.pipeline import FramePipeline  # noqa: E402
from synthetic import make_workload  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
S = int(args[0]) if args else 1
iters = int(args[1]) if len(args) > 1 else 20
warm = "--warm" in sys.argv
ws = [make_workload(seed=1000 + i, n_landmarks=12000, map_points=5000, images=True,
                    offset=0.05 * i) for i in range(4)]
cap_kp = (max(max(len(w.left.u), len(w.right.u)) for w in ws) + 31) // 32 * 32
pipe = FramePipeline(ws[0].cam, n_streams=S, cap_kp=cap_kp, cap_points=5120,
                     pyramid_geometry=ws[0].pyr_left)
for s in range(S):
    w = ws[s % 4]
    pipe.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
pipe.capture()
pipe.replay(copies=True)
pipe.synchronize()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
ts = []
for _ in range(iters):
    with torch.cuda.stream(pipe.stream):
        if not warm:
            flush.fill_(1)
            flush.view(torch.int64).sum()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(pipe.stream)
    pipe.replay(copies=False)
    b.record(pipe.stream)
    pipe.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
print(f"S={S} warm={warm} median_ms={ms:.4f} us_per_frame={1e3 * ms / S:.2f} "
      f"frames_per_s={S / (ms / 1e3):.0f}")
