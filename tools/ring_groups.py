"""Persistent ring value vs step groups: cfg2 frames resident in R
pipelines (> 2x L2), ONE ft_track_frames_ring launch of K steps, groups
G in {1,2,3,4} (G frames in flight on disjoint SMs), CUDA events; every
pipeline's outputs checked against the oracle after each configuration."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10757_b200.pipeline import FramePipeline, run_ring  # noqa: E402

NF = 8
frames = bench.make_frames(NF, 1000, True)
ck = int(max(max(len(f.left.u), len(f.right.u)) for f in frames) + 31) // 32 * 32
cp = int(max(len(f.local.point_ids) for f in frames) + 255) // 256 * 256
args = type("A", (), {"no_map_table": False})()
table, _ = bench.make_table(args, frames, cp)
w0 = frames[0]
probe = FramePipeline(w0.cam, 1, ck, cp, pyramid_geometry=w0.pyr_left, map_table=table)
R = -(-(256 << 20) // probe.in_end)
RM = int(os.environ.get("RING_R_MULT", "112"))  # R: a multiple of every group count tried
R = (R + RM - 1) // RM * RM
pipes = []
for i in range(R):
    p = FramePipeline(w0.cam, 1, ck, cp, pyramid_geometry=w0.pyr_left, map_table=table)
    f = frames[i % NF]
    p.load_frame(0, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
    p.capture()
    pipes.append(p)
torch.cuda.synchronize()
s = pipes[0].stream
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
ok_all = True
for G in [int(x) for x in os.environ.get("RING_GROUPS", "1,2,3,4").split(",")]:
    for K in (20, 200):
        try:
            run_ring(pipes, max(R, 2 * G), s, groups=G)  # plans + warm
        except Exception as e:  # noqa: BLE001
            print(f"G={G}: {type(e).__name__}: {e}")
            break
        torch.cuda.synchronize()
        best = None
        for rep in range(3):
            a, b = ev(), ev()
            a.record(s)
            run_ring(pipes, K, s, groups=G)
            b.record(s)
            torch.cuda.synchronize()
            ms = a.elapsed_time(b)
            best = ms if best is None else min(best, ms)
        # parity: outputs cleared, one ring pass over every pipeline, vs the oracle
        for p in pipes:
            p.dev[p.out_begin:p.out_end].fill_(0x5A)
        torch.cuda.synchronize()
        run_ring(pipes, R, s, groups=G)
        torch.cuda.synchronize()
        ok = True
        for i in range(0, R, max(1, R // 12)):
            pipes[i].copy_outputs()
            try:
                ok &= bool(bench.spot_check(pipes[i], frames[i % NF]))
            except SystemExit:
                ok = False
        ok_all &= ok
        print(f"G={G} K={K}: {1e3 * best / K:.2f} us/frame -> {K / best * 1e3:.0f} frames/s "
              f"(parity {ok})", flush=True)
print("ALL_OK" if ok_all else "PARITY_FAIL")
