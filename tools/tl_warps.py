"""Debug (FT_TL_WARPS build): per-warp end times of the map role's first
projection round, one ring step at G step groups: python tools/tl_warps.py G"""
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
tl_path = "/tmp/ring_tl.txt"
os.environ["FT_DEBUG_TIMELINE"] = tl_path
os.environ["FT_DEBUG_PERSIST"] = "/tmp/ring_ts.txt"
if os.path.exists(tl_path):
    os.remove(tl_path)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10757_b200.pipeline import FramePipeline, run_ring  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 10
frames = bench.make_frames(8, 1000, True)
ck = int(max(max(len(f.left.u), len(f.right.u)) for f in frames) + 31) // 32 * 32
cp = int(max(len(f.local.point_ids) for f in frames) + 255) // 256 * 256
table, _ = bench.make_table(type("A", (), {"no_map_table": False})(), frames, cp)
w0 = frames[0]
pipes = []
for i in range(140):
    p = FramePipeline(w0.cam, 1, ck, cp, pyramid_geometry=w0.pyr_left, map_table=table)
    f = frames[i % 8]
    p.load_frame(0, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
    p.dev[:p.in_end].copy_(p.host[:p.in_end])
    pipes.append(p)
torch.cuda.synchronize()
run_ring(pipes, 140, groups=G)
run_ring(pipes, 200, groups=G)
torch.cuda.synchronize()
pipes[0].lib.ft_internal_persist_dump()
lines = open(tl_path).read().strip().split("\n")
starts = [i for i, ln in enumerate(lines) if ln.startswith("launch")]
hdr = lines[starts[-1]]
T = np.array([[int(x) for x in ln.split()[1:]] for ln in lines[starts[-1] + 1:]], dtype=np.float64)
Gs = int(hdr.split("Gs=")[1].split()[0])
Gm = int(hdr.split("Gm=")[1].split()[0])
per = Gs + Gm
print(hdr)
for b in [i for i in range(len(T)) if i % per >= Gs][:8]:
    t = T[b]
    t = t[t > 0]
    if len(t) == 0:
        continue
    rel = np.sort((t - t.min()) / 1e3)
    print(f"map block {b}: warp end times (us after the first) {np.round(rel, 2).tolist()}")
