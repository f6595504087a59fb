"""Per-block phase timeline of one step of the ring kernel at G step groups
(the last step group 0 ran; FT_DEBUG_TIMELINE marks):
    python tools/ring_timeline.py G K"""
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
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
frames = bench.make_frames(8, 1000, True)
ck = int(max(max(len(f.left.u), len(f.right.u)) for f in frames) + 31) // 32 * 32
cp = int(max(len(f.local.point_ids) for f in frames) + 255) // 256 * 256
table, _ = bench.make_table(type("A", (), {"no_map_table": False})(), frames, cp)
w0 = frames[0]
R = 140
pipes = []
for i in range(R):
    p = FramePipeline(w0.cam, 1, ck, cp, pyramid_geometry=w0.pyr_left, map_table=table)
    f = frames[i % 8]
    p.load_frame(0, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
    p.dev[:p.in_end].copy_(p.host[:p.in_end])
    pipes.append(p)
torch.cuda.synchronize()
run_ring(pipes, R, groups=G)
run_ring(pipes, K, groups=G)
torch.cuda.synchronize()
pipes[0].lib.ft_internal_persist_dump()
lines = open(tl_path).read().strip().split("\n")
starts = [i for i, ln in enumerate(lines) if ln.startswith("launch")]
hdr = lines[starts[-1]]
T = np.array([[int(x) for x in ln.split()[1:]] for ln in lines[starts[-1] + 1:]], dtype=np.float64)
print(hdr)
Gs = int(hdr.split("Gs=")[1].split()[0])
Gm = int(hdr.split("Gm=")[1].split()[0])
per = Gs + Gm
t0 = T[:, 0][T[:, 0] > 0].min()
names = {"stereo": ["start", "staged+csr", "phase1/2 done", "barrier", "end", "-", "table landed",
                    "-", "B phase 1", "G geometry", "C SAD sweeps", "-", "-", "gathered", "median"],
         "map": ["start", "staged+csr+hash", "projected (last round)", "searched", "barrier", "end",
                 "table landed", "points landed", "round 0 projecting", "round 0 done",
                 "round 1 projecting", "round 1 done", "round 2 projecting", "round 2 done",
                 "round 3 projecting", "round 3 done"]}
for role, sel in (("stereo", [i for i in range(len(T)) if i % per < Gs]),
                  ("map", [i for i in range(len(T)) if i % per >= Gs])):
    Rr = T[sel]
    print(f"== {role}: {len(sel)} blocks (us since the step's first block start)")
    for k, name in enumerate(names[role]):
        if name == "-":
            continue
        col = Rr[:, k]
        col = col[col > 0]
        if len(col) == 0:
            continue
        rel = (col - t0) / 1e3
        print(f"  {name:20s} min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f}")
