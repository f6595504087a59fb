"""Per-block phase timeline of ft_track_frames (debug tool, run on the GPU box):
    FT_DEBUG_TIMELINE=gpurun_out/tl.txt python tools/debug_timeline.py"""
import os
import sys

sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import torch

from paper_2509_10757_b200.pipeline import FramePipeline
from synthetic import make_workload

path = os.environ.get("FT_DEBUG_TIMELINE", "/tmp/tl.txt")
streams = int(sys.argv[1]) if len(sys.argv) > 1 else 1
warm = "--warm" in sys.argv
codewarm = "--codewarm" in sys.argv  # flush, then run once on other data (warm code, cold data)
if os.path.exists(path):
    os.remove(path)
w = make_workload(seed=1000, n_landmarks=12000, map_points=5000, images=True)
table = None
if "--table" in sys.argv:
    from paper_2509_10757_b200.maptable import MapTable
    table = MapTable(capacity=8192)
    table.upsert(w.local.point_ids, w.local.soa)
pipe = FramePipeline(w.cam, n_streams=streams, cap_kp=1280, cap_points=5120,
                     pyramid_geometry=w.pyr_left, map_table=table)
pipe2 = FramePipeline(w.cam, n_streams=streams, cap_kp=1280, cap_points=5120,
                      pyramid_geometry=w.pyr_left, map_table=table) if codewarm else None
if pipe2 is not None:
    for s in range(streams):
        pipe2.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    with torch.cuda.stream(pipe.stream):
        pipe2.dev[:pipe2.in_end].copy_(pipe2.host[:pipe2.in_end], non_blocking=True)
for s in range(streams):
    pipe.load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
with torch.cuda.stream(pipe.stream):
    pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end], non_blocking=True)
for it in range(6):
    if not warm:
        with torch.cuda.stream(pipe.stream):
            flush.fill_(1)
            flush.view(torch.int64).sum()
    if pipe2 is not None:
        os.environ.pop("FT_DEBUG_TIMELINE_OFF", None)
        pipe2.launch_track(pipe.stream)
    pipe.launch_track(pipe.stream)
    pipe.synchronize()
# parse the last launch
blocks = []
with open(path) as fp:
    lines = fp.read().strip().split("\n")
starts = [i for i, l in enumerate(lines) if l.startswith("launch")]
hdr = lines[starts[-1]]
for l in lines[starts[-1] + 1:]:
    blocks.append([int(x) for x in l.split()[1:]])
T = np.array(blocks, dtype=np.float64)
print(hdr)
Gs = int(hdr.split("Gs=")[1].split()[0])
Gm = int(hdr.split("Gm=")[1].split()[0])
per = Gs + Gm
t0 = T[:, 0][T[:, 0] > 0].min()
names = {"stereo": ["start", "staged+csr", "phase1/2 done", "barrier", "end", "-", "table landed",
                    "-", "w0 kp loaded", "w0 phase1", "w0 right strip", "w0 sweep", "w0 out",
                    "gathered", "median"],
         "map": ["start", "staged+csr+hash", "projected", "searched", "barrier", "end",
                 "table landed", "points landed"]}
for role, sel in (("stereo", [i for i in range(len(T)) if i % per < Gs]),
                  ("map", [i for i in range(len(T)) if i % per >= Gs])):
    if not sel:
        continue
    R = T[sel]
    print(f"== {role}: {len(sel)} blocks (us since first block start)")
    for k, name in enumerate(names[role]):
        col = R[:, k]
        col = col[col > 0]
        if len(col) == 0:
            continue
        rel = (col - t0) / 1e3
        print(f"  {name:18s} min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f}")
