"""Target for ncu: the bench's value kernel -- ONE ft_track_frames_ring launch
of K steps over R resident cfg2 pipelines (> 2x L2) with G step groups.
Launch 0 is a warm ring; launch 1 is the captured one:
    ncu --set full -k regex:track_persist_kernel -s 1 -c 1 python tools/ncu_ring.py G K"""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2509_10757_b200.pipeline import FramePipeline, run_ring  # noqa: E402

G = int(sys.argv[1]) if len(sys.argv) > 1 else 4
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20
frames = bench.make_frames(8, 1000, True)
ck = int(max(max(len(f.left.u), len(f.right.u)) for f in frames) + 31) // 32 * 32
cp = int(max(len(f.local.point_ids) for f in frames) + 255) // 256 * 256
table, _ = bench.make_table(type("A", (), {"no_map_table": False})(), frames, cp)
w0 = frames[0]
probe = FramePipeline(w0.cam, 1, ck, cp, pyramid_geometry=w0.pyr_left, map_table=table)
R = (-(-(256 << 20) // probe.in_end) + 139) // 140 * 140  # a multiple of 1, 2, 4, 10, 14 (bench)
pipes = []
for i in range(R):
    p = FramePipeline(w0.cam, 1, ck, cp, pyramid_geometry=w0.pyr_left, map_table=table)
    f = frames[i % 8]
    p.load_frame(0, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
    p.dev[:p.in_end].copy_(p.host[:p.in_end])
    pipes.append(p)
torch.cuda.synchronize()
run_ring(pipes, R, groups=G)       # launch 0: warm (plans, L2 / TLB state like the bench)
torch.cuda.synchronize()
run_ring(pipes, K, groups=G)       # launch 1: captured
torch.cuda.synchronize()
for i in range(0, R, R // 8):
    pipes[i].copy_outputs()
    bench.spot_check(pipes[i], frames[i % 8])
print(f"ring G={G} K={K} R={R} ok")
