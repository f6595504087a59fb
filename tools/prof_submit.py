"""Where the single-stream AsyncRunner step goes: host time inside submit()
and wait(), the loop's wall time per step, and compute-graph replays alone
(cfg2 shape, ship mode with level ranges, resident map table)."""
import ctypes
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from paper_2509_10757_b200.maptable import MapTable  # noqa: E402
from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline  # noqa: E402
from synthetic import make_workload  # noqa: E402

import os  # noqa: E402
if os.environ.get("NUMA"):
    from paper_2509_10757_b200.runtime import bind_host_to_gpu_numa
    print("numa cpus:", bind_host_to_gpu_numa(0))
NF = int(os.environ.get("NF", "4"))
if os.environ.get("BENCH_FRAMES"):
    sys.path.insert(0, str(ROOT))
    import bench  # noqa: E402
    ws = bench.make_frames(NF, 1000, True)
else:
    ws = [make_workload(seed=1000 + i, n_landmarks=12000, map_points=5000, images=True,
                        id_base=100_000 * (i + 1), offset=0.05 * i) for i in range(NF)]
CK = int(max(max(len(f.left.u), len(f.right.u)) for f in ws) + 31) // 32 * 32
print("cap_kp", CK, "kps", [len(f.left.u) for f in ws], "min oct",
      [int(f.left.octave.min()) for f in ws])
table = MapTable(capacity=NF * 5120 + 1024)
for w in ws:
    table.upsert(w.local.point_ids, w.local.soa)
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 4
pipes = [FramePipeline(ws[0].cam, n_streams=1, cap_kp=CK, cap_points=5120,
                       pyramid_geometry=ws[0].pyr_left, map_table=table) for _ in range(NS)]
ring = pipes[0].staging_ring(NF)
ranges = []
for k, w in enumerate(ws):
    pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    pipes[0].stage_into(ring[k])
    ranges.append(pipes[0].input_range())
print("range bytes:", [hi - lo for lo, hi in ranges])
for p in pipes:
    p.capture()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 2000


def comp_alone():
    s = pipes[0].stream
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for _ in range(N):
            pipes[0].graph_compute.replay()
    s.synchronize()
    return 1e6 * (time.perf_counter() - t0) / N


def runner_loop(raw_ctypes: bool):
    r = AsyncRunner(pipes)
    lib, h = r.lib, r._r
    rg = [(ctypes.c_uint64 * 2)(lo, hi) for lo, hi in ranges]
    ptrs = [ring[k].data_ptr() for k in range(NF)]
    t_sub = t_wait = 0.0
    n = r.n
    for k in range(8):
        if k >= n:
            r.wait(k - n)
        r.submit(k, ring[k % NF], ranges[k % NF])
    r.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        a = time.perf_counter()
        if k >= n:
            if raw_ctypes:
                lib.ft_runner_wait(h, k - n)
            else:
                r.wait(k - n)
        b = time.perf_counter()
        if raw_ctypes:
            lib.ft_runner_submit_ranges(h, k, ptrs[k % NF], rg[k % NF], 1)
        else:
            r.submit(k, ring[k % NF], ranges[k % NF])
        c = time.perf_counter()
        t_wait += b - a
        t_sub += c - b
    for k in range(N - n, N):
        r.wait(k)
    dt = time.perf_counter() - t0
    r.close()
    return {"wall_us": 1e6 * dt / N, "submit_us": 1e6 * t_sub / N, "wait_us": 1e6 * t_wait / N}


for _ in range(2):
    print("compute alone (graph replays back to back) us/step:", round(comp_alone(), 2))
    print("runner (python submit):", {k: round(v, 2) for k, v in runner_loop(False).items()})
    print("runner (raw ctypes):   ", {k: round(v, 2) for k, v in runner_loop(True).items()})
