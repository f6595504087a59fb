"""Persistent runner vs graph runner, single stream cfg2 shape (ship mode,
level ranges, resident map table): wall us per step over N steps."""
import os
import sys
import time
from pathlib import Path

import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402
from paper_2509_10757_b200.maptable import MapTable  # noqa: E402
from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline  # noqa: E402

NF = int(os.environ.get("NF", "8"))
ws = bench.make_frames(NF, 1000, True)
CK = int(max(max(len(f.left.u), len(f.right.u)) for f in ws) + 31) // 32 * 32
table = MapTable(capacity=NF * 5120 + 1024)
for w in ws:
    table.upsert(w.local.point_ids, w.local.soa)
NS = int(sys.argv[2]) if len(sys.argv) > 2 else 4
N = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
pipes = [FramePipeline(ws[0].cam, n_streams=1, cap_kp=CK, cap_points=5120,
                       pyramid_geometry=ws[0].pyr_left, map_table=table) for _ in range(NS)]
ring = pipes[0].staging_ring(NF)
ranges = []
for k, w in enumerate(ws):
    pipes[0].load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    pipes[0].stage_into(ring[k])
    rr = pipes[0].input_ranges()
    if os.environ.get("TRUNC_KB"):  # timing experiment: ship only the first TRUNC_KB of each range
        rr = [(lo, min(hi, lo + 1024 * int(os.environ["TRUNC_KB"]))) for lo, hi in rr]
    ranges.append(AsyncRunner.ranges_arg(rr))
for i, p in enumerate(pipes):
    if not os.environ.get("PERSIST_TL_ONLY"):  # (the timeline hook syncs: no capture)
        p.capture()
    p.dev[:p.in_end].copy_(ring[i % NF])  # resident inputs for the no-H2D loops
torch.cuda.synchronize()


def loop(persistent, full=False, empty=False):
    r = AsyncRunner(pipes, persistent=persistent)
    n = r.n
    k = 0
    t0 = time.perf_counter()
    while k < 64 or time.perf_counter() - t0 < 0.3:
        if k >= n:
            r.wait(k - n)
        r.submit(k, ring[k % NF], [] if empty else (None if full else ranges[k % NF]))
        k += 1
    for j in range(k - n, k):
        r.wait(j)
    k0 = k
    t0 = time.perf_counter()
    tw = ts = 0.0
    for k in range(k0, k0 + N):
        a = time.perf_counter()
        if k - k0 >= n:
            r.wait(k - n)
        b = time.perf_counter()
        r.submit(k, ring[k % NF], [] if empty else (None if full else ranges[k % NF]))
        c = time.perf_counter()
        tw += b - a
        ts += c - b
    for j in range(k0 + N - n, k0 + N):
        r.wait(j)
    dt = time.perf_counter() - t0
    r.close()
    print(f"   (host: wait {1e6 * tw / N:.2f} us, submit {1e6 * ts / N:.2f} us per step)")
    return 1e6 * dt / N


if os.environ.get("PERSIST_TL_ONLY"):  # tools/persist_timeline.py
    print("persistent us/step:",
          round(loop(True, empty=os.environ["PERSIST_TL_ONLY"] == "empty"), 2))
for _ in range(2 if not os.environ.get("PERSIST_TL_ONLY") else 0):
    print("graph runner      us/step:", round(loop(False), 2))
    print("persistent runner us/step:", round(loop(True), 2))
if not os.environ.get("PERSIST_TL_ONLY"):
    print("persistent, whole inputs us/step:", round(loop(True, True), 2))
    print("graph, no H2D us/step:", round(loop(False, empty=True), 2))
    print("persistent, no H2D us/step:", round(loop(True, empty=True), 2))


def ts_stats(label):
    """per-step (start, done) device timestamps of the last persistent run
    (FT_DEBUG_PERSIST=<file>)"""
    import numpy as np
    path = os.environ.get("FT_DEBUG_PERSIST")
    if not path or not os.path.exists(path):
        return
    t = np.loadtxt(path, dtype=np.float64)[:, 1:]
    t = t[(t[:, 0] > 0) & (t[:, 1] > 0)]
    t = t[np.argsort(t[:, 0])][-2000:]
    dur = (t[:, 1] - t[:, 0]) / 1e3
    gap = np.diff(t[:, 0]) / 1e3
    print(f"{label}: step start->done us median {np.median(dur):.2f} p10 "
          f"{np.percentile(dur, 10):.2f} p90 {np.percentile(dur, 90):.2f}; start->start "
          f"median {np.median(gap):.2f}")


if os.environ.get("FT_DEBUG_PERSIST") and not os.environ.get("PERSIST_TL_ONLY"):
    loop(True, empty=True)
    ts_stats("persistent no H2D")
    loop(True)
    ts_stats("persistent ranges")
