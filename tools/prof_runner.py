"""Diagnose AsyncRunner overlap: per-step wall time of (a) the native runner,
(b) a torch-stream version of the same schedule, (c) H2D alone, (d) compute
alone, on the cfg2 single-stream pipeline."""
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

w = make_workload(seed=1000, n_landmarks=12000, map_points=5000, images=True, id_base=1)
table = MapTable(capacity=8192)
table.upsert(w.local.point_ids, w.local.soa)
pipes = [FramePipeline(w.cam, n_streams=1, cap_kp=1280, cap_points=5120,
                       pyramid_geometry=w.pyr_left, map_table=table) for _ in range(2)]
for p in pipes:
    p.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
    p.capture()
staged = pipes[0].staged_inputs()
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200
many = [pipes[0].staged_inputs() for _ in range(8)]


def run_native_many():
    r = AsyncRunner(pipes)
    for k in range(2):
        r.submit(k, many[k % 8])
    r.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        if k >= 2:
            r.wait(k - 2)
        r.submit(k, many[k % 8])
    r.wait(N - 1)
    r.wait(N - 2)
    dt = time.perf_counter() - t0
    r.close()
    return 1e6 * dt / N


def run_native():
    r = AsyncRunner(pipes)
    for k in range(2):
        r.submit(k, staged)
    r.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        if k >= 2:
            r.wait(k - 2)
        r.submit(k, staged)
    r.wait(N - 1)
    r.wait(N - 2)
    dt = time.perf_counter() - t0
    r.close()
    return 1e6 * dt / N


def run_torch():
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    ev = [{k: torch.cuda.Event() for k in ("h2d", "comp", "d2h")} for _ in pipes]

    def submit(k):
        i = k % 2
        p, e = pipes[i], ev[i]
        h2d.wait_event(e["comp"])
        with torch.cuda.stream(h2d):
            p.dev[:p.in_end].copy_(staged, non_blocking=True)
            e["h2d"].record(h2d)
        comp.wait_event(e["h2d"])
        comp.wait_event(e["d2h"])
        with torch.cuda.stream(comp):
            p.graph_compute.replay()
            e["comp"].record(comp)
        d2h.wait_event(e["comp"])
        with torch.cuda.stream(d2h):
            p.host[p.out_begin:p.out_end].copy_(p.dev[p.out_begin:p.out_end], non_blocking=True)
            e["d2h"].record(d2h)

    for k in range(2):
        submit(k)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        if k >= 2:
            ev[(k - 2) % 2]["d2h"].synchronize()
        submit(k)
    torch.cuda.synchronize()
    return 1e6 * (time.perf_counter() - t0) / N


def run_h2d():
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for k in range(N):
            pipes[0].dev[:pipes[0].in_end].copy_(staged, non_blocking=True)
    s.synchronize()
    return 1e6 * (time.perf_counter() - t0) / N


def run_comp():
    s = torch.cuda.Stream()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    with torch.cuda.stream(s):
        for k in range(N):
            pipes[0].graph_compute.replay()
    s.synchronize()
    return 1e6 * (time.perf_counter() - t0) / N


for name, fn in (("h2d alone", run_h2d), ("h2d alone", run_h2d), ("compute alone", run_comp),
                 ("native runner", run_native), ("native 8 bufs", run_native_many),
                 ("native 8 bufs", run_native_many), ("torch schedule", run_torch),
                 ("native runner", run_native)):
    print(f"{name:16s} {fn():8.1f} us/step")


def run_h2d_split(parts):
    ss = [torch.cuda.Stream() for _ in range(parts)]
    n = pipes[0].in_end
    bounds = [n * i // parts // 256 * 256 for i in range(parts)] + [n]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                pipes[0].dev[bounds[i]:bounds[i + 1]].copy_(staged[bounds[i]:bounds[i + 1]],
                                                            non_blocking=True)
    torch.cuda.synchronize()
    return 1e6 * (time.perf_counter() - t0) / N


for parts in (1, 2, 4, 1, 2, 4):
    print(f"h2d split {parts}    {run_h2d_split(parts):8.1f} us/step")


def run_native_split():
    """Host time per submit / per wait in the 2-deep loop."""
    r = AsyncRunner(pipes)
    for k in range(4):
        if k >= 2:
            r.wait(k - 2)
        r.submit(k, staged)
    r.synchronize()
    ts, tw = [], []
    for k in range(N):
        t0 = time.perf_counter()
        if k >= 2:
            r.wait(k - 2)
        t1 = time.perf_counter()
        r.submit(k, staged)
        t2 = time.perf_counter()
        tw.append(t1 - t0)
        ts.append(t2 - t1)
    r.synchronize()
    r.close()
    return 1e6 * np.median(ts), 1e6 * np.median(tw)


print("native submit/wait host us: %.1f / %.1f" % run_native_split())


def run_native_ranges(rng, n_slots):
    """Per-step wall time of the native runner with n_slots pipelines and the
    given per-step H2D ranges ([] = no upload)."""
    ps = pipes + [FramePipeline(w.cam, n_streams=1, cap_kp=1280, cap_points=5120,
                                pyramid_geometry=w.pyr_left, map_table=table)
                  for _ in range(n_slots - 2)]
    for p in ps[2:]:
        p.load_frame(0, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
        p.capture()
    r = AsyncRunner(ps)
    for k in range(8):
        if k >= n_slots:
            r.wait(k - n_slots)
        r.submit(k, staged, rng)
    r.synchronize()
    t0 = time.perf_counter()
    for k in range(N):
        if k >= n_slots:
            r.wait(k - n_slots)
        r.submit(k, staged, rng)
    r.synchronize()
    dt = time.perf_counter() - t0
    r.close()
    return 1e6 * dt / N


lo_hi = pipes[0].input_range()
for n_slots in (2, 4):
    print(f"slots={n_slots}: no upload {run_native_ranges([], n_slots):.1f} us/step, "
          f"level range {run_native_ranges([lo_hi], n_slots):.1f} us/step")
