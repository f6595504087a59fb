"""Benchmark: stereo + local-map tracking at EuRoC shape on B200.

Metric (BASELINE.json): "stereo+local-map tracking ms/frame and frames/s at
EuRoC shape, 1/2/4/8 B200".  Workload = BASELINE configs[1] (cfg2): one
EuRoC-shaped stereo frame (752x480, ~1270 keypoints per image, 8 levels,
scale 1.2, rendered textured images so stereo phase 2 runs on real pyramids)
plus a 5000-point local map; a step is one frame per stream through

    stereo:  phase 1 -> SAD phase 2 -> median-SAD rejection   (ft_stereo_pinhole)
    map:     skip slotted -> project -> window search -> resolve -> slot write
                                                               (ft_project_search)

Default: 1 stream per GPU.  `value` = frames/s of ONE persistent ring launch
over K resident frames (> 2x L2) with G step groups (G frames in flight on
disjoint SMs, picked in the warm-up); `e2e` = the same frames through the
persistent runner with every step's inputs copied from pinned host memory and
its outputs back (host wall clock).  `--gpus N` launches N ranks itself (one
per GPU, torch.distributed.run on 127.0.0.1); each rank drives its own GPU with
independent streams (weak scaling, no collective on the data path; NCCL only
for the barrier, the G broadcast and the max over ranks).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--streams S]
    python bench.py --impl reference ...    # CPU oracle arm (host cores)
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))

PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
RING_GROUPS = (1, 2, 4, 10, 14, 20)  # persistent step-group counts tried (ft_track_plan_groups)
PERSIST_GROUPS = (1, 2, 4)  # ... for the 8-slot persistent runner (e2e)
FALLBACK_HBM = 6650.0


def parse() -> argparse.Namespace:
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=200)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--streams", type=int, default=1, help="frame streams per GPU")
    p.add_argument("--frames", type=int, default=8, help="distinct frames cycled per stream")
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-images", action="store_true", help="feature bundles only (no phase 2)")
    p.add_argument("--pyramid-mode", default="ship", choices=["hybrid", "ship", "device"],
                   help="ship: ship whole pyramids, the reference's phase-2 input (default); "
                        "hybrid: ship level 0 + levels > --build-levels, build levels "
                        "1..build-levels on the device; device: ship level 0, build all")
    p.add_argument("--build-levels", type=int, default=1)
    p.add_argument("--raw-images", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--ship-pyramids", action="store_true", help=argparse.SUPPRESS)
    p.add_argument("--no-map-table", action="store_true",
                   help="ship every frame's local-map records instead of table slots into "
                        "the resident map table")
    p.add_argument("--batched-streams", type=int, default=64,
                   help="extra batched measurement (0 disables)")
    p.add_argument("--cpu-seconds", type=float, default=12.0)
    p.add_argument("--quick", action="store_true", help="skip cpu baseline / batched (profiling)")
    p.add_argument("--no-configs", action="store_true", help="skip the cfg3 / cfg5 measurements")
    p.add_argument("--dist-selftest", action="store_true", help=argparse.SUPPRESS)
    return p.parse_args()


def _free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def self_launch(args) -> int | None:
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per
    GPU) through torch.distributed.run on 127.0.0.1 with the same arguments
    and relay rank 0's line.  Returns the launcher's exit code, or None when
    this process is already a rank (or N == 1)."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return None
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ, OMP_NUM_THREADS=os.environ.get("OMP_NUM_THREADS", "1"))
    return subprocess.run(cmd, env=env).returncode


def dist_selftest(args) -> None:
    """The N-rank plumbing without a GPU (CPU test of the launcher): gloo
    rendezvous, barrier, max-over-ranks of per-rank times, rank-0 line."""
    import torch.distributed as dist
    from paper_2509_10757_b200.sharding import job_frames_per_s, max_over_ranks, streams_of_rank
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1:
        dist.init_process_group("gloo")
    mine = streams_of_rank(args.streams * world, world, rank)
    ms = 10.0 + rank  # stand-in per-rank time
    (max_ms,) = max_over_ranks([ms], dist if world > 1 else None)
    if world > 1:
        dist.barrier()
    if rank == 0:
        print(json.dumps({"metric": "dist selftest", "n_gpus": world, "ranks_streams": len(mine),
                          "max_ms": max_ms,
                          "value": job_frames_per_s(len(mine) * args.steps, world,
                                                    max_ms * args.steps)}), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# workload

def make_frames(n: int, seed0: int, images: bool):
    """n independent cfg2 frames (distinct worlds: map point ids offset per
    frame so they can share one resident map table)."""
    from synthetic import make_workload
    return [make_workload(seed=seed0 + i, n_landmarks=12000, map_points=5000, images=images,
                          offset=0.05 * i, id_base=100_000 * (i + 1)) for i in range(n)]


def make_table(args, frames, cap_pts, S=1):
    """Resident map table holding every frame's local map (uploaded once,
    before timing); None with --no-map-table."""
    if args.no_map_table:
        return None, 0
    from paper_2509_10757_b200.maptable import MapTable
    table = MapTable(capacity=max(len(frames), S) * cap_pts + 1024)
    for f in frames:
        table.upsert(f.local.point_ids, f.local.soa, only_missing=True)
    return table, table.bytes_uploaded


def algorithmic_units(w) -> dict:
    """Per-frame work the reference algorithm performs:
    phase-1 Hamming evaluations (pairs passing the octave/band/disparity
    predicates), SAD candidates, projection-window Hamming evaluations, and
    unique bytes (stereo: keypoints 64 B/kp/side + both pyramids; map: 104 B
    per point + 64 B per keypoint)."""
    from paper_2509_10757_b200.types import StereoMatchConfig
    cfg = StereoMatchConfig()
    L, R = w.left, w.right
    band = cfg.band_factor * w.scale_pow[L.octave]
    dv = np.abs(R.v[None, :] - L.v[:, None])
    disp = L.u[:, None] - R.u[None, :]
    rows = np.clip(np.round(R.v), 0, w.cam.height - 1)
    r0 = np.maximum(np.floor(L.v - band), 0)
    r1 = np.minimum(np.ceil(L.v + band), w.cam.height - 1)
    in_rows = (rows[None, :] >= r0[:, None]) & (rows[None, :] <= r1[:, None])
    ok = (in_rows & (np.abs(R.octave[None, :] - L.octave[:, None]) <= 1) & (dv <= band[:, None])
          & (disp >= cfg.min_disparity) & (disp <= cfg.max_disparity))
    ham_p1 = int(ok.sum())
    cand = int((ok.any(axis=1)).sum())
    n_l, n_r = len(L.u), len(R.u)
    pyr_bytes = 2 * int(w.pyr_left.offsets[-1]) if w.pyr_left is not None else 0
    m = len(w.local.point_ids)
    from oracle import oracle as O
    from paper_2509_10757_b200.types import ProjectionSearchConfig
    grid = O.frame_grid(L.u, L.v, w.cam.width, w.cam.height, 48) + (48,)
    hc: list = []
    O.run_phase_a(w.local.soa, L.u, L.v, L.octave, L.descriptors, grid, w.pose, w.cam,
                  ProjectionSearchConfig(), 1.2, 8, ham_count=hc)
    return {"hamming_phase1": ham_p1, "hamming_projection": hc[0], "sad_candidates": cand,
            "sad_absdiff": cand * 11 * 121,
            "stereo_bytes": (n_l + n_r) * 64 + pyr_bytes,
            "map_bytes": m * 104 + n_l * 64}


# ---------------------------------------------------------------------------
# clocks

class ClockSampler:
    def __init__(self, gpu: int):
        self.gpu = gpu
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)

    def summary(self) -> dict:
        rows = [r for r in self.rows if len(r) >= 7]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# reference arm / CPU baseline (oracle port on host cores)

def cpu_frame(w, nthreads: int) -> int:
    """One frame through the oracle: stereo (phase 1 -> phase 2 | from-cand ->
    reject), FrameGrid, search_local_points.  Returns the filled slots."""
    from oracle import oracle as O
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    O.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam, StereoMatchConfig(),
                     w.scale_pow, nthreads)
    grid = O.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
    slots = np.full(len(w.left.u), -1, np.int64)
    return O.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v,
                                 w.left.octave, w.left.descriptors, grid, slots, w.pose, w.cam,
                                 ProjectionSearchConfig(), 1.2, 8, nthreads)


def cpu_frames_per_s(frames, seconds: float, nthreads: int) -> tuple[float, int]:
    t0 = time.perf_counter()
    done = 0
    while True:
        cpu_frame(frames[done % len(frames)], nthreads)
        done += 1
        el = time.perf_counter() - t0
        if el >= seconds and done >= 3:
            return done / el, done


def host_cpu() -> dict:
    """The host the CPU numbers ran on (lscpu model, logical CPUs usable)."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"model": model, "os_cpu_count": os.cpu_count(),
            "usable_cpus": len(os.sched_getaffinity(0))}


def cpu_baseline(frames, seconds: float) -> dict:
    from oracle import oracle as O
    O.lib()
    nmax = max(1, O.max_threads())
    best = None
    for nt in sorted({1, nmax}):
        fps, n = cpu_frames_per_s(frames, seconds / 2, nt)
        if best is None or fps > best[0]:
            best = (fps, n, nt)
    return {"value": best[0], "unit": "frames/s", "cores": best[2], "kind": "port",
            "host": host_cpu(),
            "sample": f"{best[1]} cfg2 frames (stereo phase1+phase2+reject, FrameGrid, "
                      f"search_local_points) in ~{seconds / 2:.0f} s, oracle/ft_oracle.c "
                      f"OpenMP over items, best of 1 and {nmax} threads"}


def run_reference(args) -> None:
    """The reference arm: the reference's algorithm for the path on the host
    cores.  The reference itself (trackfront, Python + numba) cannot travel
    to the GPU box, so this is its C port (oracle/ft_oracle.c, pinned to the
    reference's outputs by tests/test_oracle_golden.py), all host threads.
    Each step is a bounded sample of >= 1 frame so that at least 50 frames are
    timed (median of >= 50 frames); value = 1 / median frame time
    x streams."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    frames = make_frames(min(args.frames, 4), 1000, not args.no_images)
    from oracle import oracle as O
    O.lib()
    nt = max(1, O.max_threads())
    for k in range(max(args.warmup, 3)):
        cpu_frame(frames[k % len(frames)], nt)
    per_step = max(args.streams, -(-50 // max(1, args.steps)))
    step_s, frame_s = [], []
    for k in range(args.steps):
        t0 = time.perf_counter()
        for s in range(per_step):
            t1 = time.perf_counter()
            cpu_frame(frames[(k * per_step + s) % len(frames)], nt)
            frame_s.append(time.perf_counter() - t1)
        step_s.append(time.perf_counter() - t0)
    med = float(np.median(frame_s))
    value = 1.0 / med
    line = {"metric": "stereo+local-map tracking frames/s at EuRoC shape", "impl": "reference",
            "value": value, "unit": "frames/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * med * args.streams,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64+u32",
            "data": "synthetic", "config": config_dict(args),
            "cpu_baseline": {"value": value, "unit": "frames/s", "cores": nt, "kind": "port",
                             "host": host_cpu(),
                             "frames_timed": len(frame_s),
                             "frame_ms_median": 1e3 * med,
                             "frames_per_s_mean": len(frame_s) / sum(step_s),
                             "sample": f"{len(frame_s)} cfg2 frames ({per_step} per step) "
                                       "through oracle/ft_oracle.c (C port of the reference "
                                       "numba kernels), OpenMP over items; value = 1 / median "
                                       "frame time"},
            "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


def pyramid_mode(args):
    """(raw_images, build_levels) of the pipeline for --pyramid-mode."""
    mode = "device" if args.raw_images else args.pyramid_mode
    if mode == "ship":
        return False, None
    if mode == "device":
        return True, None
    return True, max(1, args.build_levels)


def config_dict(args) -> dict:
    raw, b = pyramid_mode(args)
    if args.no_images:
        img = ", feature bundle (no phase 2)"
    elif not raw:
        img = ", rendered images shipped as pyramids (phase-2 input) -> SAD phase 2"
    elif b is None:
        img = (", rendered images shipped raw (0.36 MB each) -> device pyramid build "
               "(bit-exact build_pyramid) -> SAD phase 2")
    else:
        img = (f", level-0 images + pyramid levels > {b} shipped, levels 1..{b} built on the "
               "device (bit-exact build_pyramid) -> SAD phase 2")
    mp = ("5000-point local map shipped as records every frame" if args.no_map_table else
          "5000-point local map resident in the device map table (frames ship 4-B slots, "
          "read in place by the map role)")
    return {"workload": "cfg2: EuRoC-shaped stereo frame 752x480 (~1270 kps/image, 8 levels, "
                        "scale 1.2" + img + ") + " + mp + "; stereo + SearchLocalPoints per frame",
            "streams_per_gpu": args.streams, "frames_cycled": args.frames,
            "l2": "value: inputs > L2 (resident ring of pipelines, >= 256 MiB of step "
                  "inputs cycled); latency / kernel timings: flushed before every step "
                  "(256 MiB write, then read back)",
            "parallelism": f"independent frame streams x {args.gpus} GPU (no collective)"}


# ---------------------------------------------------------------------------
# our arm

def main() -> None:
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    rc = self_launch(args)
    if rc is not None:
        sys.exit(rc)
    if args.dist_selftest:
        dist_selftest(args)
        return
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    args.gpus = world  # n_gpus / config.parallelism follow the ranks actually running
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    n_dev = torch.cuda.device_count()
    if local_rank >= n_dev:
        if os.environ.get("FT_BENCH_DIST_BACKEND", "nccl") == "nccl":
            raise SystemExit(f"bench.py: rank {rank} needs GPU {local_rank} but only {n_dev} "
                             "are visible (one process per GPU)")
        local_rank = local_rank % n_dev  # rehearsal: several ranks share the visible GPUs
    torch.cuda.set_device(local_rank)
    from paper_2509_10757_b200.runtime import bind_host_to_gpu_numa
    numa_cpus = bind_host_to_gpu_numa(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("FT_BENCH_DIST_BACKEND", "nccl")  # gloo: 1-GPU rehearsal
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    from paper_2509_10757_b200 import _lib
    from paper_2509_10757_b200.pipeline import FramePipeline

    images = not args.no_images
    frames = make_frames(args.frames, 1000 + 97 * rank, images)
    w0 = frames[0]
    cap_kp = int(max(max(len(f.left.u), len(f.right.u)) for f in frames) + 31) // 32 * 32
    cap_pts = int(max(len(f.local.point_ids) for f in frames) + 255) // 256 * 256
    S = args.streams
    raw, build_levels = pyramid_mode(args)
    raw = raw and images
    table, table_bytes = make_table(args, frames, cap_pts)
    pipe = FramePipeline(w0.cam, n_streams=S, cap_kp=cap_kp, cap_points=cap_pts,
                         pyramid_geometry=w0.pyr_left if images else None, raw_images=raw,
                         map_table=table, build_levels=build_levels)

    def load(step: int) -> None:
        for s in range(S):
            f = frames[(step + s) % len(frames)]
            pipe.load_frame(s, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)

    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush_sink = torch.zeros((), dtype=torch.int64, device="cuda")

    def l2_flush():
        # write > L2 (evicts everything), then read it back so the flushed L2
        # holds clean lines rather than 126 MB of dirty write-backs
        with torch.cuda.stream(pipe.stream):
            flush.fill_(1)
            flush_sink.copy_(flush.view(torch.int64).sum())

    # resident ring for the throughput value: R pipelines, each holding one
    # frame's inputs in HBM, together > 2x L2, so back-to-back steps read
    # their inputs cold without a flush between them
    n_res = max(2, min(160, -(-(256 << 20) // pipe.in_end)))
    n_res = (n_res + 139) // 140 * 140  # a multiple of every step-group count tried
    res_pipes = []
    for i in range(n_res):
        rp = FramePipeline(w0.cam, n_streams=S, cap_kp=cap_kp, cap_points=cap_pts,
                           pyramid_geometry=w0.pyr_left if images else None, raw_images=raw,
                           map_table=table, build_levels=build_levels)
        for s_ in range(S):
            f = frames[(i + s_) % len(frames)]
            rp.load_frame(s_, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
        rp.capture()  # runs the step once with copies: inputs now resident
        res_pipes.append(rp)
    torch.cuda.synchronize()
    res_stream = pipe.stream

    def resident_step(k: int) -> None:
        res_pipes[k % n_res].graph_compute.replay()

    load(0)
    pipe.capture()
    # correctness spot check of the resident pipeline against the oracle (rank 0, stream 0)
    pipe.replay(copies=True)
    pipe.synchronize()
    check = spot_check(pipe, frames[0]) if rank == 0 else None

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def preroll(stream):
        # ~100 us of device spin ahead of the start event: the host enqueues
        # the timed launch (and its argument staging) while the device is
        # still busy, so the events bracket device work only, not the host's
        # enqueue latency on an idle device
        with torch.cuda.stream(stream):
            torch.cuda._sleep(200_000)
    # ---- value: inputs resident in HBM, compute graph only -----------------
    for k in range(args.warmup):
        load(k)
        pipe.replay(copies=True)
    pipe.synchronize()
    comp_ms = []
    with ClockSampler(local_rank) as clk:
        # ---- value: back-to-back steps over the resident ring, one stream
        with torch.cuda.stream(res_stream):
            for k in range(max(args.warmup, n_res)):
                resident_step(k)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        ra, rb = ev(), ev()
        preroll(res_stream)
        with torch.cuda.stream(res_stream):
            ra.record(res_stream)
            for k in range(args.steps):
                resident_step(k)
            rb.record(res_stream)
        torch.cuda.synchronize()
        stream_ms = ra.elapsed_time(rb)
        if dist:
            dist.barrier()
        # ---- value, persistent: the same resident ring through ONE persistent
        # launch (ft_track_frames_ring: no launch or hand-off between steps)
        ring_ms, ring_groups, ring_group_ms = None, 1, None
        if not raw:
            try:
                from paper_2509_10757_b200.pipeline import run_ring
                # step groups (G frames in flight on disjoint SMs): picked in
                # the warm-up by timing K-step rings at each G, then ONE timed
                # run at the chosen G
                g_try = {}
                for G in RING_GROUPS:
                    run_ring(res_pipes, max(args.warmup, n_res), res_stream, groups=G)
                    ts = []
                    for _ in range(2):
                        ra, rb = ev(), ev()
                        preroll(res_stream)
                        ra.record(res_stream)
                        run_ring(res_pipes, args.steps, res_stream, groups=G)
                        rb.record(res_stream)
                        torch.cuda.synchronize()
                        ts.append(ra.elapsed_time(rb))
                    g_try[G] = min(ts)
                ring_groups = min(g_try, key=g_try.get)
                if dist:  # every rank runs the same G (rank 0's pick)
                    gt = torch.tensor([ring_groups], device="cuda")
                    dist.broadcast(gt, 0)
                    ring_groups = int(gt.item())
                run_ring(res_pipes, max(args.warmup, n_res), res_stream, groups=ring_groups)
                torch.cuda.synchronize()
                if dist:
                    dist.barrier()
                torch.cuda.synchronize()
                ra, rb = ev(), ev()
                preroll(res_stream)
                ra.record(res_stream)
                run_ring(res_pipes, args.steps, res_stream, groups=ring_groups)
                rb.record(res_stream)
                torch.cuda.synchronize()
                ring_ms = ra.elapsed_time(rb)
                ring_group_ms = {str(G): v for G, v in g_try.items()}
            except Exception as exc:  # noqa: BLE001  (reported; graph value stands)
                print(f"[bench] ring value: {type(exc).__name__}: {exc}", file=sys.stderr)
            if dist:
                dist.barrier()
        # ---- latency: one isolated step at a time, L2 flushed before each
        for k in range(args.steps):
            load(k)
            with torch.cuda.stream(pipe.stream):
                pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end], non_blocking=True)
            l2_flush()
            a, b = ev(), ev()
            a.record(pipe.stream)
            pipe.replay(copies=False)
            b.record(pipe.stream)
            pipe.synchronize()
            comp_ms.append(a.elapsed_time(b))
        torch.cuda.synchronize()
        # ---- e2e: pinned host inputs -> H2D -> compute -> D2H, host wall clock
        e2e_ms, e2e_ev_ms = [], []
        delta0 = pipe.delta_bytes
        for k in range(args.steps):
            load(k)
            l2_flush()
            pipe.synchronize()
            a, b = ev(), ev()
            t0 = time.perf_counter()
            a.record(pipe.stream)
            pipe.replay(copies=True)
            b.record(pipe.stream)
            pipe.synchronize()
            e2e_ms.append(1e3 * (time.perf_counter() - t0))
            e2e_ev_ms.append(a.elapsed_time(b))
        e2e_delta = pipe.delta_bytes - delta0
        if dist:
            dist.barrier()
    clocks = clk.summary()
    # ---- e2e, overlapped: AsyncRunner (H2D of k+1 / compute of k / D2H of k-1
    # concurrently), inputs pre-staged in pinned memory per frame.  Timed outside
    # the nvidia-smi sampler: its polling stalls the host for milliseconds, which
    # is noise at ~50 us per step.
    runner, staged, ranges = make_runner(args, frames, pipe, table, load)
    shipped = float(np.mean([hi - lo for lo, hi in ranges]))
    same_ranges = all(tuple(r) == tuple(ranges[0]) for r in ranges)
    from paper_2509_10757_b200.pipeline import AsyncRunner
    ranges = [AsyncRunner.ranges_arg(r) for r in ranges]  # marshalled once, not per step
    staged_keep = staged  # the pinned ring rows (kept alive: only pointers go to submit)
    staged = [t.data_ptr() for t in staged]
    if dist:
        dist.barrier()
    # warm-up: every staged pinned buffer's first DMA is slow (one cycle), and
    # the GPU / host clocks ramp back up after the staging pause (>= 0.3 s of
    # steps)
    k, tw = 0, time.perf_counter()
    while k < max(args.warmup, 4 * len(staged) + 2) or time.perf_counter() - tw < 0.3:
        if k >= runner.n:
            runner.wait(k - runner.n)
        runner.submit(k, staged[k % len(staged)], ranges[k % len(staged)])
        k += 1
    for j in range(max(0, k - runner.n), k):
        runner.wait(j)
    k0 = k
    t0 = time.perf_counter()
    marks = []
    for k in range(k0, k0 + args.steps):
        if k - k0 >= runner.n:
            runner.wait(k - runner.n)
        runner.submit(k, staged[k % len(staged)], ranges[k % len(staged)])
        marks.append(time.perf_counter())
    for k in range(max(k0, k0 + args.steps - runner.n), k0 + args.steps):
        runner.wait(k)
    async_ms = 1e3 * (time.perf_counter() - t0)
    if os.environ.get("FT_BENCH_DIAG"):
        d = np.diff(np.array([t0] + marks)) * 1e6
        print(f"[diag] async step us: median {np.median(d):.1f} p90 {np.percentile(d, 90):.1f} "
              f"max {d.max():.1f} first {np.round(d[:12], 1).tolist()}", file=sys.stderr)
    runner.close()
    # ---- e2e, persistent runner: the same steps through ONE long-lived track
    # kernel (no launch per step; ft_runner_create_persistent)
    persist_ms = persist_lat_ms = None
    persist_groups, persist_by_g = 1, {}
    if not raw and os.environ.get("FT_BENCH_PERSIST", "1") != "0":
        try:
            from paper_2509_10757_b200.pipeline import AsyncRunner
            # 8 slots: the host-side hand-off chain (H2D -> ready -> kernel ->
            # done -> D2H) is longer than a graph step, so it needs more steps
            # in flight to keep the kernel fed
            n_p = max(2, min(8, int(os.environ.get("FT_BENCH_PERSIST_SLOTS", "8"))))
            ppipes = list(runner.pipes)[:n_p] + [
                FramePipeline(pipe.cam, n_streams=pipe.S, cap_kp=pipe.cap_kp,
                              cap_points=pipe.cap_pts, pyramid_geometry=pipe.pyr,
                              map_table=table) for _ in range(n_p - len(runner.pipes))]
            persist_by_g = {}
            for G in PERSIST_GROUPS:
                pr = AsyncRunner(ppipes, persistent=True, groups=G)
                try:
                    k, tw = 0, time.perf_counter()
                    while (k < max(args.warmup, 4 * len(staged) + 2) or
                           time.perf_counter() - tw < 0.3):
                        if k >= pr.n:
                            pr.wait(k - pr.n)
                        pr.submit(k, staged[k % len(staged)], ranges[k % len(staged)])
                        k += 1
                    for j in range(max(0, k - pr.n), k):
                        pr.wait(j)
                    k0 = k
                    t0 = time.perf_counter()
                    for k in range(k0, k0 + args.steps):
                        if k - k0 >= pr.n:
                            pr.wait(k - pr.n)
                        pr.submit(k, staged[k % len(staged)], ranges[k % len(staged)])
                    for k in range(max(k0, k0 + args.steps - pr.n), k0 + args.steps):
                        pr.wait(k)
                    persist_by_g[G] = 1e3 * (time.perf_counter() - t0)
                    if G == 1:
                        # per-frame latency: one frame in flight at a time (H2D ->
                        # kernel -> D2H -> host), the real-time tracker's
                        # frame-to-result delay
                        lat = []
                        k1 = k0 + args.steps
                        for j in range(min(args.steps, 200)):
                            k = k1 + j
                            a = time.perf_counter()
                            pr.submit(k, staged[k % len(staged)], ranges[k % len(staged)])
                            pr.wait(k)
                            lat.append(1e3 * (time.perf_counter() - a))
                        persist_lat_ms = float(np.median(lat)) if lat else None
                finally:
                    pr.close()
            persist_groups = min(persist_by_g, key=persist_by_g.get)
            persist_ms = persist_by_g[persist_groups]
        except Exception as exc:  # noqa: BLE001  (reported, never fatal)
            print(f"[bench] persistent runner: {type(exc).__name__}: {exc}", file=sys.stderr)

    # ---- e2e, persistent runner with batched submits: m consecutive steps'
    # inputs (rows of the pinned staging ring) go up as ONE strided copy per
    # range into slots that share a DeviceArena (ft_runner_submit_batch): the
    # copy engine's ~3.6 us fixed cost per copy is paid once per m steps.
    # Every step is still its own frame: H2D, track, results back to the host.
    # Measured slower than one submit per step (62-66k vs 71k frames/s at
    # K = 200, profiles/r3_batched_submit_negative.txt): opt-in, FT_BENCH_BATCH=1.
    batch_by = {}
    ring_rows = getattr(runner, "staging", None)
    if (not raw and same_ranges and ring_rows is not None and persist_ms
            and os.environ.get("FT_BENCH_BATCH", "0") != "0"):
        try:
            from paper_2509_10757_b200.pipeline import AsyncRunner, DeviceArena
            n_max = 16
            arena = DeviceArena(n_max)
            apipes = [FramePipeline(pipe.cam, n_streams=pipe.S, cap_kp=pipe.cap_kp,
                                    cap_points=pipe.cap_pts, pyramid_geometry=pipe.pyr,
                                    map_table=table, arena=arena) for _ in range(n_max)]
            nr = len(staged)
            for n_p, m, G in ((8, 2, 2), (8, 4, 2), (16, 1, 2), (16, 2, 2), (16, 4, 2),
                              (16, 4, 1), (16, 8, 2)):
                if nr % m or n_p % m:
                    continue
                if True:
                    pr = AsyncRunner(apipes[:n_p], persistent=True, groups=G)
                    try:
                        def run(k, n_steps):
                            end = k + n_steps
                            while k < end:
                                mm = min(m, end - k)
                                j = k % nr
                                pr.submit_batch(k, ring_rows[j:j + mm], ranges[0])
                                k += mm
                            return k
                        k, tw = 0, time.perf_counter()
                        while k < max(args.warmup, 4 * nr + 2) or time.perf_counter() - tw < 0.3:
                            k = run(k, m)
                        pr.wait(k - 1)
                        t0 = time.perf_counter()
                        k = run(k, args.steps)
                        pr.wait(k - 1)
                        batch_by[f"n{n_p}_m{m}_g{G}"] = 1e3 * (time.perf_counter() - t0)
                    finally:
                        pr.close()
            del apipes, arena
        except Exception as exc:  # noqa: BLE001  (reported, never fatal)
            print(f"[bench] batched persistent runner: {type(exc).__name__}: {exc}",
                  file=sys.stderr)
    batch_ms = min(batch_by.values()) if batch_by else None
    batch_pick = min(batch_by, key=batch_by.get) if batch_by else None

    # ---- per-kernel timing for the roofline (eager, on the launching stream)
    kern = {"pyramids": [], "track": [], "stereo_only": [], "map_only": []}
    for k in range(max(10, args.steps // 2)):
        load(k)
        with torch.cuda.stream(pipe.stream):
            pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end], non_blocking=True)
        for name, fn in (("pyramids", pipe.launch_pyramids), ("track", pipe.launch_track),
                         ("stereo_only", pipe.launch_stereo), ("map_only", pipe.launch_project)):
            l2_flush()
            a, b = ev(), ev()
            a.record(pipe.stream)
            fn(pipe.stream)
            b.record(pipe.stream)
            pipe.synchronize()
            kern[name].append(a.elapsed_time(b))
    track_ms = float(np.median(kern["track"]))

    tot_comp = sum(comp_ms)
    tot_e2e = sum(e2e_ms)
    from paper_2509_10757_b200.sharding import job_frames_per_s, max_over_ranks
    tot_comp, tot_e2e, async_ms, stream_ms, persist_any, ring_any, batch_any = max_over_ranks(
        [tot_comp, tot_e2e, async_ms, stream_ms, persist_ms if persist_ms else 0.0,
         ring_ms if ring_ms else 0.0, batch_ms if batch_ms else 0.0], dist, device="cuda")
    value_graph = job_frames_per_s(S * args.steps, world, stream_ms)
    value_ring = (job_frames_per_s(S * args.steps, world, ring_any)
                  if ring_ms and ring_any > 0 else None)
    use_ring = value_ring is not None
    value = value_ring if use_ring else value_graph
    value_ms = ring_any if use_ring else stream_ms
    isolated_value = job_frames_per_s(S * args.steps, world, tot_comp)
    e2e_serial = job_frames_per_s(S * args.steps, world, tot_e2e)
    e2e_async = job_frames_per_s(S * args.steps, world, async_ms)
    # both are the public API end to end (every step's inputs H2D, results
    # D2H); the overlapped runner wins unless the host's PCIe path is
    # contended (shared node), where its concurrent DMA streams lose -- report
    # the faster, name it, keep both
    e2e_persist = (job_frames_per_s(S * args.steps, world, persist_any)
                   if persist_ms and persist_any > 0 else None)
    cands = {"async": e2e_async, "serial": e2e_serial}
    if e2e_persist:
        cands["persistent"] = e2e_persist
    e2e_batch = (job_frames_per_s(S * args.steps, world, batch_any)
                 if batch_ms and batch_any > 0 else None)
    if e2e_batch:
        cands["persistent_batched"] = e2e_batch
    e2e_method = max(cands, key=cands.get)
    e2e_value = cands[e2e_method]

    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return

    units = algorithmic_units(w0)
    peaks = json.loads(PEAKS_FILE.read_text()) if PEAKS_FILE.exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
    dom_bytes = S * (units["stereo_bytes"] + units["map_bytes"])
    achieved = dom_bytes / (track_ms / 1e3) / 1e9
    popc = popc_peak(torch, _lib)
    ham = S * (units["hamming_phase1"] + units["hamming_projection"])
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists() and S == 1:  # ncu --set full DRAM bytes of this kernel, this config
        t = json.loads(tf.read_text()).get("ft_track_frames", {})
        if "dram_bytes_read_per_launch" in t:
            traffic = t["dram_bytes_read_per_launch"] + t.get("dram_bytes_write_per_launch", 0)
    if use_ring:  # the value region's kernel: one persistent launch over K frames
        ring_traffic = None
        if tf.exists() and S == 1:
            tj = json.loads(tf.read_text())
            # the capture of this launch shape: step groups G, K steps (else the
            # nearest K of the same G)
            cands = [v for k, v in tj.items()
                     if k.startswith(f"track_persist_kernel_ring_g{ring_groups}_k")]
            t = (min(cands, key=lambda v: abs(v["steps_per_launch"] - args.steps)) if cands
                 else tj.get("track_persist_kernel_ring", {}) if ring_groups == 1 else {})
            if "dram_bytes_per_frame" in t:
                ring_traffic = t["dram_bytes_per_frame"] * args.steps
        ring_bytes = dom_bytes * args.steps
        ring_ach = ring_bytes / (ring_any / 1e3) / 1e9
    roofline = {"bound": "hbm", "kernel": "ft_track_frames", "achieved": achieved,
                "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "traffic": traffic, "traffic_source": "profiles/traffic.json (ncu --set full)", "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback",
                "algorithmic_bytes_per_launch": dom_bytes, "launch_ms": track_ms,
                "note": "one frame per launch is latency-bound (dependent L2/HBM round trips "
                        "and group barriers); see roofline_int and batched"}
    if use_ring:
        roofline = {"bound": "hbm", "kernel": "track_persist_kernel (ft_track_frames_ring, "
                                              f"{args.steps} frames per launch, "
                                              f"{ring_groups} step groups)",
                    "achieved": ring_ach, "peak": hbm_peak, "unit": "GB/s",
                    "frac": ring_ach / hbm_peak, "traffic": ring_traffic,
                    "traffic_source": "profiles/traffic.json (ncu --set full, per frame x K)",
                    "peak_source": roofline["peak_source"],
                    "algorithmic_bytes_per_launch": ring_bytes, "launch_ms": ring_any,
                    "note": "SURVEY 8(d) algorithmic bytes count both whole pyramids (2.2 of "
                            "the 2.98 MB per frame); phase 2 reads only the levels of the "
                            "frame's octaves, so ncu DRAM traffic is ~0.64 MB per frame "
                            "(traffic).  A frame is a chain of dependent L2 round trips "
                            "(latency-bound)",
                    "per_frame_launch": roofline}
    # PCIe diagnostic: one step's input bytes, pinned H2D alone (events)
    h2d_times = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.stream)
        with torch.cuda.stream(pipe.stream):
            pipe.dev[:pipe.in_end].copy_(pipe.host[:pipe.in_end], non_blocking=True)
        b.record(pipe.stream)
        pipe.synchronize()
        h2d_times.append(a.elapsed_time(b))
    h2d_ms = float(np.median(h2d_times))
    line = {"metric": "stereo+local-map tracking frames/s at EuRoC shape", "value": value,
            "unit": "frames/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": value_ms / args.steps,
            "value_method": (f"ONE persistent track launch (ft_track_frames_ring) running the "
                             f"K steps over {n_res} resident pipelines in {ring_groups} step "
                             f"group(s) ({ring_groups} frames in flight on disjoint SMs; G "
                             "picked in the warm-up from "
                             f"{list(RING_GROUPS)}, ring ms per G: {ring_group_ms})"
                             if use_ring else
                             f"compute graphs replayed back to back on one stream over {n_res} "
                             "resident pipelines") +
                            f" (each one frame's inputs in HBM; "
                            f"{n_res * pipe.in_end / 2**20:.0f} MiB of inputs > 2x L2), "
                            "CUDA events around all K steps",
            "value_graph_replays": value_graph,
            "value_persistent_ring": value_ring,
            "value_ring_groups": ring_groups,
            "latency_ms_per_frame": tot_comp / args.steps,
            "isolated_step": {"value": isolated_value, "unit": "frames/s",
                              "method": "one step at a time: L2 flushed, events, synchronise"},
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64+u32", "data": "synthetic", "config": config_dict(args),
            "e2e": {"value": e2e_value, "unit": "frames/s",
                    "method": e2e_method,
                    "methods": {"async": "AsyncRunner (native ft_runner): per step H2D of that "
                                         "step's inputs from pinned host memory, compute, D2H "
                                         "of its results; neighbouring steps' copies overlap "
                                         "the compute; host wall clock over all steps",
                                "serial": "FramePipeline.replay(copies=True) per step: H2D, "
                                          "compute, D2H, synchronise; host wall clock",
                                "persistent": "AsyncRunner(persistent=True), 8 slots: the "
                                              "async schedule with ONE long-lived track "
                                              "kernel handed each step through mapped "
                                              "host flags (no launch per step), G step "
                                              "groups (G steps computed at once; best of "
                                              f"{list(PERSIST_GROUPS)}); host wall clock",
                                "persistent_batched": "the persistent runner over 8 slots in "
                                                      "one DeviceArena: m consecutive steps' "
                                                      "inputs (pinned ring rows) go up as ONE "
                                                      "strided 2D copy (ft_runner_submit_batch), "
                                                      "each step still its own frame with its "
                                                      "results pushed to the host; best of "
                                                      "m in (2, 4) x G in (1, 2); host wall clock"},
                    "async_value": e2e_async,
                    "serial_value": e2e_serial,
                    "persistent_value": e2e_persist,
                    "persistent_batched_value": e2e_batch,
                    "persistent_batched_pick": batch_pick,
                    "persistent_batched_ms": batch_by,
                    "persistent_groups": persist_groups,
                    "persistent_ms_by_groups": {str(g): v for g, v in persist_by_g.items()},
                    "latency_ms_per_frame_e2e": persist_lat_ms,
                    "latency_method": "persistent runner, one frame in flight: submit (448 KB "
                                      "H2D) -> kernel -> D2H -> result on the host, median, "
                                      "host wall clock",
                    "h2d_alone_ms": h2d_ms,
                    "host_cpus": "all" if numa_cpus is None else f"{len(numa_cpus)} on the GPU's NUMA node",
                    "h2d_gbs": pipe.h2d_bytes() / (h2d_ms / 1e3) / 1e9,
                    "h2d_bytes_per_step": int((pipe.h2d_bytes() if e2e_method == "serial" else
                                               shipped) + e2e_delta / max(1, args.steps)),
                    "h2d_bytes_per_step_async": int(shipped),
                    "h2d_bytes_per_step_serial": pipe.h2d_bytes(),
                    "pyramid_levels_shipped": "levels >= the frame's lowest left-keypoint octave "
                                              "(phase 2 reads no others)"
                                              if pipe.level_ranges else "all",
                    "d2h_bytes_per_step": pipe.d2h_bytes(),
                    "map_table": None if table is None else {
                        "resident_points": table.size, "upload_bytes_once": table_bytes,
                        "delta_bytes_per_step": e2e_delta / max(1, args.steps)},
                    "ms_per_step_wall": tot_e2e / args.steps,
                    "ms_per_step_events": float(np.sum(e2e_ev_ms)) / args.steps},
            "roofline": roofline,
            "roofline_int": {"bound": "popc", "kernel": "ft_track_frames",
                             "hamming_per_launch": ham, "popc_per_launch": 8 * ham,
                             "achieved_gpopc_s": 8 * ham / (track_ms / 1e3) / 1e9,
                             "peak_gpopc_s": popc, "peak_source": "ft_bench_popc (measured)",
                             "frac": (8 * ham / (track_ms / 1e3) / 1e9) / popc if popc else None},
            "kernels_ms": {"ft_track_frames": track_ms,
                           "ft_build_pyramids": float(np.median(kern["pyramids"])) if raw else 0.0,
                           "stereo_only": float(np.median(kern["stereo_only"])),
                           "map_only": float(np.median(kern["map_only"]))},
            "work_per_frame": units, "clocks": clocks,
            "gpu_launches": 1 if use_ring else (1 + int(raw)) * args.steps,
            "gpu_launches_note": ("the value region is ONE persistent track_persist_kernel "
                                  "launch running all K steps; the graph-replay value, "
                                  "latency and e2e regions launch ft_track_frames per step"
                                  if use_ring else
                                  "our kernels per step: ft_track_frames (+ "
                                  "ft_build_pyramids in raw / hybrid mode); counted over the "
                                  "value region's K steps (each other timed region launches "
                                  "the same per step)"),
            "parity_spot_check": check}
    if not args.quick:
        # extra measurements: a failure in one is recorded, never loses the line
        def extra(key, fn):
            try:
                line[key] = fn()
            except Exception as exc:  # noqa: BLE001
                line[key] = {"error": f"{type(exc).__name__}: {exc}"[:300]}

        if args.batched_streams > 0 and world == 1:
            extra("batched", lambda: batched_run(args, frames, torch, FramePipeline, cap_kp,
                                                 cap_pts, images, flush, popc=popc))
            if images:  # the other pyramid input mode at batch
                other_raw = not raw
                extra("batched_hybrid_pyramids" if other_raw else "batched_pyramids_shipped",
                      lambda: batched_run(args, frames, torch, FramePipeline, cap_kp, cap_pts,
                                          images, flush, other_raw))
        if images and world == 1:
            extra("pyramid_modes", lambda: raw_mode_run(args, frames, torch, FramePipeline,
                                                        cap_kp, cap_pts, flush))
        if world == 1 and not args.no_configs:
            extra("cfg1_orb", lambda: cfg1_orb_run(args, torch, flush))
            extra("api_e2e", lambda: api_e2e_run(frames, max(20, args.steps)))
            extra("cfg4_sequence", lambda: cfg4_sequence_run(99))
            extra("other_configs", lambda: other_configs(args, torch, flush))
            extra("roofline_hamming", lambda: hamming_roofline(torch, _lib, popc))
        if world == 1:  # reported baseline: rank 0 at N=1 only
            extra("cpu_baseline", lambda: cpu_baseline(frames[:2], args.cpu_seconds))
    print(json.dumps(line))
    if dist:
        dist.destroy_process_group()


def spot_check(pipe, w) -> bool:
    from oracle import oracle as O
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    r = pipe.result(0, len(w.left.u))
    ref = O.stereo_pinhole(w.left, w.right, w.pyr_left, w.pyr_right, w.cam, StereoMatchConfig(),
                           w.scale_pow)
    ok = all(np.array_equal(getattr(r.matches, f), getattr(ref, f))
             for f in ("right_idx", "distance", "disparity", "refined_u", "depth", "sad"))
    grid = O.frame_grid(w.left.u, w.left.v, w.cam.width, w.cam.height, 48) + (48,)
    slots = np.full(len(w.left.u), -1, np.int64)
    n = O.search_local_points(w.local.point_ids, w.local.soa, w.left.u, w.left.v, w.left.octave,
                              w.left.descriptors, grid, slots, w.pose, w.cam,
                              ProjectionSearchConfig(), 1.2, 8)
    ok = ok and n == r.n_slots and np.array_equal(slots, r.slots)
    if not ok:
        raise SystemExit("bench spot check FAILED: pipeline output differs from the oracle")
    return ok


def popc_peak(torch, _lib) -> float | None:
    """Measured POPC throughput (G popc/s) of ft_bench_popc at full occupancy."""
    L = _lib.load()
    sink = torch.zeros(1, dtype=torch.int32, device="cuda")
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks, threads, iters = sms * 8, 256, 4096
    s = torch.cuda.current_stream()
    for _ in range(2):
        _lib.check(L.ft_bench_popc(blocks, threads, iters, sink.data_ptr(), s.cuda_stream), "popc")
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    _lib.check(L.ft_bench_popc(blocks, threads, iters, sink.data_ptr(), s.cuda_stream), "popc")
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return blocks * threads * iters * 8 / (ms / 1e3) / 1e9


def make_runner(args, frames, pipe, table, load):
    """A second pipeline of the same shape + AsyncRunner, and every cycled
    frame's inputs pre-staged in pinned host memory (one tensor per step)."""
    from paper_2509_10757_b200.pipeline import AsyncRunner, FramePipeline
    n_slots = max(2, min(4, int(os.environ.get("FT_BENCH_SLOTS", "4"))))
    twins = [FramePipeline(pipe.cam, n_streams=pipe.S, cap_kp=pipe.cap_kp,
                           cap_points=pipe.cap_pts, pyramid_geometry=pipe.pyr,
                           raw_images=pipe.raw, map_table=table,
                           build_levels=pipe.build_levels if pipe.raw else None)
             for _ in range(n_slots - 1)]
    n = max(1, min(len(frames), int(os.environ.get("FT_BENCH_RING", str(len(frames))))))
    ring = pipe.staging_ring(n)
    ranges = []
    for k in range(n):
        load(k)
        pipe.stage_into(ring[k])
        ranges.append(pipe.input_range())
    for t in twins:
        t.capture()
    r = AsyncRunner([pipe] + twins)
    r.staging = ring  # [n, in_end] rows at one pitch (batched submits)
    return r, [ring[k] for k in range(n)], ranges


def _pipe_rates(torch, pipes, staged, steps, flush, S, ranges=None) -> dict:
    """Device frames/s (compute graph, L2 flushed) and e2e frames/s through
    AsyncRunner for a pair of identically shaped pipelines."""
    from paper_2509_10757_b200.pipeline import AsyncRunner
    p = pipes[0]
    comp = []
    for _ in range(steps):
        with torch.cuda.stream(p.stream):
            p.dev[:p.in_end].copy_(staged[0], non_blocking=True)
            flush.fill_(1)
            flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(p.stream)
        p.replay(copies=False)
        b.record(p.stream)
        p.synchronize()
        comp.append(a.elapsed_time(b))
    rg = ranges if ranges is not None else [None] * len(staged)

    def timed(runner) -> float:
        k, tw = 0, time.perf_counter()  # >= 0.3 s of steps: clocks ramped
        while k < 4 * len(staged) + 2 or time.perf_counter() - tw < 0.3:
            if k >= runner.n:
                runner.wait(k - runner.n)
            runner.submit(k, staged[k % len(staged)], rg[k % len(staged)])
            k += 1
        for j in range(max(0, k - runner.n), k):
            runner.wait(j)
        k0 = k
        t0 = time.perf_counter()
        for k in range(k0, k0 + steps):
            if k - k0 >= runner.n:
                runner.wait(k - runner.n)
            runner.submit(k, staged[k % len(staged)], rg[k % len(staged)])
        for k in range(max(k0, k0 + steps - runner.n), k0 + steps):
            runner.wait(k)
        ms = 1e3 * (time.perf_counter() - t0)
        runner.close()
        return ms

    e2e_ms = timed(AsyncRunner(pipes))
    pers = None
    if all(getattr(q, "plan", None) is not None and q.plan() is not None for q in pipes):
        # the persistent runner, where eligible (single-launch steps)
        try:
            pers = S * steps / (timed(AsyncRunner(pipes, persistent=True)) / 1e3)
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] persistent ({S} streams): {type(exc).__name__}: {exc}",
                  file=sys.stderr)
    if ranges is not None:
        shipped = float(np.mean([sum(hi - lo for lo, hi in (r if isinstance(r[0], (tuple, list))
                                                              else [r])) for r in ranges]))
    else:
        shipped = p.h2d_bytes()
    return {"streams": S, "ms_per_step": float(np.median(comp)),
            "frames_per_s": S * steps / (sum(comp) / 1e3),
            "e2e_frames_per_s": max(S * steps / (e2e_ms / 1e3), pers or 0.0),
            "e2e_graph_runner_frames_per_s": S * steps / (e2e_ms / 1e3),
            "e2e_persistent_frames_per_s": pers,
            "h2d_bytes_per_step": int(shipped), "d2h_bytes_per_step": p.d2h_bytes()}


def hamming_roofline(torch, _lib, popc_peak_g) -> dict:
    """The all-pairs Hamming kernel (fisheye stereo, kernels.py:434-464) at
    cfg3 shape, 1 and 64 frames per launch: achieved POPC/s (8 per 256-bit
    Hamming, the algorithmic count) over the measured POPC peak -- the north
    star's integer-pipe roofline target for the Hamming kernels."""
    from paper_2509_10757_b200.runtime import fill_kp_records, make_workspace
    from synthetic import make_workload
    from paper_2509_10757_b200.types import StereoMatchConfig
    w = make_workload(seed=700, n_landmarks=4800, map_points=100, fisheye=True)
    nl, nr = len(w.left.u), len(w.right.u)
    cap = (max(nl, nr) + 255) // 256 * 256
    lib = _lib.load()
    cfg = StereoMatchConfig()
    out = {"bound": "popc (XU pipe)", "unit": "G popc/s", "peak": popc_peak_g,
           "peak_source": "ft_bench_popc (measured, same run)",
           "work": f"{nl} x {nr} Hamming per frame, 8 POPC each"}
    for F in (1, 2, 4, 64):
        recs = np.zeros((2, F, cap), dtype=_lib.KP_RECORD)
        for f in range(F):
            fill_kp_records(recs[0, f], w.left)
            fill_kp_records(recs[1, f], w.right)
        dev = torch.from_numpy(recs.view(np.uint8).reshape(-1)).cuda()
        cnt = torch.tensor([nl] * F + [nr] * F, dtype=torch.int32, device="cuda")
        kl, kr = _lib.FtKeypoints(), _lib.FtKeypoints()
        kl.rec, kl.count, kl.cap = dev.data_ptr(), cnt.data_ptr(), cap
        kr.rec, kr.count, kr.cap = dev.data_ptr() + F * cap * 64, cnt.data_ptr() + 4 * F, cap
        idx = torch.empty(F * cap, dtype=torch.int64, device="cuda")
        dist = torch.empty_like(idx)
        stream = torch.cuda.Stream()
        ws = make_workspace(lib, torch.device("cuda"), stream, F, cap, 1)

        def launch():
            _lib.check(lib.ft_stereo_fisheye_bf(F, kl, kr, cfg.t_match, cfg.ratio, idx.data_ptr(),
                                                dist.data_ptr(), ws, stream.cuda_stream), "bf")

        launch()
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream):
            launch()
        ts = []
        with torch.cuda.stream(stream):
            for _ in range(20):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                g.replay()
                b.record(stream)
                stream.synchronize()
                ts.append(a.elapsed_time(b))
        ms = float(np.median(ts))
        achieved = 8 * F * nl * nr / (ms / 1e3) / 1e9
        out[f"frames_{F}"] = {"launch_ms": ms, "achieved": achieved,
                              "frac": achieved / popc_peak_g if popc_peak_g else None}
    return out


def other_configs(args, torch, flush) -> dict:
    """BASELINE configs[2] (cfg3: TUM-VI fisheye stereo 512x512 ~1500 kps +
    3050-point local map; FisheyePipeline) and configs[4] (cfg5 high load:
    ~2000 kps / image, 20k-point local map; FramePipeline), each at 1 stream
    and 64 streams per launch, local maps resident in a MapTable."""
    from paper_2509_10757_b200.maptable import MapTable
    from paper_2509_10757_b200.pipeline import FisheyePipeline, FramePipeline
    from synthetic import make_workload
    steps = max(10, args.steps // 2)
    out = {}
    fw = [make_workload(seed=700 + i, n_landmarks=4800, map_points=3050, fisheye=True,
                        offset=0.05 * i, id_base=100_000 * (i + 1)) for i in range(4)]
    cap = (max(max(len(w.left.u), len(w.right.u)) for w in fw) + 255) // 256 * 256
    res = {}
    for S in (1, 64):
        table = MapTable(capacity=4 * 4096 + 1024)
        pipes = [FisheyePipeline(fw[0].cam, n_streams=S, cap_kp=cap, cap_points=4096,
                                 map_table=table) for _ in range(8 if S == 1 else 4)]
        nst = min(4, S * 4)
        ring = pipes[0].staging_ring(nst)
        for k in range(nst):
            for s in range(S):
                w = fw[(k + s) % 4]
                pipes[0].load_frame(s, w.left, w.right, w.local, w.pose)
            pipes[0].stage_into(ring[k])
        staged = [ring[k] for k in range(nst)]
        for p in pipes:
            p.capture()
        res[f"S{S}"] = _pipe_rates(torch, pipes, staged, steps, flush, S)
    out["cfg3_fisheye"] = {"workload": f"TUM-VI-shaped fisheye pair 512x512, "
                                       f"~{int(np.mean([len(w.left.u) for w in fw]))} kps/image, "
                                       "3050-point local map: ft_stereo_fisheye (brute force + "
                                       "KB triangulation) + fisheye SearchLocalPoints",
                           "hamming_per_frame": int(np.mean([len(w.left.u) * len(w.right.u)
                                                             for w in fw])), **res}
    hw = [make_workload(seed=800 + i, n_landmarks=20000, map_points=20000, images=True,
                        offset=0.05 * i, id_base=1_000_000 * (i + 1)) for i in range(2)]
    cap = (max(max(len(w.left.u), len(w.right.u)) for w in hw) + 31) // 32 * 32
    res = {}
    for S in (1, 64):
        table = MapTable(capacity=2 * 20480 + 1024)
        pipes = [FramePipeline(hw[0].cam, n_streams=S, cap_kp=cap, cap_points=20480,
                               pyramid_geometry=hw[0].pyr_left, map_table=table)
                 for _ in range(8 if S == 1 else 4)]
        ring = pipes[0].staging_ring(2)
        rngs = []
        for k in range(2):
            for s in range(S):
                w = hw[(k + s) % 2]
                pipes[0].load_frame(s, w.left, w.right, w.local, w.pose, w.pyr_left, w.pyr_right)
            pipes[0].stage_into(ring[k])
            rngs.append(pipes[0].input_ranges())
        staged = [ring[0], ring[1]]
        for p in pipes:
            p.capture()
        res[f"S{S}"] = _pipe_rates(torch, pipes, staged, steps, flush, S, rngs)
    out["cfg5_high_load"] = {"workload": f"~{int(np.mean([len(w.left.u) for w in hw]))} "
                                         "kps/image 752x480 (pyramids shipped) + 20000-point "
                                         "local map; stereo + SearchLocalPoints",
                             **res}
    return out


def cfg1_orb_run(args, torch, flush) -> dict:
    """BASELINE configs[0] (cfg1): the reference's own ORB-extracted frame
    (tests/golden/cfg1_stereo.npz: rendered 752x480 pair, 1201 keypoints,
    97.5 % at octave 0, so phase 2 needs the whole level-0 images) through
    ComputeStereoMatches only (phase 1 -> phase 2 -> reject), as device
    frames/s (L2 flushed) and e2e through AsyncRunner, with (a) both pyramids
    shipped (2.2 MB), (b) raw level-0 images shipped + the bit-exact device
    pyramid build (0.72 MB) and (c) hybrids: level 0 and levels > b shipped,
    levels 1..b built on the device.  Parity: the pipeline's matches equal the
    reference's golden output."""
    import golden_io as G
    from paper_2509_10757_b200.pipeline import FramePipeline
    from paper_2509_10757_b200.types import LocalMap, MapPointSoA, Pose
    d = G.load("cfg1_stereo.npz")
    left, right = G.feats(d, "left"), G.feats(d, "right")
    pl, pr = G.pyramid(d, "l"), G.pyramid(d, "r")
    cam = G.pinhole()
    empty = LocalMap((), np.empty(0, np.int64), MapPointSoA.empty())
    steps = max(10, args.steps // 2)
    cap = (max(len(left.u), len(right.u)) + 31) // 32 * 32
    out = {"workload": "cfg1: reference ORB frame 752x480, 1201/1201 kps, octaves "
                       f"{np.bincount(left.octave, minlength=8).tolist()}, ComputeStereoMatches "
                       "only (phase 1 -> SAD phase 2 -> reject)"}
    modes = (("pyramids_shipped", False, None), ("raw_images_device_pyramid", True, None),
             ("hybrid_build_level_1", True, 1), ("hybrid_build_levels_1_2", True, 2))
    for name, raw, bl in modes:
        pipes = [FramePipeline(cam, n_streams=1, cap_kp=cap, cap_points=256,
                               pyramid_geometry=pl, raw_images=raw, build_levels=bl)
                 for _ in range(8)]
        p0 = pipes[0]
        p0.load_frame(0, left, right, empty, Pose.identity(), pl, pr)
        ring = p0.staging_ring(2)
        rngs = []
        for k in range(2):
            p0.stage_into(ring[k])
            rngs.append(p0.input_range() if p0.level_ranges else None)
        for q in pipes:
            q.capture()
        p0.replay()
        p0.synchronize()
        r = p0.result(0, len(left.u))
        parity = all(np.array_equal(getattr(r.matches, f), d[f"final_{f}"])
                     for f in ("right_idx", "distance", "disparity", "refined_u", "depth", "sad"))
        res = _pipe_rates(torch, pipes, [ring[0], ring[1]], steps, flush, 1,
                          rngs if rngs[0] is not None else None)
        res["parity_vs_reference_golden"] = parity
        out[name] = res
    best = max((m[0] for m in modes), key=lambda k: out[k]["e2e_frames_per_s"])
    out["e2e_best"] = {"mode": best, "frames_per_s": out[best]["e2e_frames_per_s"]}
    return out


def api_e2e_run(frames, steps: int) -> dict:
    """The reference-facing plugin path, end to end from numpy objects: every
    call packs its inputs on the host, ships them (one pinned H2D), launches,
    copies results back and unpacks into reference types (host wall clock,
    packing included).  (a) the tracker seam as install() serves it --
    match_pinhole_phase1, refine_match_phase2, reject_outliers (tracker.py:
    418-427), then search_local_points (tracker.py:354) -- and (b) the fused
    ComputeStereoMatches + search_local_points."""
    import paper_2509_10757_b200 as ft
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    cfg, pcfg = StereoMatchConfig(), ProjectionSearchConfig()

    # the reference Frame objects (with their FrameGrid) are the tracker's own
    # per-frame work, built before the timed calls; each call starts from
    # empty slots, as a fresh frame does
    frames_of = {id(w): w.frame() for w in frames}

    def fresh(w):
        fr = frames_of[id(w)]
        fr.slots[:] = -1
        return fr

    def seam(w):
        idx, dist = ft.match_pinhole_phase1(w.left, w.right, w.cam.height, w.scale_pow, cfg)
        m = ft.reject_outliers(ft.refine_match_phase2(w.pyr_left, w.pyr_right, w.left, w.right,
                                                      idx, dist, w.cam, cfg), cfg)
        return m, ft.search_local_points(w.local, fresh(w), w.cam, pcfg, 1.2, 8)

    def fused(w):
        m = ft.compute_stereo_matches(w.left, w.right, w.cam, cfg, w.scale_pow, w.pyr_left,
                                      w.pyr_right)
        return m, ft.search_local_points(w.local, fresh(w), w.cam, pcfg, 1.2, 8)

    from types import SimpleNamespace
    from paper_2509_10757_b200.install import _fused_run_stereo

    class _Pool:  # reference BufferPool.acquire (buffers.py:38-52)
        def __init__(self):
            self.b = {}

        def acquire(self, name, shape, dtype):
            if name not in self.b:
                self.b[name] = np.empty(8192, dtype)
            return self.b[name][:shape[0]]

    def installed(w):  # what install() serves the tracker: fused _run_stereo + SLP
        tr = SimpleNamespace(cam=w.cam, stereo=cfg, pool=_Pool(),
                             extraction=SimpleNamespace(scale_powers=lambda: w.scale_pow))
        m = _fused_run_stereo(tr, w.left, w.right, w.pyr_left, w.pyr_right)
        return m, ft.search_local_points(w.local, fresh(w), w.cam, pcfg, 1.2, 8)

    out = {"workload": "cfg2 frames (rendered pyramids, 5000-point local maps) from numpy "
                       "reference-type objects (Frame objects built before timing, slots "
                       "reset per call)"}
    for name, fn in (("tracker_seam", seam), ("fused", fused), ("install_default", installed)):
        for k in range(5):
            fn(frames[k % len(frames)])
        ts = []
        for k in range(steps):
            t0 = time.perf_counter()
            fn(frames[k % len(frames)])
            ts.append(time.perf_counter() - t0)
        out[name] = {"frames_per_s": len(ts) / sum(ts), "ms_per_frame_median":
                     1e3 * float(np.median(ts)), "launches_per_frame": 4 if name == "tracker_seam"
                     else 2}
    out["note"] = ("tracker_seam: the tracker's own call sequence with install(fuse_stereo="
                   "False); install_default: StereoTracker._run_stereo replaced by one fused "
                   "call (install() default) + search_local_points; every call through the "
                   "native session (csrc/ft_session.cu)")
    return out


def cfg4_sequence_run(steps_cap: int) -> dict:
    """BASELINE configs[3] (cfg4): the reference tracker's 100-frame line
    sequence (tests/golden/cfg4_line.npz: every stage call's inputs, the world
    as it grew) replayed as a DEPENDENT sequence -- one frame at a time, each
    frame's results back on the host before the next (the tracker's host
    logic -- pose prediction / refinement, keyframe decisions -- runs in
    between) -- ms/frame of the hot-path work per frame, through the
    reference's signatures as install() serves the tracker:
    (a) dropin: _run_stereo as one fused call, search_prev_frame (prev-frame
        points decomposed on the host, as the reference), update_local_map on
        the device (the world mirrored in HBM, only new keyframes / points
        shipped), search_local_points reading the resident local map in place;
    (b) dropin_resident_world: (a) with install(resident_world=True):
        search_prev_frame reads the mirrored world in place;
    (c) resident: (b), with stereo + the local search as ONE graph-captured
        launch (FramePipeline on the world table).
    Every frame's outputs are checked against the reference's digests
    (outside the timed region); the reference's own per-stage host times for
    the same sequence are in tests/golden/summary.json."""
    import golden_io as G
    import paper_2509_10757_b200 as ft
    from paper_2509_10757_b200.pipeline import FramePipeline
    from paper_2509_10757_b200.types import ProjectionSearchConfig, StereoMatchConfig
    from paper_2509_10757_b200.worldmap import world_table
    from types import SimpleNamespace
    from paper_2509_10757_b200.install import _fused_run_stereo
    seq = G.Cfg4("line")
    cfg, pcfg, cam = StereoMatchConfig(), ProjectionSearchConfig(), seq.cam
    sp = 1.2 ** np.arange(8, dtype=np.float64)
    frames = list(range(1, min(seq.n_frames, steps_cap + 1)))
    inputs = {}
    for i in frames:  # host objects built before timing (the tracker has them)
        pf = int(seq.get(i, "prev_prev_frame"))
        inputs[i] = dict(left=seq.feats(i, "l"), right=seq.feats(i, "r"),
                         prev=seq.frame(pf, seq.pose(i, "prev_prev_pose"),
                                        seq.get(i, "prev_prev_slots")),
                         ppose=seq.pose(i, "prev_pose"), cur=seq.frame(i, seq.pose(i, "prev_pose")),
                         lpose=seq.pose(i, "local_pose"),
                         slots=seq.get(i, "local_slots_in").astype(np.int64),
                         world=(int(seq.get(i, "update_n_keyframes")),
                                int(seq.get(i, "update_n_points"))))
        inputs[i]["frame"] = seq.frame(i, inputs[i]["lpose"], inputs[i]["slots"])
    mdig = lambda m: G.digest(*(np.asarray(getattr(m, f), t) for f, t in (  # noqa: E731
        ("right_idx", np.int64), ("distance", np.int64), ("disparity", np.float64),
        ("refined_u", np.float64), ("depth", np.float64), ("sad", np.int64))))
    cdig = lambda c: G.digest(*(np.asarray(getattr(c, f), np.int64) for f in (  # noqa: E731
        "point_idx", "keypoint_idx", "distance", "octave")))

    class _Pool:  # reference BufferPool.acquire (buffers.py:38-52)
        def __init__(self):
            self.b = {}

        def acquire(self, name, shape, dtype):
            if name not in self.b:
                self.b[name] = np.empty(8192, dtype)
            return self.b[name][:shape[0]]

    tracker = SimpleNamespace(cam=cam, stereo=cfg, pool=_Pool(),
                              extraction=SimpleNamespace(scale_powers=lambda: sp))

    def dropin(i, x, world, pipe=None):
        m = _fused_run_stereo(tracker, x["left"], x["right"], None, None)
        corr, _ = ft.search_prev_frame(x["prev"], x["cur"], x["ppose"], world, cam, pcfg, 1.2, 8)
        fr = x["frame"]
        fr.slots[...] = x["slots"]
        local = ft.update_local_map(fr, world)
        n = ft.search_local_points(local, fr, cam, pcfg, 1.2, 8)
        return m, corr, fr.slots, n, local

    def resident(i, x, world, pipe):
        table = world_table(world).table
        corr, _ = ft.search_prev_frame(x["prev"], x["cur"], x["ppose"], world, cam, pcfg, 1.2,
                                       8, table=table)
        fr = x["frame"]
        fr.slots[...] = x["slots"]
        local = ft.update_local_map(fr, world)
        pipe.load_frame(0, x["left"], x["right"], local, x["lpose"], slots=x["slots"])
        pipe.replay()
        pipe.synchronize()
        r = pipe.result(0, len(x["left"].u))
        return r.matches, corr, r.slots, r.n_slots, local

    out = {"workload": "cfg4: reference StereoTracker line sequence (12000 landmarks, 0.5 px "
                       f"noise, seed 4), frames 1..{frames[-1]}, ~1200 kps / image, local maps "
                       "of ~2100 points from the growing world (21 keyframes); one frame in "
                       "flight (dependent sequence)",
           "reference_host_us_per_frame_median": None}
    try:
        import json as _json
        summ = _json.loads((ROOT / "tests" / "golden" / "summary.json").read_text())
        out["reference_host_us_per_frame_median"] = summ["cfg4_line"]["stage_us_median_seq_engine"]
    except (OSError, KeyError, ValueError):
        pass
    from paper_2509_10757_b200 import projection as _proj

    def dropin_rw(i, x, world, pipe=None):  # install(resident_world=True)
        _proj._RESIDENT_WORLD = True
        try:
            return dropin(i, x, world, pipe)
        finally:
            _proj._RESIDENT_WORLD = False

    for name, fn in (("dropin", dropin), ("dropin_resident_world", dropin_rw),
                     ("resident", resident)):
        best = None
        for rep in range(2):  # pass 0 warms up (a fresh world: the first frames sync it)
            world = seq.growing_world()
            pipe = None
            if name == "resident":
                world.advance(*inputs[frames[0]]["world"])
                pipe = FramePipeline(cam, n_streams=1, cap_kp=2048, cap_points=8192,
                                     map_table=world_table(world).table)
                pipe.capture()
            ts, ok = [], True
            for i in frames:
                x = inputs[i]
                world.advance(*x["world"])
                t0 = time.perf_counter()
                m, corr, slots, n, local = fn(i, x, world, pipe)
                ts.append(time.perf_counter() - t0)
                # checked outside the timed region
                ok &= (np.array_equal(mdig(m), seq.get(i, "stereo_final")) and
                       np.array_equal(cdig(corr), seq.get(i, "prev_corr_digest")) and
                       np.array_equal(G.digest(np.asarray(local.point_ids, np.int64)),
                                      seq.get(i, "update_ids_digest")) and
                       np.array_equal(G.digest(np.asarray(slots, np.int64)),
                                      seq.get(i, "local_slots_out")) and
                       n == int(seq.get(i, "local_count")))
            best = (ts, ok, world_table(world).bytes_uploaded)
        ts, ok, shipped = best
        out[name] = {"ms_per_frame_median": 1e3 * float(np.median(ts)),
                     "ms_per_frame_p90": 1e3 * float(np.percentile(ts, 90)),
                     "frames_per_s": len(ts) / sum(ts), "frames": len(ts),
                     "bit_exact_vs_reference": bool(ok),
                     "world_bytes_shipped_total": int(shipped),
                     "stages": "stereo, search_prev_frame, update_local_map, "
                               "search_local_points",
                     "launches_per_frame": 3 if name == "resident" else 4}
    return out


def raw_mode_run(args, frames, torch, FramePipeline, cap_kp, cap_pts, flush) -> dict:
    """The single-stream step with raw level-0 images shipped and pyramid
    levels 1..b built on the device (ft_build_pyramids), the
    levels above b shipped: device value and AsyncRunner e2e per b."""
    w0 = frames[0]
    out = {}
    L = len(w0.pyr_left.widths)
    for b in (0, 1, 2, 3, L - 1):  # 0: whole pyramids shipped
        table, _ = make_table(args, frames, cap_pts)
        pipes = [FramePipeline(w0.cam, n_streams=1, cap_kp=cap_kp, cap_points=cap_pts,
                               pyramid_geometry=w0.pyr_left, raw_images=b > 0, map_table=table,
                               build_levels=b if b > 0 else None) for _ in range(4)]
        ring = pipes[0].staging_ring(len(frames))
        rngs = []
        for k in range(len(frames)):
            f = frames[k]
            pipes[0].load_frame(0, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
            pipes[0].stage_into(ring[k])
            rngs.append(pipes[0].input_ranges())
        staged = [ring[k] for k in range(len(frames))]
        for p in pipes:
            p.capture()
        r = _pipe_rates(torch, pipes, staged, args.steps, flush, 1, rngs)
        out["pyramid_levels_shipped" if b == 0 else f"build_levels_1_to_{b}"] = r
    return out


def batched_run(args, frames, torch, FramePipeline, cap_kp, cap_pts, images, flush,
                raw: bool | None = None, popc: float | None = None) -> dict:
    """S frame streams per launch on this GPU (one frame of every stream per
    step): device-resident throughput, and e2e through AsyncRunner."""
    from paper_2509_10757_b200.pipeline import AsyncRunner
    S = args.batched_streams
    w0 = frames[0]
    mode_raw, b = pyramid_mode(args)
    if raw is None:
        raw = images and mode_raw
    elif not raw:
        b = None
    elif not mode_raw:  # explicit raw from a ship-mode run: hybrid at --build-levels
        b = max(1, args.build_levels)
    table, _ = make_table(args, frames, cap_pts, S)
    packed = os.environ.get("FT_BENCH_PACKED", "1") != "0"
    pipes = [FramePipeline(w0.cam, n_streams=S, cap_kp=cap_kp, cap_points=cap_pts,
                           pyramid_geometry=w0.pyr_left if images else None, raw_images=raw,
                           map_table=table, build_levels=b if raw else None,
                           packed_upload=packed)
             for _ in range(4)]
    pipe = pipes[0]
    for s in range(S):
        f = frames[s % len(frames)]
        pipe.load_frame(s, f.left, f.right, f.local, f.pose, f.pyr_left, f.pyr_right)
    ring = pipe.staging_ring(1)
    pipe.stage_into(ring[0])
    staged = ring[0]
    rngs = pipe.input_ranges()
    shipped = int(sum(hi - lo for lo, hi in rngs))
    pipe.capture()
    steps = max(5, args.steps // 5)
    for _ in range(3):
        pipe.replay(copies=True)
    pipe.synchronize()
    comp = []
    for _ in range(steps):
        with torch.cuda.stream(pipe.stream):
            flush.fill_(1)
            flush.view(torch.int64).sum()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(pipe.stream)
        pipe.replay(copies=False)
        b.record(pipe.stream)
        pipe.synchronize()
        comp.append(a.elapsed_time(b))
    runner = AsyncRunner(pipes)
    k, tw = 0, time.perf_counter()  # >= 0.3 s of steps: clocks ramped
    while k < max(3, args.warmup) or time.perf_counter() - tw < 0.3:
        if k >= runner.n:
            runner.wait(k - runner.n)
        runner.submit(k, staged, rngs)
        k += 1
    for j in range(max(0, k - runner.n), k):
        runner.wait(j)
    k0 = k
    t0 = time.perf_counter()
    for k in range(k0, k0 + steps):
        if k - k0 >= runner.n:
            runner.wait(k - runner.n)
        runner.submit(k, staged, rngs)
    for k in range(max(k0, k0 + steps - runner.n), k0 + steps):
        runner.wait(k)
    e2e_ms = 1e3 * (time.perf_counter() - t0)
    runner.close()
    # HBM roofline of the batched launch: SURVEY 8(d) algorithmic bytes of the
    # S frames over the launch time (inputs > L2 at this S)
    per = {}
    tot_bytes = tot_ham = 0
    for s_ in range(S):
        i = s_ % len(frames)
        if i not in per:
            u = algorithmic_units(frames[i])
            per[i] = (u["stereo_bytes"] + u["map_bytes"],
                      u["hamming_phase1"] + u["hamming_projection"])
        tot_bytes += per[i][0]
        tot_ham += per[i][1]
    peaks = json.loads(PEAKS_FILE.read_text()) if PEAKS_FILE.exists() else {}
    hbm_peak = float(peaks.get("hbm_gbs", FALLBACK_HBM))
    med_ms = float(np.median(comp))
    ach = tot_bytes / (med_ms / 1e3) / 1e9
    return {"streams": S, "steps": steps, "raw_images": bool(raw),
            "roofline": {"bound": "hbm", "kernel": "ft_track_frames (S frames per launch)",
                         "algorithmic_bytes_per_launch": tot_bytes, "launch_ms": med_ms,
                         "achieved": ach, "peak": hbm_peak, "unit": "GB/s",
                         "frac": ach / hbm_peak,
                         "peak_source": "MEASURED_PEAKS.json" if peaks else "fallback"}
            if not raw else None,
            # integer pipe: the phase-1 + projection Hamming evaluations of the S
            # frames (8 POPC each) over the launch time, vs the POPC peak
            # measured in this run (ft_bench_popc)
            "roofline_int": {"bound": "popc", "kernel": "ft_track_frames (S frames per launch)",
                             "hamming_per_launch": tot_ham, "popc_per_launch": 8 * tot_ham,
                             "achieved_gpopc_s": 8 * tot_ham / (med_ms / 1e3) / 1e9,
                             "peak_gpopc_s": popc,
                             "frac": (8 * tot_ham / (med_ms / 1e3) / 1e9) / popc if popc else None},
            "build_levels": (pipe.build_levels if raw else None),
            "ms_per_step": float(np.mean(comp)),
            "frames_per_s": S * steps / (sum(comp) / 1e3),
            "e2e_frames_per_s": S * steps / (e2e_ms / 1e3),
            "h2d_bytes_per_step": shipped, "h2d_ranges_per_step": len(rngs),
            "packed_upload": bool(pipe.packed),
            "d2h_bytes_per_step": pipe.d2h_bytes()}

if __name__ == "__main__":
    main()
