"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 path: stream
sharding is a partition, and the max-over-ranks timing reduction / whole-job
throughput follow bench.py's contract."""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2509_10757_b200.sharding import (job_frames_per_s, max_over_ranks, rank_of_stream,
                                            streams_of_rank)


def test_streams_partition():
    for world in (1, 2, 4, 8):
        owned = [streams_of_rank(37, world, r) for r in range(world)]
        flat = sorted(s for o in owned for s in o)
        assert flat == list(range(37))
        for r, o in enumerate(owned):
            assert all(rank_of_stream(s, world) == r for s in o)
    with pytest.raises(ValueError):
        streams_of_rank(4, 2, 2)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mine = streams_of_rank(10, world, rank)
        # rank r "took" 10 + 5 r ms and processed len(mine) frames per step
        t = max_over_ranks([10.0 + 5.0 * rank, float(len(mine))], dist)
        dist.barrier()
        q.put((rank, mine, t))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_max_over_ranks():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0][1] == [0, 2, 4, 6, 8] and out[1][1] == [1, 3, 5, 7, 9]
    for _, _, t in out:
        assert t == [15.0, 5.0]  # every rank sees the slowest rank's time
    assert job_frames_per_s(5, world, 15.0) == pytest.approx(10 / 0.015)


def test_bench_self_launch_gloo_world2():
    """`python bench.py --gpus 2` outside torchrun launches two ranks itself
    (torch.distributed.run on 127.0.0.1) and rank 0 alone prints one line with
    n_gpus 2 -- the driver's N-GPU invocation, rehearsed on CPU over gloo."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parent.parent
    env = dict(os.environ, FT_BENCH_DIST_BACKEND="gloo")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--steps", "3",
                        "--dist-selftest"], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["max_ms"] == 11.0
