"""cProfile of bench.cfg4_sequence_run's two paths (drop-in seam, resident
pipeline) over the cfg4 line sequence."""
import cProfile
import pstats
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import bench  # noqa: E402

bench.cfg4_sequence_run(99)  # warm
pr = cProfile.Profile()
pr.enable()
out = bench.cfg4_sequence_run(99)
pr.disable()
print({k: v for k, v in out.items() if k != "workload"})
pstats.Stats(pr).sort_stats("tottime").print_stats(30)
