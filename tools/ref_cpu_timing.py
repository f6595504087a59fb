"""CPU calibration of the reference arm (run in the build container, where
/root/reference exists): the reference's own numba path -- ExecutionEngine
"seq" (1 core) and "par" (all cores) -- against its C port (oracle/, what
`bench.py --impl reference` runs on the GPU box) on the SAME host and inputs:
the cfg1 ORB frame through phase 1 -> phase 2 -> reject (the reference's
golden inputs).  Median of >= 50 repetitions after warm-up.
    python tools/ref_cpu_timing.py > profiles/r2_reference_numba_vs_port.txt"""
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
sys.path.insert(0, str(ROOT / "tests" / "golden"))
import make_golden as MG  # noqa: E402  (reference imports + loaders)
from trackfront.engine import ExecutionEngine  # noqa: E402
from trackfront.stereo import (StereoMatchConfig, match_pinhole_phase1,  # noqa: E402
                               refine_match_phase2, reject_outliers)
from trackfront.synthetic import default_pinhole  # noqa: E402

import golden_io as G  # noqa: E402
from oracle import oracle as O  # noqa: E402
from paper_2509_10757_b200.types import StereoMatchConfig as OurCfg  # noqa: E402


def med_us(fn, n=60):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e6 * float(np.median(ts))


d = MG._load("cfg1_stereo.npz")
left, right = MG._feats(d, "left"), MG._feats(d, "right")
pl, pr = MG._pyr(d, "l"), MG._pyr(d, "r")
cam, cfg, sp = default_pinhole(), StereoMatchConfig(), d["scale_pow"]


def ref_stereo(engine):
    idx, dist = match_pinhole_phase1(left, right, cam.height, sp, cfg, engine=engine)
    m = refine_match_phase2(pl, pr, left, right, idx, dist, cam, cfg, engine=engine)
    return reject_outliers(m, cfg)


ncpu = os.cpu_count() or 1
rows = {}
for name, eng in (("reference numba seq (1 core)", ExecutionEngine("seq")),
                  (f"reference numba par ({ncpu} workers)", ExecutionEngine("par", workers=ncpu))):
    rows[name] = med_us(lambda: ref_stereo(eng))
gl, gr = G.feats(d, "left"), G.feats(d, "right")
gpl, gpr = G.pyramid(d, "l"), G.pyramid(d, "r")
gcam, gcfg = G.pinhole(), OurCfg()
O.lib()
for nt in (1, O.max_threads()):
    rows[f"C port (oracle/ft_oracle.c), {nt} thread(s)"] = med_us(
        lambda: O.stereo_pinhole(gl, gr, gpl, gpr, gcam, gcfg, d["scale_pow"], nt))
m_ref = ref_stereo(ExecutionEngine("seq"))
m_port = O.stereo_pinhole(gl, gr, gpl, gpr, gcam, gcfg, d["scale_pow"])
same = all(np.array_equal(getattr(m_ref, f), getattr(m_port, f)) for f in
           ("right_idx", "distance", "disparity", "refined_u", "depth", "sad"))
print(f"cfg1 ORB frame (1201 keypoints, phase 1 -> phase 2 -> reject), host: "
      f"{os.cpu_count()} CPUs (build container, not the GPU box); outputs identical: {same}")
for k, v in rows.items():
    print(f"  {k:45s} {v:9.1f} us / frame")
